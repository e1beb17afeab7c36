// sm_100a kernels of the bucket-elimination backend.
//
//  * bucket_kernel     — one fused bucket over HBM: out[o] = sum_v prod_t T_t[idx_t(o,v)]
//                        (replaces the `_product` einsum chain + `.sum`,
//                        /root/reference/pkg/src/qtnsim/contraction.py:42-54, 90-96).
//                        The primary operand streams aligned with the output
//                        (16-byte vector loads), small operands are pre-multiplied
//                        into shared-memory lookup tables, the v-sum happens in
//                        registers, arithmetic in float64.
//  * smem_net_kernel   — a whole small network per warp, resident in shared
//                        memory: program, packed inputs and intermediates; one
//                        launch for many networks x many angle sets.
//  * tensorgen_kernel  — gate tensors generated on device from the angles
//                        (circuit.py:186-205 conventions, network.py:153-165 slicing).
//  * fold / energy     — scalar fold (contraction.py:77-81, 108-110) and the
//                        MaxCut energy sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "qtn_internal.h"
#include "qtn_setmajor.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

using namespace qtn;

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 ld_c(const void* p, uint64_t i, uint32_t c64) {
  if (c64) {
    float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return make_double2(f.x, f.y);
  }
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
__device__ __forceinline__ void st_c(void* p, uint64_t i, uint32_t c64, double2 v) {
  if (c64)
    reinterpret_cast<float2*>(p)[i] = make_float2((float)v.x, (float)v.y);
  else
    reinterpret_cast<double2*>(p)[i] = v;
}
__device__ __forceinline__ uint64_t gather64(uint64_t o, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((o >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}
__device__ __forceinline__ uint64_t gather_lo(uint32_t e, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= (uint64_t)((e >> s) & ((1u << l) - 1)) << d;
  }
  return idx;
}

constexpr int kThreads = 256;

// Element-wise body shared by both kernel variants: accumulate every
// non-primary operand (gathered or tabulated) for output o = obase + e.
__device__ __forceinline__ void accumulate_rest(const BucketArgs& a, uint32_t g_first, uint32_t e,
                                                const uint64_t* gbase, const uint32_t* tbase,
                                                const double2* tab, double2& a0, double2& a1) {
#pragma unroll
  for (int i = 0; i < kMaxG; ++i) {
    if (i < (int)g_first || i >= (int)a.ng) continue;
    const GOpArg& g = a.g[i];
    const uint64_t idx = gbase[i] + gather_lo(e, g.lo, g.n_lo);
    a0 = cmul(a0, ld_c(g.ptr, idx, g.c64));
    a1 = cmul(a1, ld_c(g.ptr, idx + (1ull << g.vshift), g.c64));
  }
#pragma unroll
  for (int j = 0; j < kMaxT; ++j) {
    if (j >= (int)a.nt) continue;
    const TableArg& t = a.t[j];
    const uint32_t ti = (tbase[j] | (uint32_t)gather_lo(e, t.lo, t.n_lo)) << 1;
    const double2* tp = tab + t.smem_off + ti;
    a0 = cmul(a0, tp[0]);
    a1 = cmul(a1, tp[1]);
  }
}

template <bool kFast>
__global__ void __launch_bounds__(kThreads) bucket_kernel(const __grid_constant__ BucketArgs a) {
  extern __shared__ double2 tab[];
  // ---- lookup tables: T_j[bits, v] = prod over the folded small operands
  for (uint32_t j = 0; j < a.nt; ++j) {
    const TableArg& t = a.t[j];
    const uint32_t n = 2u << t.nbits;
    for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
      const uint32_t bits = e >> 1, v = e & 1;
      double2 acc = make_double2(1.0, 0.0);
      for (uint32_t k = 0; k < t.n_ops; ++k) {
        const TOpArg& op = a.top[t.first_op + k];
        const uint64_t idx = gather_lo(bits, op.runs, op.n_runs) | ((uint64_t)v << op.vshift);
        acc = cmul(acc, ld_c(op.ptr, idx, op.c64));
      }
      tab[t.smem_off + e] = acc;
    }
  }
  __syncthreads();

  const uint32_t tile_bits = a.R < (uint32_t)kTileBits ? a.R : (uint32_t)kTileBits;
  const uint64_t n_tiles = a.n_out >> tile_bits;
  const uint32_t tile_elems = 1u << tile_bits;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t obase = tile << tile_bits;
    uint64_t gbase[kMaxG];
    uint32_t tbase[kMaxT];
#pragma unroll
    for (int i = 0; i < kMaxG; ++i)
      gbase[i] = i < (int)a.ng ? gather64(obase, a.g[i].hi, a.g[i].n_hi) : 0;
#pragma unroll
    for (int j = 0; j < kMaxT; ++j)
      tbase[j] = j < (int)a.nt ? (uint32_t)gather64(obase, a.t[j].hi, a.t[j].n_hi) : 0;

    if constexpr (kFast) {
      // primary complex64, aligned, output complex64: two outputs per thread,
      // 16-byte loads/stores.  tile_elems >= 2 here.
      const GOpArg& p = a.g[0];
      const float* P = reinterpret_cast<const float*>(p.ptr);
      float* O = reinterpret_cast<float*>(a.out);
      const uint64_t vstep = 1ull << a.p_k;
#pragma unroll 4
      for (uint32_t e = 2 * threadIdx.x; e < tile_elems; e += 2 * kThreads) {
        const uint64_t idx = gbase[0] + gather_lo(e, p.lo, p.n_lo);
        float4 x, y;
        double2 a0, a1, b0, b1;  // (o,v=0) (o,v=1) (o+1,v=0) (o+1,v=1)
        if (a.p_k == 0) {
          x = __ldg(reinterpret_cast<const float4*>(P + 2 * idx));
          y = __ldg(reinterpret_cast<const float4*>(P + 2 * (idx + 2)));
          a0 = make_double2(x.x, x.y); a1 = make_double2(x.z, x.w);
          b0 = make_double2(y.x, y.y); b1 = make_double2(y.z, y.w);
        } else {
          x = __ldg(reinterpret_cast<const float4*>(P + 2 * idx));
          y = __ldg(reinterpret_cast<const float4*>(P + 2 * (idx + vstep)));
          a0 = make_double2(x.x, x.y); b0 = make_double2(x.z, x.w);
          a1 = make_double2(y.x, y.y); b1 = make_double2(y.z, y.w);
        }
        accumulate_rest(a, 1, e, gbase, tbase, tab, a0, a1);
        accumulate_rest(a, 1, e + 1, gbase, tbase, tab, b0, b1);
        const double2 r0 = cadd(a0, a1), r1 = cadd(b0, b1);
        float4 r = make_float4((float)r0.x, (float)r0.y, (float)r1.x, (float)r1.y);
        *reinterpret_cast<float4*>(O + 2 * (obase + e)) = r;
      }
    } else {
      for (uint32_t e = threadIdx.x; e < tile_elems; e += kThreads) {
        double2 a0 = make_double2(1.0, 0.0), a1 = a0;
        accumulate_rest(a, 0, e, gbase, tbase, tab, a0, a1);
        st_c(a.out, obase + e, a.out_c64, cadd(a0, a1));
      }
    }
  }
}

int g_num_sms = 0;

int cuda_fail(cudaError_t e, const char* what) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  set_error(buf);
  return QTN_ECUDA;
}

// ------------------------------------------------------- SMEM executor

__device__ __forceinline__ void copy16(void* dst, const void* src, uint32_t bytes, uint32_t t,
                                       uint32_t nt) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  const uint32_t n = bytes / 16;
  uint32_t i = t;
  for (; i + 3 * nt < n; i += 4 * nt) {
    uint4 x0 = __ldg(s + i), x1 = __ldg(s + i + nt), x2 = __ldg(s + i + 2 * nt),
          x3 = __ldg(s + i + 3 * nt);
    d[i] = x0; d[i + nt] = x1; d[i + 2 * nt] = x2; d[i + 3 * nt] = x3;
  }
  for (; i < n; i += nt) d[i] = __ldg(s + i);
}

// Gate tensor entry from the parameter phase ph = e^{-it} (or a literal).
__device__ __forceinline__ double2 gen_entry(uint32_t kind, uint32_t i, double2 ph) {
  const double s = 0.70710678118654757;  // 1/sqrt(2), circuit.py:179
  switch (kind) {
    case QTN_GATE_INIT: return make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    case QTN_GATE_H: return make_double2(i == 3 ? -s : s, 0.0);
    case QTN_GATE_ZPOW: return i == 0 ? make_double2(1.0, 0.0) : (i == 3 ? ph : make_double2(0.0, 0.0));
    case QTN_GATE_ZPOW_DIAG: return i == 0 ? make_double2(1.0, 0.0) : ph;
    case QTN_GATE_XPOW: {
      const bool d = (i == 0 || i == 3);
      return d ? make_double2(0.5 * (1.0 + ph.x), 0.5 * ph.y) : make_double2(0.5 * (1.0 - ph.x), -0.5 * ph.y);
    }
    case QTN_GATE_CNOT: {
      const uint32_t row = i >> 2, col = i & 3;
      return make_double2(col == (row < 2 ? row : (row ^ 1)) ? 1.0 : 0.0, 0.0);
    }
    case QTN_GATE_ZZ: {  // diag(r, r*, r*, r), r = e^{i g} = conj(ph)
      const uint32_t row = i >> 2, col = i & 3;
      if (row != col) return make_double2(0.0, 0.0);
      return (row == 0 || row == 3) ? make_double2(ph.x, -ph.y) : ph;
    }
    case QTN_GATE_ZZ_DIAG: return (i == 0 || i == 3) ? make_double2(ph.x, -ph.y) : ph;
    case QTN_GATE_SCALAR: return ph;
  }
  return make_double2(0.0, 0.0);
}

struct SmemArgs {
  const uint8_t* progs;
  const uint64_t* prog_off;
  const uint64_t* in_off;
  const int32_t* out_index;
  const double2* inputs;       // packed inputs (NULL when generating from angles)
  int64_t set_elems;
  double2* results;
  const double* angles;        // n_sets x n_angles (NULL: copy inputs)
  int32_t n_angles;
  int32_t n_sets;
  int32_t n_total;
  uint32_t prog_max;           // bytes reserved for the program (CTA-shared)
  uint32_t set_bytes;          // bytes of one angle set's data region
  int32_t lanes_per_set;       // L: lanes per set (power of two); 32/L sets per warp
};

constexpr int kNetWarps = 4;   // warps per CTA (upper bound)

// One CTA = one network.  A warp evaluates G = 32/L angle sets; each set is
// handled by L lanes (L = A.lanes_per_set, a power of two).  With L = 1
// every lane runs the whole bucket program for its own set, sequentially,
// with no cross-lane dependency at all; larger L splits each bucket's
// outputs over L lanes (for networks whose per-set data is too large to
// keep 32 sets resident).  Set s's element x lives at D[G*x + s]: lanes of
// different sets hit different banks.  The program, gather tables and
// generator entries are staged once per CTA and read as warp-uniform
// broadcasts; every operand index is one table lookup (two for R > 5);
// input tensors are generated from the set's angles right before their
// bucket.
__global__ void __launch_bounds__(32 * kNetWarps) smem_net_kernel(const __grid_constant__ SmemArgs A) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int net = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = A.lanes_per_set, G = 32 / L;
  const int sub = lane & (L - 1), gs = lane / L;  // lane within the set, set within the warp
  const int wset0 = (blockIdx.y * (int)(blockDim.x >> 5) + warp) * G;
  const int set = wset0 + gs;
  const uint8_t* gp = A.progs + A.prog_off[net];
  const SmemHeader h = *reinterpret_cast<const SmemHeader*>(gp);
  copy16(sm, gp, h.prog_bytes, threadIdx.x, blockDim.x);
  __syncthreads();
  if (wset0 >= A.n_sets) return;
  const bool live = set < A.n_sets;
  double2* D = reinterpret_cast<double2*>(sm + A.prog_max + (size_t)warp * G * A.set_bytes) + gs;
  const bool gen = A.angles && h.n_recs;
  const SmemGenRec* grec = reinterpret_cast<const SmemGenRec*>(sm + h.gen_off +
                                                               sizeof(SmemGenParam) * h.n_params);
  const SmemIn* sin = reinterpret_cast<const SmemIn*>(sm + h.in_off);
  const double2* src_in = A.inputs + (int64_t)(live ? set : 0) * A.set_elems + A.in_off[net];
  if (gen) {
    const SmemGenParam* par = reinterpret_cast<const SmemGenParam*>(sm + h.gen_off);
    const double* ang = A.angles + (int64_t)(live ? set : 0) * A.n_angles;
    for (uint32_t k = sub; k < h.n_params; k += L) {
      const SmemGenParam q = par[k];
      double2 ph;
      if (q.angle == -2) {
        ph = make_double2(q.scale, q.offset);
      } else {
        const double t = q.angle >= 0 ? q.scale * ang[q.angle] + q.offset : q.offset;
        double sn, cs;
        sincos(t, &sn, &cs);
        ph = make_double2(cs, -sn);
      }
      D[G * (h.data_elems + k)] = ph;
    }
    if (L > 1) __syncwarp();
  }
  auto materialise = [&](uint32_t gfirst, uint32_t gcnt, uint32_t first, uint32_t cnt) {
    if (gen) {
      for (uint32_t i = gfirst + sub; i < gfirst + gcnt; i += L) {
        const SmemGenRec g = grec[i];
        D[G * g.sm_off] = gen_entry(g.kind, g.full, D[G * (h.data_elems + g.param)]);
      }
    } else {
      for (uint32_t i = first; i < first + cnt; ++i) {
        const SmemIn r = sin[i];
        for (uint32_t e = sub; e < (1u << r.rank); e += L) D[G * (r.sm_off + e)] = src_in[r.in_off + e];
      }
    }
    if (L > 1) __syncwarp();
  };
  materialise(0, h.n_init_gen, 0, h.n_init);
  const SmemBucket* bk = reinterpret_cast<const SmemBucket*>(sm + sizeof(SmemHeader));
  const SmemOp* ops = reinterpret_cast<const SmemOp*>(sm + sizeof(SmemHeader) +
                                                      sizeof(SmemBucket) * h.n_buckets);
  const uint16_t* tab = reinterpret_cast<const uint16_t*>(sm + h.tab_off);
  for (uint32_t bi = 0; bi < h.n_buckets; ++bi) {
    const SmemBucket b = bk[bi];
    materialise(b.first_gen, b.n_gen, b.first_in, b.n_in);
    const SmemOp* bo = ops + b.first_op;
    const uint32_t R = b.R;
    const uint32_t n = 1u << R;
    for (uint32_t e = sub; e < n; e += L) {
      const uint32_t hi_e = e >> 5, lo_e = e & 31;
      SmemOp o = bo[0];
      uint32_t idx = o.off + tab[o.lo + lo_e] + (R > 5 ? tab[o.hi + hi_e] : 0u);
      double2 a0 = D[G * idx], a1 = D[G * (idx + o.vstep)];
      for (uint32_t k = 1; k < b.n_ops; ++k) {
        o = bo[k];
        idx = o.off + tab[o.lo + lo_e] + (R > 5 ? tab[o.hi + hi_e] : 0u);
        a0 = cmul(a0, D[G * idx]);
        a1 = cmul(a1, D[G * (idx + o.vstep)]);
      }
      D[G * (b.out_off + e)] = cadd(a0, a1);
    }
    if (L > 1) __syncwarp();
  }
  if (live && sub == 0) {
    const uint16_t* sc = reinterpret_cast<const uint16_t*>(
        sm + sizeof(SmemHeader) + sizeof(SmemBucket) * h.n_buckets + sizeof(SmemOp) * h.n_ops);
    double2 r = make_double2(ldexp(1.0, (int)h.pow2), 0.0);
    for (uint32_t i = 0; i < h.n_scalars; ++i) r = cmul(r, D[G * sc[i]]);
    A.results[(int64_t)set * A.n_total + A.out_index[net]] = r;
  }
}

// Final scalar fold of the HBM-executor networks: 2^n_empty times every
// rank-0 tensor (contraction.py:77-81, 108-110), one thread per (network, set).
__global__ void hbm_fold_kernel(const uint64_t* __restrict__ tags, const uint8_t* __restrict__ c64,
                                const uint32_t* __restrict__ first, const int32_t* __restrict__ pow2,
                                const int32_t* __restrict__ out_index, int n_hbm, int n_total,
                                const char* in_base, int64_t in_set_stride,
                                const int64_t* __restrict__ net_in_off, const char* ws_base,
                                int64_t ws_set_stride, const int64_t* __restrict__ net_ws_off,
                                double2* __restrict__ results) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_hbm) return;
  const int set = blockIdx.y;
  const char* in = in_base + (int64_t)set * in_set_stride + net_in_off[i];
  const char* ws = ws_base + (int64_t)set * ws_set_stride + net_ws_off[i];
  double2 r = make_double2(ldexp(1.0, pow2[i]), 0.0);
  for (uint32_t k = first[i]; k < first[i + 1]; ++k) {
    const uint64_t t = tags[k];
    const uint64_t sel = t >> kSelShift, off = t & kOffMask;
    const char* p = sel == 1 ? in + off : (sel == 2 ? ws + off : reinterpret_cast<const char*>(off));
    r = cmul(r, ld_c(p, 0, c64[k]));
  }
  results[(int64_t)set * n_total + out_index[i]] = r;
}

struct FoldArgs {
  const void* ptrs[32];
  uint8_t c64[32];
};
__global__ void fold_kernel_p(const __grid_constant__ FoldArgs f, int n, int pow2,
                              double2* result, int accumulate) {
  double2 r = accumulate ? *result : make_double2(ldexp(1.0, pow2), 0.0);
  for (int i = 0; i < n; ++i) r = cmul(r, ld_c(f.ptrs[i], 0, f.c64[i]));
  *result = r;
}

// ------------------------------------------------------- tensor generation

__device__ double2 gate_entry(int kind, double t, uint32_t i, double sre, double sim) {
  const double s = 0.70710678118654757;  // 1/sqrt(2), circuit.py:179
  double sn, cs;
  switch (kind) {
    case QTN_GATE_INIT:
      return make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    case QTN_GATE_H:
      return make_double2(i == 3 ? -s : s, 0.0);
    case QTN_GATE_ZPOW:  // diag(1, e^{-it})
      if (i == 0) return make_double2(1.0, 0.0);
      if (i == 3) { sincos(t, &sn, &cs); return make_double2(cs, -sn); }
      return make_double2(0.0, 0.0);
    case QTN_GATE_ZPOW_DIAG:
      if (i == 0) return make_double2(1.0, 0.0);
      sincos(t, &sn, &cs);
      return make_double2(cs, -sn);
    case QTN_GATE_XPOW: {  // H diag(1, e) H = 1/2 [[1+e, 1-e], [1-e, 1+e]]
      sincos(t, &sn, &cs);
      const bool diag = (i == 0 || i == 3);
      return diag ? make_double2(0.5 * (1.0 + cs), -0.5 * sn)
                  : make_double2(0.5 * (1.0 - cs), 0.5 * sn);
    }
    case QTN_GATE_CNOT: {  // row = i >> 2, col = i & 3
      const uint32_t row = i >> 2, col = i & 3;
      const uint32_t img = row < 2 ? row : (row ^ 1);
      return make_double2(col == img ? 1.0 : 0.0, 0.0);
    }
    case QTN_GATE_ZZ: {  // diag(r, r*, r*, r), r = e^{i g}
      const uint32_t row = i >> 2, col = i & 3;
      if (row != col) return make_double2(0.0, 0.0);
      sincos(t, &sn, &cs);
      return (row == 0 || row == 3) ? make_double2(cs, sn) : make_double2(cs, -sn);
    }
    case QTN_GATE_ZZ_DIAG: {
      sincos(t, &sn, &cs);
      return (i == 0 || i == 3) ? make_double2(cs, sn) : make_double2(cs, -sn);
    }
    case QTN_GATE_SCALAR:
      return make_double2(sre, sim);
  }
  return make_double2(0.0, 0.0);
}

__global__ void tensorgen_kernel(const qtn_tensor_recipe* __restrict__ rec, int64_t n,
                                 const double* __restrict__ angles, int n_angles,
                                 int64_t set_elems, double2* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int set = blockIdx.y;
  const qtn_tensor_recipe r = rec[k];
  const double t = r.angle >= 0 ? r.scale * angles[(int64_t)set * n_angles + r.angle] + r.offset
                                : r.offset;
  const int fr = r.full_rank;
  int kept = 0;
  for (int q = 0; q < fr; ++q) kept += (r.keep_mask >> q) & 1;
  double2* dst = out + (int64_t)set * set_elems + r.out_offset;
  for (uint32_t e = 0; e < (1u << kept); ++e) {
    uint32_t full = 0;
    int kb = kept - 1;
    for (int q = 0; q < fr; ++q) {  // position q is the (fr-1-q)th bit, MSB first
      uint32_t bit;
      if ((r.keep_mask >> q) & 1) bit = (e >> kb--) & 1;
      else bit = (r.fixed_bits >> q) & 1;
      full = (full << 1) | bit;
    }
    dst[e] = gate_entry(r.kind, t, full, r.scale, r.offset);
  }
}

// One 128-thread CTA per input set: strided partial sums, then a fixed-order
// shuffle + shared-memory tree (deterministic for a given n).
__global__ void __launch_bounds__(128) energy_kernel(const double2* __restrict__ vals,
                                                     const double* __restrict__ w, int n,
                                                     double* energies, double2* zz) {
  const int s = blockIdx.x;
  double e = 0.0, zr = 0.0, zi = 0.0;
  for (int i = threadIdx.x; i < n; i += 128) {
    const double2 v = vals[(int64_t)s * n + i];
    e += ((w ? w[i] : 1.0) - v.x) / 2.0;
    zr += v.x;
    zi += v.y;
  }
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_xor_sync(0xffffffffu, e, o);
    zr += __shfl_xor_sync(0xffffffffu, zr, o);
    zi += __shfl_xor_sync(0xffffffffu, zi, o);
  }
  __shared__ double red[3][4];
  const int wp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][wp] = e;
    red[1][wp] = zr;
    red[2][wp] = zi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    e = (red[0][0] + red[0][1]) + (red[0][2] + red[0][3]);
    zr = (red[1][0] + red[1][1]) + (red[1][2] + red[1][3]);
    zi = (red[2][0] + red[2][1]) + (red[2][2] + red[2][3]);
    if (energies) energies[s] = e;
    if (zz) zz[s] = make_double2(zr, zi);
  }
}

}  // namespace

namespace qtn {

int device_check() {
  if (g_num_sms > 0) return QTN_OK;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device: the B200 backend has no CPU fallback");
    return QTN_ENODEV;
  }
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return QTN_OK;
}

int launch_bucket(const BucketArgs& a, void* stream) {
  int rc = device_check();
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint32_t tile_bits = a.R < (uint32_t)kTileBits ? a.R : (uint32_t)kTileBits;
  const uint64_t n_tiles = a.n_out >> tile_bits;
  const size_t smem = (size_t)a.table_entries * sizeof(double2);
  const bool fast = a.primary && a.ng >= 1 && a.g[0].c64 && a.out_c64 && a.R >= 1;
  static std::atomic<uint64_t> attr_set{0};
  if (needs_setup(attr_set)) {
    cudaFuncSetAttribute(bucket_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(bucket_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    mark_setup(attr_set);
  }
  const uint64_t max_blocks = (uint64_t)g_num_sms * 8;
  const unsigned blocks = (unsigned)std::min<uint64_t>(n_tiles, max_blocks);
  if (fast)
    bucket_kernel<true><<<blocks, kThreads, smem, st>>>(a);
  else
    bucket_kernel<false><<<blocks, kThreads, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "bucket_kernel launch");
  return QTN_OK;
}

int launch_fold(const void* const* ptrs, const uint8_t* c64, int n, int pow2, void* result,
                bool accumulate, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int done = 0;
  bool acc = accumulate;
  do {
    FoldArgs f;
    std::memset(&f, 0, sizeof(f));
    const int m = std::min(32, n - done);
    for (int i = 0; i < m; ++i) {
      f.ptrs[i] = ptrs[done + i];
      f.c64[i] = c64[done + i];
    }
    fold_kernel_p<<<1, 1, 0, st>>>(f, m, pow2, reinterpret_cast<double2*>(result), acc ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fold_kernel launch");
    done += m;
    acc = true;
  } while (done < n);
  return QTN_OK;
}

int device_alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) {
    cuda_fail(e, "cudaMalloc");
    return QTN_ENOMEM;
  }
  return QTN_OK;
}
int device_free(void* p) {
  if (p) cudaFree(p);
  return QTN_OK;
}
int h2d(void* dst, const void* src, size_t bytes) {
  cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
  return QTN_OK;
}

}  // namespace qtn

// ------------------------------------------------------------- batches

template <typename T>
static int upload(T** dst, const std::vector<T>& v) {
  int rc = device_alloc((void**)dst, std::max<size_t>(v.size(), 1) * sizeof(T));
  if (rc) return rc;
  if (!v.empty()) rc = h2d(*dst, v.data(), v.size() * sizeof(T));
  return rc;
}

// The launch sequence of one evaluation (tensorgen, level launches, folds)
// is captured once per (buffers, set count) into a CUDA graph and replayed:
// one launch instead of up to ~80 (QTN_GRAPHS=0 disables).
struct GraphKey {
  const void *angles, *inputs, *ws, *results;
  int32_t n_angles, n_sets;
  bool sm;
  bool operator<(const GraphKey& o) const {
    return std::tie(angles, inputs, ws, results, n_angles, n_sets, sm) <
           std::tie(o.angles, o.inputs, o.ws, o.results, o.n_angles, o.n_sets, o.sm);
  }
};

struct qtn_batch {
  int n = 0;
  int64_t set_elems = 0;
  std::vector<int64_t> in_offsets;
  // SMEM executor part
  int n_smem = 0;
  int64_t max_smem = 0;
  uint8_t* d_prog = nullptr;
  uint64_t* d_prog_off = nullptr;
  uint64_t* d_in_off = nullptr;
  int32_t* d_smem_index = nullptr;
  std::vector<std::vector<uint8_t>> smem_progs;  // host copies (gen sections appended later)
  std::vector<int32_t> smem_global;              // batch index of each SMEM network
  uint32_t prog_max = 0;                         // bytes reserved per CTA for the program
  uint32_t warp_bytes = 0;                       // bytes per warp data region
  bool has_recipes = false;
  qtn::SetMajor* sm = nullptr;                   // set-major form of the SMEM networks
  std::vector<const qtn_plan*> smem_plans;
  qtn_tensor_recipe* d_hbm_rec = nullptr;        // recipes of the HBM networks
  int64_t n_hbm_rec = 0;
  // HBM executor part (level-synchronous)
  int n_hbm = 0;
  int64_t ws_per_set = 0;
  uint8_t* d_desc = nullptr;
  uint64_t* d_item_desc = nullptr;
  uint32_t* d_item_net = nullptr;
  uint64_t* d_tile_prefix = nullptr;
  int64_t* d_net_in_off = nullptr;
  int64_t* d_net_ws_off = nullptr;
  std::vector<uint32_t> level_item0;    // first item of each level (+ end)
  std::vector<uint64_t> level_prefix0;  // first prefix entry of each level
  std::vector<uint64_t> level_tiles;    // tiles of one set per level
  // small buckets (R <= kSmallR) of each level: warp-per-bucket kernel
  uint64_t* d_sitem_desc = nullptr;
  uint32_t* d_sitem_net = nullptr;
  std::vector<uint32_t> level_sitem0;   // first small item of each level (+ end)
  std::vector<uint32_t> level_smax_r;   // widest small item of each level
  std::vector<uint8_t> level_tiny;      // small_kernel-only level with <= QTN_CHAIN_ELEMS outputs
  std::vector<uint32_t> chain_len;      // per level: length of the tiny-level chain starting here (0: none)
  uint32_t* d_level_sitem0 = nullptr;
  // single-operand buckets of each level (trace_kernel)
  qtn::R1Dev* d_r1 = nullptr;
  uint64_t* d_r1prefix = nullptr;
  std::vector<uint32_t> level_r1item0;  // first trace item of each level (+ end)
  std::vector<uint64_t> level_r1prefix0, level_r1chunks, level_r1chunk0;
  uint32_t* d_r1chunk_item = nullptr;   // per trace chunk: its item within the level
  // expanding buckets of each level (expand_kernel)
  qtn::XDesc* d_xdesc = nullptr;
  uint32_t* d_xitem_desc = nullptr;
  uint32_t* d_xitem_net = nullptr;
  uint64_t* d_xprefix = nullptr;
  std::vector<uint32_t> level_xitem0;   // first expand item of each level (+ end)
  std::vector<uint64_t> level_xprefix0, level_xtiles;
  std::vector<uint32_t> level_xstage;   // stage bytes (max over the level's items)
  // expanding bucket + consumer pairs (xt_kernel), same shape as the expand lists
  qtn::YDesc* d_ydesc = nullptr;
  uint32_t* d_yitem_desc = nullptr;
  uint32_t* d_yitem_net = nullptr;
  uint64_t* d_yprefix = nullptr;
  std::vector<uint32_t> level_yitem0;
  std::vector<uint64_t> level_yprefix0, level_ytiles;
  std::vector<uint32_t> level_ystage;
  // weighted full sums: the tail chains (wsum_kernel)
  qtn::WsDesc* d_wsdesc = nullptr;
  uint32_t* d_wsitem_desc = nullptr;
  uint32_t* d_wsitem_net = nullptr;
  uint32_t* d_wsprefix = nullptr;
  std::vector<uint32_t> level_ws0;      // first tail item of each level (+ end)
  std::vector<uint32_t> level_wsprefix0, level_wsctas;
  // fused product chains per level (fused_kernel)
  qtn::FDesc* d_fdesc = nullptr;
  uint32_t* d_ftab = nullptr;
  qtn::FCta* d_fctas = nullptr;
  uint8_t* d_fblob = nullptr;
  uint32_t* d_fitem_desc = nullptr;
  uint32_t* d_fitem_net = nullptr;
  uint64_t* d_fprefix = nullptr;
  uint64_t* d_cprefix = nullptr;        // split items: combine CTAs (units)
  // a level's fused items in groups of one math type (one launch each):
  // items [item0, item0 + n_items), CTA prefix at fprefix[prefix0 ..]
  struct FGroup {
    uint32_t item0, n_items;
    uint64_t prefix0, ctas, cctas;
    uint64_t cta0;                      // first per-CTA record (fused_kernel)
    uint32_t smem;
    uint8_t f64;
    uint8_t warp;                       // warp-granular chains (fusedw_kernel): recs [cta0, cta0 + ctas)
  };
  std::vector<FGroup> fgroups;
  uint8_t* d_wblob = nullptr;           // warp-granular chain blobs (qtn_fusedw.cu)
  qtn::WRec* d_wrecs = nullptr;         // one record per warp of one set
  std::vector<uint32_t> level_fgroup0;  // first group of each level (+ end)
  std::vector<uint64_t> level_fctas;    // fused CTAs of one set per level (0: none)
  // tiny subtrees per level (subtree_kernel)
  qtn::SubItem* d_sub_items = nullptr;
  uint64_t* d_sub_desc = nullptr;
  std::vector<uint32_t> level_sub0;     // first subtree item of each level (+ end)
  std::vector<uint32_t> level_sub_smem;
  // fused single-operand chains per level (reduce_kernel)
  qtn::RedDev* d_red = nullptr;
  uint32_t* d_red_prefix = nullptr;
  std::vector<uint32_t> level_red0, level_rprefix0, level_rchunks;
  // captured evaluations (qtn_batch_execute_angles)
  std::map<GraphKey, cudaGraphExec_t> graphs;
  // captured host-facing calls (qtn_batch_energies_host): angles H2D from the
  // pinned staging, the evaluation, the energy reduction and the D2H
  std::map<std::vector<uintptr_t>, cudaGraphExec_t> egraphs;
  cudaStream_t cap_stream = nullptr;
  // concurrent launches of one HBM level (independent buckets): side
  // streams forked from / joined into the caller's stream with events
  static constexpr int kSide = 7;  // up to 8 concurrent launches per level
  // network groups (QTN_HBM_GROUPS): each an independent level sequence on
  // its own stream lane (group 0: the caller's stream), with its own side
  // streams for the concurrent launches of a level
  static constexpr int kMaxGroups = 4;
  int n_groups = 1;
  int32_t lev_per_group = 0;
  cudaStream_t gside[kMaxGroups][kSide] = {};
  cudaEvent_t gfork[kMaxGroups] = {};
  cudaEvent_t gjoin[kMaxGroups][kSide] = {};
  cudaStream_t lane[kMaxGroups] = {};
  cudaEvent_t ev_lanes = nullptr;
  cudaEvent_t ev_lane_done[kMaxGroups] = {};
  // pinned staging of qtn_batch_energies_host
  double* pin = nullptr;
  size_t pin_doubles = 0;
  uint64_t* d_fold_tags = nullptr;
  uint8_t* d_fold_c64 = nullptr;
  uint32_t* d_fold_first = nullptr;
  int32_t* d_fold_pow2 = nullptr;
  int32_t* d_hbm_index = nullptr;
};

// xt_kernel launches of one level (one per group count present)
static int y_launches(const qtn_batch* B, size_t lev) {
  int c = 0;
  for (int gq = 0; gq <= qtn::kYMaxGB; ++gq) c += B->level_ytiles[lev * (qtn::kYMaxGB + 1) + gq] ? 1 : 0;
  return c;
}

extern "C" int qtn_batch_destroy(qtn_batch* B) {
  if (!B) return QTN_OK;
  for (auto& kv : B->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : B->egraphs) cudaGraphExecDestroy(kv.second);
  if (B->cap_stream) cudaStreamDestroy(B->cap_stream);
  for (int g = 0; g < qtn_batch::kMaxGroups; ++g) {
    for (int k = 0; k < qtn_batch::kSide; ++k) {
      if (B->gside[g][k]) cudaStreamDestroy(B->gside[g][k]);
      if (B->gjoin[g][k]) cudaEventDestroy(B->gjoin[g][k]);
    }
    if (B->gfork[g]) cudaEventDestroy(B->gfork[g]);
    if (B->lane[g]) cudaStreamDestroy(B->lane[g]);
    if (B->ev_lane_done[g]) cudaEventDestroy(B->ev_lane_done[g]);
  }
  if (B->ev_lanes) cudaEventDestroy(B->ev_lanes);
  if (B->pin) cudaFreeHost(B->pin);
  for (void* p : {(void*)B->d_prog, (void*)B->d_prog_off, (void*)B->d_in_off,
                  (void*)B->d_smem_index, (void*)B->d_desc, (void*)B->d_item_desc,
                  (void*)B->d_item_net, (void*)B->d_tile_prefix, (void*)B->d_net_in_off,
                  (void*)B->d_net_ws_off, (void*)B->d_fold_tags, (void*)B->d_fold_c64,
                  (void*)B->d_fold_first, (void*)B->d_fold_pow2, (void*)B->d_hbm_index,
                  (void*)B->d_hbm_rec, (void*)B->d_sitem_desc, (void*)B->d_sitem_net,
                  (void*)B->d_red, (void*)B->d_red_prefix, (void*)B->d_xdesc,
                  (void*)B->d_wblob, (void*)B->d_wrecs,
                  (void*)B->d_xitem_desc, (void*)B->d_xitem_net, (void*)B->d_xprefix,
                  (void*)B->d_ydesc, (void*)B->d_yitem_desc, (void*)B->d_yitem_net, (void*)B->d_yprefix,
                  (void*)B->d_level_sitem0, (void*)B->d_r1, (void*)B->d_r1prefix, (void*)B->d_r1chunk_item,
                  (void*)B->d_fdesc, (void*)B->d_fitem_desc, (void*)B->d_fitem_net,
                  (void*)B->d_fprefix, (void*)B->d_cprefix, (void*)B->d_ftab,
                  (void*)B->d_fctas, (void*)B->d_fblob,
                  (void*)B->d_sub_items, (void*)B->d_sub_desc, (void*)B->d_wsdesc,
                  (void*)B->d_wsitem_desc, (void*)B->d_wsitem_net, (void*)B->d_wsprefix})
    device_free(p);
  qtn::setmajor_destroy(B->sm);
  delete B;
  return QTN_OK;
}

extern "C" int qtn_batch_create(qtn_plan* const* plans, int32_t n, qtn_batch** out) {
  if (!plans || n < 1 || !out) {
    set_error("qtn_batch_create: bad arguments");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  qtn_batch* B = new qtn_batch();
  B->n = n;
  // input layout shared by both executors: networks in order, 32-byte aligned
  int64_t in = 0;
  for (int i = 0; i < n; ++i) {
    if (!plans[i]) {
      delete B;
      set_error("qtn_batch_create: null plan");
      return QTN_EINVAL;
    }
    B->in_offsets.push_back(in);
    in += (plans[i]->input_elems + 1) & ~1ll;
  }
  B->set_elems = std::max<int64_t>(in, 2);
  // ---- SMEM networks
  std::vector<uint8_t> blob;
  std::vector<uint64_t> poff, ioff;
  std::vector<int32_t> sidx;
  // ---- HBM networks
  std::vector<uint8_t> desc;
  std::vector<int32_t> hidx;
  std::vector<int64_t> net_in, net_ws;
  int32_t max_lev = 0;
  for (int i = 0; i < n; ++i) {
    const qtn_plan* P = plans[i];
    if (P->executor == QTN_EXEC_SMEM) {
      B->smem_progs.push_back(P->program);
      B->smem_plans.push_back(P);
      B->smem_global.push_back(i);
      B->prog_max = std::max<uint32_t>(B->prog_max, (uint32_t)P->program.size());
      {
        const SmemHeader* hh = reinterpret_cast<const SmemHeader*>(P->program.data());
        B->warp_bytes = std::max<uint32_t>(B->warp_bytes, 16u * hh->data_elems);
      }
      poff.push_back(blob.size());
      blob.insert(blob.end(), P->program.begin(), P->program.end());
      ioff.push_back((uint64_t)B->in_offsets[i]);
      sidx.push_back(i);
      B->max_smem = std::max(B->max_smem, P->smem_bytes);
    } else {
      hidx.push_back(i);
      net_in.push_back(16 * B->in_offsets[i]);
      net_ws.push_back(B->ws_per_set);
      B->ws_per_set += (P->workspace_bytes + 255) & ~255ll;
      max_lev = std::max(max_lev, P->n_levels);
    }
  }
  B->n_smem = (int)sidx.size();
  B->n_hbm = (int)hidx.size();
  // QTN_HBM_ALIGN=1: shallower networks run at the end of the level range
  // (whole networks move, so their arena lifetimes stay valid)
  std::vector<int32_t> hshift(B->n_hbm, 0);
  {
    const char* av = getenv("QTN_HBM_ALIGN");
    if (av && av[0] == '1')
      for (int h = 0; h < B->n_hbm; ++h) hshift[h] = max_lev - plans[hidx[h]]->n_levels;
  }
  // QTN_HBM_GROUPS=G: the networks in G groups (LPT on algorithmic bytes),
  // each group an independent sequence of levels on its own stream lane, so
  // one group's latency-bound launches overlap another group's streaming
  // ones instead of every level waiting for its slowest launch.  Virtual
  // level = group * max_lev + level (the per-level lists below are built
  // over virtual levels).
  {
    const char* gv = getenv("QTN_HBM_GROUPS");
    int G = gv ? atoi(gv) : 1;
    G = std::max(1, std::min(G, qtn_batch::kMaxGroups));
    if (B->n_hbm < 2 * G) G = 1;
    std::vector<int> ord(B->n_hbm);
    for (int h = 0; h < B->n_hbm; ++h) ord[h] = h;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int a, int b) { return plans[hidx[a]]->alg_bytes > plans[hidx[b]]->alg_bytes; });
    std::vector<double> load(G, 0.0);
    for (int h : ord) {
      const int g = (int)(std::min_element(load.begin(), load.end()) - load.begin());
      load[g] += plans[hidx[h]]->alg_bytes;
      hshift[h] += g * max_lev;
    }
    B->n_groups = G;
    B->lev_per_group = max_lev;
    max_lev *= G;
  }
  // level-major item lists over all HBM networks
  std::vector<uint64_t> item_desc, prefix, sitem_desc;
  std::vector<uint32_t> item_net, sitem_net;
  const char* sv = getenv("QTN_SMALL_R");  // buckets up to this output rank: small kernel
  const int small_r = sv ? atoi(sv) : qtn::kSmallR;
  std::vector<uint64_t> desc_base(B->n_hbm);
  std::vector<uint32_t> xdesc_base(B->n_hbm), fdesc_base(B->n_hbm);
  std::vector<qtn::XDesc> xdescs;
  std::vector<qtn::YDesc> ydescs;
  std::vector<uint32_t> ydesc_base(B->n_hbm);
  std::vector<qtn::FDesc> fdescs;
  for (int h = 0; h < B->n_hbm; ++h) {
    const qtn_plan* P = plans[hidx[h]];
    desc_base[h] = desc.size();
    desc.insert(desc.end(), P->hbm_desc.begin(), P->hbm_desc.end());
    xdesc_base[h] = (uint32_t)xdescs.size();
    xdescs.insert(xdescs.end(), P->hbm_xdesc.begin(), P->hbm_xdesc.end());
    fdesc_base[h] = (uint32_t)fdescs.size();
    fdescs.insert(fdescs.end(), P->hbm_fdesc.begin(), P->hbm_fdesc.end());
    ydesc_base[h] = (uint32_t)ydescs.size();
    ydescs.insert(ydescs.end(), P->hbm_ydesc.begin(), P->hbm_ydesc.end());
  }
  // expanding bucket + consumer pairs, level-major over all HBM networks
  std::vector<uint32_t> yitem_desc, yitem_net;
  std::vector<uint64_t> yprefix;
  // (one list per level and group count g: a launch's items share g)
  for (int32_t lev = 0; lev < max_lev; ++lev)
   for (int gq = 0; gq <= qtn::kYMaxGB; ++gq) {
    B->level_yitem0.push_back((uint32_t)yitem_desc.size());
    B->level_yprefix0.push_back(yprefix.size());
    uint64_t yacc = 0;
    uint32_t ystage = 0;
    yprefix.push_back(0);
    for (int h = 0; h < B->n_hbm; ++h) {
      const qtn_plan* P = plans[hidx[h]];
      for (size_t y = 0; y < P->hbm_ydesc.size(); ++y) {
        if (P->hbm_ylevel[y] + hshift[h] != lev || P->hbm_ydesc[y].g != gq) continue;
        const qtn::YDesc& yd = P->hbm_ydesc[y];
        yitem_desc.push_back(ydesc_base[h] + (uint32_t)y);
        yitem_net.push_back((uint32_t)h);
        yacc += yd.n_tiles;
        yprefix.push_back(yacc);
        ystage = std::max(ystage, qtn::xt_stage_bytes(yd));
      }
    }
    B->level_ytiles.push_back(yacc);
    B->level_ystage.push_back(ystage);
  }
  B->level_yitem0.push_back((uint32_t)yitem_desc.size());
  // tail chains (weighted full sums), level-major over all HBM networks
  std::vector<qtn::WsDesc> wsdescs;
  std::vector<uint32_t> wsitem_desc, wsitem_net, wsprefix;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    B->level_ws0.push_back((uint32_t)wsitem_desc.size());
    B->level_wsprefix0.push_back((uint32_t)wsprefix.size());
    uint32_t acc = 0;
    wsprefix.push_back(0);
    for (int h = 0; h < B->n_hbm; ++h) {
      const qtn_plan* P = plans[hidx[h]];
      for (size_t w = 0; w < P->hbm_wsdesc.size(); ++w) {
        if (P->hbm_wslevel[w] + hshift[h] != lev) continue;
        wsitem_desc.push_back((uint32_t)wsdescs.size());
        wsitem_net.push_back((uint32_t)h);
        wsdescs.push_back(P->hbm_wsdesc[w]);
        acc += P->hbm_wsdesc[w].n_ctas;
        wsprefix.push_back(acc);
      }
    }
    B->level_wsctas.push_back(acc);
  }
  B->level_ws0.push_back((uint32_t)wsitem_desc.size());
  // host-built lookup tables of every fused descriptor (16-byte aligned each),
  // and the per-descriptor blob [header, sides, used ops | tables] the
  // fused kernel copies in one pass
  std::vector<uint32_t> ftabs;
  std::vector<uint8_t> fblob;
  std::vector<uint64_t> fblob_off(fdescs.size());
  std::vector<uint32_t> fdesc16(fdescs.size()), ftab16(fdescs.size());
  for (size_t i = 0; i < fdescs.size(); ++i) {
    auto& fd = fdescs[i];
    const size_t t0 = ftabs.size();
    fd.tab_off = 4ull * t0;
    qtn::fused_build_tables(fd, ftabs);
    while (ftabs.size() & 3u) ftabs.push_back(0u);
    const size_t dbytes = (offsetof(qtn::FDesc, ops) + fd.n_ops * sizeof(qtn::FOp) + 15) & ~(size_t)15;
    const size_t tbytes = 4 * (ftabs.size() - t0);
    fblob_off[i] = fblob.size();
    fdesc16[i] = (uint32_t)(dbytes / 16);
    ftab16[i] = (uint32_t)(tbytes / 16);
    const uint8_t* dp = reinterpret_cast<const uint8_t*>(&fd);
    fblob.insert(fblob.end(), dp, dp + std::min(dbytes, sizeof(qtn::FDesc)));
    fblob.resize(fblob_off[i] + dbytes, 0);
    const uint8_t* tp = reinterpret_cast<const uint8_t*>(ftabs.data() + t0);
    fblob.insert(fblob.end(), tp, tp + tbytes);
  }
  // tiny subtrees, level-major over all HBM networks
  std::vector<qtn::SubItem> sub_items;
  std::vector<uint64_t> sub_desc;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    B->level_sub0.push_back((uint32_t)sub_items.size());
    uint32_t smem = 0;
    for (int h = 0; h < B->n_hbm; ++h) {
      const qtn_plan* P = plans[hidx[h]];
      for (const auto& r : P->hbm_sub) {
        if (r.level + hshift[h] != lev) continue;
        qtn::SubItem it;
        it.net = (uint32_t)h;
        it.first = (uint32_t)sub_desc.size();
        it.count = r.count;
        it.smem = r.smem;
        for (uint32_t k = 0; k < r.count; ++k) sub_desc.push_back(desc_base[h] + P->hbm_sub_desc[r.first + k]);
        sub_items.push_back(it);
        smem = std::max(smem, r.smem);
      }
    }
    B->level_sub_smem.push_back(smem);
  }
  B->level_sub0.push_back((uint32_t)sub_items.size());
  // fused product chains, level-major over all HBM networks
  std::vector<uint32_t> fitem_desc, fitem_net;
  std::vector<uint64_t> fprefix, cprefix;
  std::vector<qtn::FCta> fctas;
  // warp-granular chains: the plans' blobs concatenated (16-byte aligned)
  std::vector<uint8_t> wblob;
  std::vector<uint64_t> wblob_base(B->n_hbm);
  for (int h = 0; h < B->n_hbm; ++h) {
    const qtn_plan* P = plans[hidx[h]];
    while (wblob.size() & 15u) wblob.push_back(0);
    wblob_base[h] = wblob.size();
    wblob.insert(wblob.end(), P->hbm_wblob.begin(), P->hbm_wblob.end());
  }
  std::vector<qtn::WRec> wrecs;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    B->level_fgroup0.push_back((uint32_t)B->fgroups.size());
    uint64_t lev_ctas = 0;
    for (int mt = 0; mt < 2; ++mt) {  // warp-granular chains of this math type
      qtn_batch::FGroup g{};
      g.warp = 1;
      g.f64 = (uint8_t)mt;
      g.cta0 = wrecs.size();
      for (int h = 0; h < B->n_hbm; ++h) {
        const qtn_plan* P = plans[hidx[h]];
        for (size_t f = 0; f < P->hbm_fdesc.size(); ++f) {
          const qtn::FDesc& fd = P->hbm_fdesc[f];
          if (P->hbm_flevel[f] + hshift[h] != lev || (fd.math_f32 ? 0 : 1) != mt || P->hbm_woff[f] < 0) continue;
          const uint64_t b16 = (wblob_base[h] + (uint64_t)P->hbm_woff[f]) / 16u;
          for (uint32_t c = 0; c < P->hbm_wwarps[f]; ++c) {
            qtn::WRec r{};
            r.blob16 = (uint32_t)b16;
            r.chunk = c;
            r.net = (uint32_t)h;
            wrecs.push_back(r);
          }
          g.n_items += 1;
        }
      }
      g.ctas = wrecs.size() - g.cta0;
      if (g.n_items) B->fgroups.push_back(g);
      lev_ctas += (g.ctas + 7) / 8;
    }
    for (int mt = 0; mt < 2; ++mt) {  // complex64 math, then complex128 math
      qtn_batch::FGroup g{};
      g.item0 = (uint32_t)fitem_desc.size();
      g.cta0 = fctas.size();
      g.prefix0 = fprefix.size();
      g.f64 = (uint8_t)mt;
      uint64_t acc = 0, cacc = 0;
      fprefix.push_back(0);
      cprefix.push_back(0);
      for (int h = 0; h < B->n_hbm; ++h) {
        const qtn_plan* P = plans[hidx[h]];
        for (size_t f = 0; f < P->hbm_fdesc.size(); ++f) {
          const qtn::FDesc& fd = P->hbm_fdesc[f];
          if (P->hbm_flevel[f] + hshift[h] != lev || (fd.math_f32 ? 0 : 1) != mt || P->hbm_woff[f] >= 0) continue;
          fitem_desc.push_back(fdesc_base[h] + (uint32_t)f);
          fitem_net.push_back((uint32_t)h);
          const uint64_t nc = fd.sk ? (fd.n_units << fd.sk) : (fd.n_units + (1ull << fd.upc_log2) - 1) >> fd.upc_log2;
          const uint32_t di = fdesc_base[h] + (uint32_t)f;
          for (uint64_t c = 0; c < nc; ++c) {
            qtn::FCta r{};
            r.blob = fblob_off[di];
            r.desc16 = fdesc16[di];
            r.tab16 = ftab16[di];
            r.net = (uint32_t)h;
            r.c = (uint32_t)c;
            fctas.push_back(r);
          }
          acc += nc;
          fprefix.push_back(acc);
          cacc += fd.sk ? fd.n_units : 0;
          cprefix.push_back(cacc);
          g.smem = std::max(g.smem, qtn::fused_smem_bytes(fd));
        }
      }
      g.n_items = (uint32_t)fitem_desc.size() - g.item0;
      g.ctas = acc;
      g.cctas = cacc;
      if (g.n_items) B->fgroups.push_back(g);
      lev_ctas += acc;
    }
    B->level_fctas.push_back(lev_ctas);
  }
  B->level_fgroup0.push_back((uint32_t)B->fgroups.size());
  // expanding buckets take the outer-product kernel (QTN_EXPAND=0: the
  // streaming kernel, for A/B measurements)
  const char* xv = getenv("QTN_EXPAND");
  const bool use_expand = !(xv && xv[0] == '0');
  std::vector<uint32_t> xitem_desc, xitem_net;
  std::vector<uint64_t> xprefix;
  // single-operand buckets of output rank >= QTN_TRACE_MIN_R take
  // trace_kernel (QTN_TRACE=0: the streaming kernel)
  const char* tv0 = getenv("QTN_TRACE");
  const bool use_trace = !(tv0 && tv0[0] == '0');
  const char* tmr = getenv("QTN_TRACE_MIN_R");
  const int trace_min_r = tmr ? atoi(tmr) : 8;
  std::vector<qtn::R1Dev> r1items;
  std::vector<uint64_t> r1prefix;
  std::vector<uint32_t> r1chunk_item;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    B->level_item0.push_back((uint32_t)item_desc.size());
    B->level_prefix0.push_back(prefix.size());
    B->level_sitem0.push_back((uint32_t)sitem_desc.size());
    B->level_xitem0.push_back((uint32_t)xitem_desc.size());
    B->level_xprefix0.push_back(xprefix.size());
    B->level_r1item0.push_back((uint32_t)r1items.size());
    B->level_r1prefix0.push_back(r1prefix.size());
    B->level_r1chunk0.push_back(r1chunk_item.size());
    uint64_t acc = 0, xacc = 0, r1acc = 0;
    uint32_t xstage = 0;
    prefix.push_back(0);
    xprefix.push_back(0);
    r1prefix.push_back(0);
    // small buckets go to the warp/CTA-per-bucket kernel, unless the level
    // launches the streaming kernel anyway and they are few (one launch less)
    // a tiny level (few output elements in all) goes entirely to the small
    // kernel: the tile pipeline's fixed cost dominates there
    int n_small = 0, n_large = 0;
    uint64_t lev_elems = 0;
    for (int h = 0; h < B->n_hbm; ++h) {
      const qtn_plan* P = plans[hidx[h]];
      for (size_t bi = 0; bi < P->hbm_level.size(); ++bi) {
        if (P->hbm_level[bi] + hshift[h] != lev || !P->hbm_tiles[bi]) continue;  // 0 tiles: fused chain
        const qtn::SHdr* sh = reinterpret_cast<const qtn::SHdr*>(P->hbm_desc.data() + P->hbm_desc_off[bi]);
        ((int)sh->R <= small_r ? n_small : n_large) += 1;
        lev_elems += 1ull << sh->R;
      }
    }
    const char* tv = getenv("QTN_TINY_LEVEL");
    const uint64_t tiny = tv ? strtoull(tv, nullptr, 10) : (1ull << 17);
    const bool all_small = lev_elems <= tiny;
    const bool split_small = all_small || (n_small > 0 && (n_large == 0 || n_small >= 148));
    // trace_kernel for this level's single-operand buckets when it saves a
    // pass: no other streamed bucket in the level (no extra launch), or
    // enough trace bytes to pay for the extra launch (QTN_TRACE_MIN_MB)
    bool trace_level = false;
    {
      const char* tmb = getenv("QTN_TRACE_MIN_MB");
      const double min_bytes = (tmb ? atof(tmb) : 4.0) * 1e6;  // re-measured with the xt chains: 32/16/8/4/1 MB -> config 3 default 2.148/2.136/2.123/2.115/2.121 ms
      double tbytes = 0.0;
      bool other = false;
      for (int h = 0; h < B->n_hbm; ++h) {
        const qtn_plan* P = plans[hidx[h]];
        for (size_t bi = 0; bi < P->hbm_level.size(); ++bi) {
          if (P->hbm_level[bi] + hshift[h] != lev || !P->hbm_tiles[bi]) continue;
          const qtn::SHdr* sh = reinterpret_cast<const qtn::SHdr*>(P->hbm_desc.data() + P->hbm_desc_off[bi]);
          if (split_small && (all_small || (int)sh->R <= small_r)) continue;
          if (use_expand && P->hbm_xidx[bi] >= 0) continue;  // expand_kernel
          if (use_trace && P->hbm_r1idx[bi] >= 0 && (int)sh->R >= trace_min_r)
            tbytes += std::ldexp(P->hbm_r1[P->hbm_r1idx[bi]].out_c64 ? 24.0 : 48.0, sh->R);
          else
            other = true;
        }
      }
      trace_level = !other || tbytes >= min_bytes;
    }
    uint32_t smax_r = 0;
    for (int h = 0; h < B->n_hbm; ++h) {
      const qtn_plan* P = plans[hidx[h]];
      for (size_t bi = 0; bi < P->hbm_level.size(); ++bi) {
        if (P->hbm_level[bi] + hshift[h] != lev || !P->hbm_tiles[bi]) continue;  // 0 tiles: fused chain
        const qtn::SHdr* sh = reinterpret_cast<const qtn::SHdr*>(P->hbm_desc.data() + P->hbm_desc_off[bi]);
        if (split_small && (all_small || (int)sh->R <= small_r)) {
          sitem_desc.push_back(desc_base[h] + P->hbm_desc_off[bi]);
          sitem_net.push_back((uint32_t)h);
          smax_r = std::max<uint32_t>(smax_r, sh->R);
          continue;
        }
        if (use_expand && P->hbm_xidx[bi] >= 0) {
          const qtn::XDesc& xd = P->hbm_xdesc[P->hbm_xidx[bi]];
          xitem_desc.push_back(xdesc_base[h] + (uint32_t)P->hbm_xidx[bi]);
          xitem_net.push_back((uint32_t)h);
          xacc += xd.n_tiles;
          xprefix.push_back(xacc);
          xstage = std::max<uint32_t>(xstage, (2u << (xd.h + xd.c)) * (xd.out_c64 ? 8u : 16u));
          continue;
        }
        if (use_trace && P->hbm_r1idx[bi] >= 0 && (int)sh->R >= trace_min_r && trace_level) {
          qtn::R1Dev r = P->hbm_r1[P->hbm_r1idx[bi]];
          r.net = (uint32_t)h;
          r1items.push_back(r);
          const uint64_t nck = ((1ull << r.R) + qtn::kTraceChunk - 1) / qtn::kTraceChunk;
          for (uint64_t c = 0; c < nck; ++c)  // chunk -> item (level-relative): no search per CTA
            r1chunk_item.push_back((uint32_t)(r1items.size() - 1 - B->level_r1item0.back()));
          r1acc += nck;
          r1prefix.push_back(r1acc);
          continue;
        }
        if (getenv("QTN_DEBUG_ROUTE"))
          fprintf(stderr, "stream-item lev=%d R=%d prank=%d pc64=%d ng=%d nt=%d ntop=%d ta=%d tn=%d nops=%zu\n",
                  lev, (int)sh->R, (int)sh->p_rank, (int)sh->p_c64, (int)sh->ng, (int)sh->nt,
                  (int)sh->ntop, (int)sh->ta, (int)sh->tn, P->buckets[bi].ops.size());
        item_desc.push_back(desc_base[h] + P->hbm_desc_off[bi]);
        item_net.push_back((uint32_t)h);
        acc += P->hbm_tiles[bi];
        prefix.push_back(acc);
      }
    }
    B->level_tiles.push_back(acc);
    B->level_smax_r.push_back(smax_r);
    {
      // chain_kernel candidates: few enough outputs for one CTA cluster
      // (a warp per bucket: every bucket of the level at most 2^QTN_CHAIN_R outputs)
      const char* ce = getenv("QTN_CHAIN_ELEMS");
      const uint64_t chain_elems = ce ? strtoull(ce, nullptr, 10) : 16384;
      const char* cr = getenv("QTN_CHAIN_R");
      const uint32_t chain_r = cr ? (uint32_t)atoi(cr) : 9;
      B->level_tiny.push_back(all_small && lev_elems <= chain_elems && smax_r <= chain_r ? 1 : 0);
    }
    B->level_xtiles.push_back(xacc);
    B->level_xstage.push_back(xstage);
    B->level_r1chunks.push_back(r1acc);
  }
  B->level_r1item0.push_back((uint32_t)r1items.size());
  B->level_item0.push_back((uint32_t)item_desc.size());
  B->level_sitem0.push_back((uint32_t)sitem_desc.size());
  B->level_xitem0.push_back((uint32_t)xitem_desc.size());
  // fused reductions, level-major over all HBM networks
  std::vector<qtn::RedDev> reds;
  std::vector<uint32_t> rprefix;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    B->level_red0.push_back((uint32_t)reds.size());
    B->level_rprefix0.push_back((uint32_t)rprefix.size());
    uint32_t acc = 0;
    for (int h = 0; h < B->n_hbm; ++h) {
      for (const auto& r : plans[hidx[h]]->hbm_red) {
        if (r.level + hshift[h] != lev) continue;
        qtn::RedDev d{};
        d.src = r.src;
        d.out = r.out;
        d.net = (uint32_t)h;
        d.src_c64 = r.src_c64;
        d.out_c64 = r.out_c64;
        d.R = r.R;
        d.k = r.k;
        for (int q = 0; q < r.k; ++q) d.pos[q] = r.pos[q];
        reds.push_back(d);
        rprefix.push_back(acc);
        const uint64_t ch = qtn::red_chunk(r.k);
        acc += (uint32_t)(((1ull << r.R) + ch - 1) / ch);
      }
    }
    rprefix.push_back(acc);
    B->level_rchunks.push_back(acc);
  }
  B->level_red0.push_back((uint32_t)reds.size());
  // runs of consecutive tiny levels (small items only) become one
  // cluster launch each (chain_kernel) with QTN_CHAIN=1.  Off by default:
  // measured equal to one small_kernel launch per level inside the captured
  // graph (config 4: 788 vs 788 /s; config 3 default 69.6 k vs 69.5 k)
  {
    const char* cv = getenv("QTN_CHAIN");
    const bool chain_on = cv && cv[0] == '1';
    const size_t nl = B->level_tiles.size();
    B->chain_len.assign(nl, 0);
    auto tiny_only = [&](size_t l) {
      return B->level_tiny[l] && !B->level_tiles[l] && !B->level_xtiles[l] && !y_launches(B, l) && !B->level_r1chunks[l] &&
             !B->level_wsctas[l] && !B->level_fctas[l] && B->level_sub0[l + 1] == B->level_sub0[l] &&
             B->level_red0[l + 1] == B->level_red0[l] && B->level_sitem0[l + 1] > B->level_sitem0[l];
    };
    for (size_t l = 0; chain_on && l < nl;) {
      size_t e = l;
      while (e < nl && tiny_only(e) && (!B->lev_per_group || e / B->lev_per_group == l / B->lev_per_group)) ++e;
      if (e - l >= 2) B->chain_len[l] = (uint32_t)(e - l);
      l = e > l ? e : l + 1;
    }
  }
  // scalar folds
  std::vector<uint64_t> ftags;
  std::vector<uint8_t> fc64;
  std::vector<uint32_t> ffirst;
  std::vector<int32_t> fpow2;
  for (int h = 0; h < B->n_hbm; ++h) {
    const qtn_plan* P = plans[hidx[h]];
    ffirst.push_back((uint32_t)ftags.size());
    fpow2.push_back(P->n_empty);
    for (int32_t id : P->scalars) {
      const auto& t = P->tensors[id];
      ftags.push_back(t.input ? tag_in(16ull * (uint64_t)t.in_off) : tag_ws((uint64_t)t.ws_off));
      fc64.push_back(t.c64 ? 1 : 0);
    }
  }
  ffirst.push_back((uint32_t)ftags.size());
  if ((rc = upload(&B->d_prog, blob)) || (rc = upload(&B->d_prog_off, poff)) ||
      (rc = upload(&B->d_in_off, ioff)) || (rc = upload(&B->d_smem_index, sidx)) ||
      (rc = (desc.resize(desc.size() + 1024, 0), upload(&B->d_desc, desc))) ||
      (rc = upload(&B->d_item_desc, item_desc)) ||
      (rc = upload(&B->d_item_net, item_net)) || (rc = upload(&B->d_tile_prefix, prefix)) ||
      (rc = upload(&B->d_sitem_desc, sitem_desc)) || (rc = upload(&B->d_sitem_net, sitem_net)) ||
      (rc = upload(&B->d_red, reds)) || (rc = upload(&B->d_red_prefix, rprefix)) ||
      (rc = upload(&B->d_xdesc, xdescs)) || (rc = upload(&B->d_xitem_desc, xitem_desc)) ||
      (rc = upload(&B->d_xitem_net, xitem_net)) || (rc = upload(&B->d_xprefix, xprefix)) ||
      (rc = upload(&B->d_ydesc, ydescs)) || (rc = upload(&B->d_yitem_desc, yitem_desc)) ||
      (rc = upload(&B->d_yitem_net, yitem_net)) || (rc = upload(&B->d_yprefix, yprefix)) ||
      (rc = upload(&B->d_wsdesc, wsdescs)) || (rc = upload(&B->d_wsitem_desc, wsitem_desc)) ||
      (rc = upload(&B->d_wsitem_net, wsitem_net)) || (rc = upload(&B->d_wsprefix, wsprefix)) ||
      (rc = upload(&B->d_level_sitem0, B->level_sitem0)) ||
      (rc = upload(&B->d_r1, r1items)) || (rc = upload(&B->d_r1prefix, r1prefix)) ||
      (rc = upload(&B->d_r1chunk_item, r1chunk_item)) ||
      (rc = upload(&B->d_fdesc, fdescs)) || (rc = upload(&B->d_fitem_desc, fitem_desc)) ||
      (rc = upload(&B->d_ftab, ftabs)) || (rc = upload(&B->d_fctas, fctas)) ||
      (rc = upload(&B->d_fblob, fblob)) || (rc = upload(&B->d_wblob, wblob)) || (rc = upload(&B->d_wrecs, wrecs)) ||
      (rc = upload(&B->d_sub_items, sub_items)) || (rc = upload(&B->d_sub_desc, sub_desc)) ||
      (rc = upload(&B->d_fitem_net, fitem_net)) || (rc = upload(&B->d_fprefix, fprefix)) ||
      (rc = upload(&B->d_cprefix, cprefix)) ||
      (rc = upload(&B->d_net_in_off, net_in)) || (rc = upload(&B->d_net_ws_off, net_ws)) ||
      (rc = upload(&B->d_fold_tags, ftags)) || (rc = upload(&B->d_fold_c64, fc64)) ||
      (rc = upload(&B->d_fold_first, ffirst)) || (rc = upload(&B->d_fold_pow2, fpow2)) ||
      (rc = upload(&B->d_hbm_index, hidx))) {
    qtn_batch_destroy(B);
    return rc;
  }
  *out = B;
  return QTN_OK;
}

extern "C" int qtn_batch_input_elems(const qtn_batch* B, int64_t* out) {
  if (!B || !out) return QTN_EINVAL;
  *out = B->set_elems;
  return QTN_OK;
}

extern "C" int qtn_batch_input_offsets(const qtn_batch* B, int64_t* out) {
  if (!B || !out) return QTN_EINVAL;
  std::copy(B->in_offsets.begin(), B->in_offsets.end(), out);
  return QTN_OK;
}

// Set-major pays ~7 us per level launch but streams at HBM speed; the
// warp-resident executor has one launch but its throughput falls with the
// per-set footprint (occupancy).  Measured crossovers (B200): config 2
// (<= 8 KiB per set) between 64 and 128 sets, config 3 (up to 78 KiB per
// set) below 64.  QTN_SETMAJOR_MIN_SETS overrides (read per call).
static bool use_setmajor(const qtn_batch* B, int32_t n_sets) {
  const char* v = getenv("QTN_SETMAJOR_MIN_SETS");
  const int min_sets = v ? atoi(v) : (B->warp_bytes <= 8192u ? 128 : 32);
  return B->sm && min_sets > 0 && n_sets >= min_sets;
}

extern "C" int qtn_batch_workspace_bytes(const qtn_batch* B, int32_t n_sets, int64_t* out) {
  if (!B || !out || n_sets < 1) return QTN_EINVAL;
  *out = B->ws_per_set * n_sets + (B->sm ? qtn::setmajor_workspace(B->sm, n_sets) : 0);
  return QTN_OK;
}

static bool use_setmajor(const qtn_batch* B, int32_t n_sets);

extern "C" int qtn_batch_launches(const qtn_batch* B, int32_t n_sets, int32_t* out) {
  if (!B || !out) return QTN_EINVAL;
  int c = B->n_smem ? 1 : 0;
  if (B->n_smem && use_setmajor(B, n_sets)) c = qtn::setmajor_launches(B->sm, n_sets);
  if (B->n_hbm) {
    for (size_t lev = 0; lev < B->level_tiles.size(); ++lev) {
      if (B->chain_len[lev]) {
        c += 1;
        lev += B->chain_len[lev] - 1;
        continue;
      }
      c += (B->level_tiles[lev] ? 1 : 0) + (B->level_sitem0[lev + 1] > B->level_sitem0[lev] ? 1 : 0) +
           (B->level_red0[lev + 1] > B->level_red0[lev] ? 1 : 0) + (B->level_xtiles[lev] ? 1 : 0) +
           y_launches(B, lev) + (B->level_r1chunks[lev] ? 1 : 0) + (B->level_sub0[lev + 1] > B->level_sub0[lev] ? 1 : 0) +
           (B->level_wsctas[lev] ? 2 : 0);
      for (uint32_t gi = B->level_fgroup0[lev]; gi < B->level_fgroup0[lev + 1]; ++gi)
        c += 1 + (B->fgroups[gi].cctas ? 1 : 0);
    }
    c += 1;
  }
  *out = c;
  return QTN_OK;
}

extern "C" int qtn_batch_uses_setmajor(const qtn_batch* B, int32_t n_sets, int32_t* out) {
  if (!B || !out) return QTN_EINVAL;
  *out = (B->n_smem && use_setmajor(B, n_sets)) ? 1 : 0;
  return QTN_OK;
}

extern "C" int qtn_batch_setmajor_elem_bytes(const qtn_batch* B, int32_t n_sets, int32_t* out) {
  if (!B || !out) return QTN_EINVAL;
  *out = (B->n_smem && use_setmajor(B, n_sets)) ? qtn::setmajor_elem_bytes(B->sm) : 0;
  return QTN_OK;
}

static int run_batch(qtn_batch* B, const void* inputs, int64_t set_stride, const double* angles,
                     int32_t n_angles, int32_t n_sets, void* workspace, void* results,
                     void* stream);

extern "C" int qtn_batch_execute(qtn_batch* B, const void* inputs, int64_t set_stride,
                                 int32_t n_sets, void* workspace, void* results, void* stream) {
  return run_batch(B, inputs, set_stride, nullptr, 0, n_sets, workspace, results, stream);
}

// Host-to-host contraction of one set of packed inputs (the drop-in
// contract() call): H2D from the caller's pinned buffer, the evaluation, D2H
// of the n results and the stream wait in one native call.
extern "C" int qtn_batch_execute_host(qtn_batch* B, const void* inputs_pinned, int64_t input_bytes,
                                      void* inputs_dev, void* workspace, void* results_dev,
                                      void* results_pinned, void* stream) {
  if (!B || !inputs_pinned || !inputs_dev || !results_dev || !results_pinned || input_bytes < 0) {
    set_error("qtn_batch_execute_host: bad arguments");
    return QTN_EINVAL;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(inputs_dev, inputs_pinned, (size_t)input_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "inputs H2D");
  const int rc = run_batch(B, inputs_dev, 0, nullptr, 0, 1, workspace, results_dev, stream);
  if (rc) return rc;
  e = cudaMemcpyAsync(results_pinned, results_dev, (size_t)B->n * sizeof(double2), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(e, "results D2H");
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "execute_host sync");
  return QTN_OK;
}

extern "C" int qtn_batch_set_recipes(qtn_batch* B, const qtn_tensor_recipe* rec,
                                     const int64_t* offsets) {
  if (!B || !rec || !offsets) {
    set_error("qtn_batch_set_recipes: bad arguments");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  // SMEM networks: append a generator section to each program
  std::vector<uint8_t> blob;
  std::vector<uint64_t> poff;
  uint32_t prog_max = 0, warp_bytes = 0;
  for (size_t k = 0; k < B->smem_progs.size(); ++k) {
    const int gi = B->smem_global[k];
    std::vector<uint8_t> prog = B->smem_progs[k];
    SmemHeader* h = reinterpret_cast<SmemHeader*>(prog.data());
    std::vector<SmemGenParam> params;
    std::vector<SmemGenRec> recs;
    // generator entries are emitted in materialisation order (the SmemIn
    // records: rank-0 inputs, then bucket by bucket), so every bucket's
    // inputs are one contiguous entry range
    const SmemIn* sin = reinterpret_cast<const SmemIn*>(prog.data() + h->in_off);
    SmemBucket* bk = reinterpret_cast<SmemBucket*>(prog.data() + sizeof(SmemHeader));
    uint32_t n_sin = h->n_init;
    for (uint32_t b = 0; b < h->n_buckets; ++b)
      n_sin = std::max<uint32_t>(n_sin, bk[b].first_in + bk[b].n_in);
    std::vector<uint32_t> entry_at(n_sin + 1, 0);
    for (uint32_t si = 0; si < n_sin; ++si) {
      entry_at[si] = (uint32_t)recs.size();
      const int64_t r = offsets[gi] + sin[si].input;
      if (r >= offsets[gi + 1]) {
        set_error("qtn_batch_set_recipes: recipes do not match the plan's inputs");
        return QTN_EINVAL;
      }
      const int32_t base = sin[si].sm_off;
      const qtn_tensor_recipe& q = rec[r];
      SmemGenParam p{};
      if (q.kind == QTN_GATE_SCALAR) {
        p.scale = q.scale;
        p.offset = q.offset;
        p.angle = -2;
      } else {
        const bool has_t = q.kind == QTN_GATE_ZPOW || q.kind == QTN_GATE_XPOW ||
                           q.kind == QTN_GATE_ZZ || q.kind == QTN_GATE_ZPOW_DIAG ||
                           q.kind == QTN_GATE_ZZ_DIAG;
        p.scale = has_t ? q.scale : 0.0;
        p.offset = has_t ? q.offset : 0.0;
        p.angle = has_t ? (q.angle >= 0 ? q.angle : -1) : -1;
      }
      size_t slot = 0;
      for (; slot < params.size(); ++slot)
        if (params[slot].scale == p.scale && params[slot].offset == p.offset &&
            params[slot].angle == p.angle)
          break;
      if (slot == params.size()) params.push_back(p);
      if (slot > 255) {
        set_error("qtn_batch_set_recipes: too many distinct gate parameters");
        return QTN_EINVAL;
      }
      // one record per kept entry: slicing (network.py:153-165) resolved here
      const int fr = q.full_rank;
      const int kept = __builtin_popcount(q.keep_mask);
      for (uint32_t e = 0; e < (1u << kept); ++e) {
        uint32_t full = 0;
        int kb = kept - 1;
        for (int pos = 0; pos < fr; ++pos) {
          const uint32_t bit = ((q.keep_mask >> pos) & 1) ? (e >> kb--) & 1 : (q.fixed_bits >> pos) & 1;
          full = (full << 1) | bit;
        }
        SmemGenRec g{};
        g.sm_off = (uint16_t)(base + e);
        g.kind = q.kind;
        g.full = (uint8_t)full;
        g.param = (uint8_t)slot;
        recs.push_back(g);
      }
    }
    entry_at[n_sin] = (uint32_t)recs.size();
    if (recs.size() > 65535) {
      set_error("qtn_batch_set_recipes: network too large for the fused generator");
      return QTN_EINVAL;
    }
    h->n_init_gen = entry_at[h->n_init];
    for (uint32_t b = 0; b < h->n_buckets; ++b) {
      bk[b].first_gen = (uint16_t)entry_at[bk[b].first_in];
      bk[b].n_gen = (uint16_t)(entry_at[bk[b].first_in + bk[b].n_in] - entry_at[bk[b].first_in]);
    }
    const size_t gen_off = prog.size();
    size_t gen_bytes = params.size() * sizeof(SmemGenParam) + recs.size() * sizeof(SmemGenRec);
    gen_bytes = (gen_bytes + 15) & ~size_t(15);
    prog.resize(gen_off + gen_bytes, 0);
    h = reinterpret_cast<SmemHeader*>(prog.data());
    std::memcpy(prog.data() + gen_off, params.data(), params.size() * sizeof(SmemGenParam));
    std::memcpy(prog.data() + gen_off + params.size() * sizeof(SmemGenParam), recs.data(),
                recs.size() * sizeof(SmemGenRec));
    h->gen_off = (uint32_t)gen_off;
    h->n_params = (uint32_t)params.size();
    h->n_recs = (uint32_t)recs.size();
    h->prog_bytes = (uint32_t)prog.size();
    prog_max = std::max<uint32_t>(prog_max, (uint32_t)prog.size());
    warp_bytes = std::max<uint32_t>(warp_bytes, 16u * (h->data_elems + h->n_params));
    poff.push_back(blob.size());
    blob.insert(blob.end(), prog.begin(), prog.end());
  }
  // captured graphs hold kernel parameters that point at the buffers freed
  // below: drop them before replacing the device program
  for (auto& kv : B->graphs) cudaGraphExecDestroy(kv.second);
  B->graphs.clear();
  for (auto& kv : B->egraphs) cudaGraphExecDestroy(kv.second);
  B->egraphs.clear();
  // HBM networks: recipes relocated into the batch input layout
  std::vector<qtn_tensor_recipe> hrec;
  for (int i = 0; i < B->n; ++i) {
    if (std::find(B->smem_global.begin(), B->smem_global.end(), i) != B->smem_global.end())
      continue;
    for (int64_t r = offsets[i]; r < offsets[i + 1]; ++r) {
      qtn_tensor_recipe q = rec[r];
      q.out_offset += B->in_offsets[i];
      hrec.push_back(q);
    }
  }
  if (!blob.empty()) {
    device_free(B->d_prog);
    device_free(B->d_prog_off);
    B->d_prog = nullptr;
    B->d_prog_off = nullptr;
    if ((rc = upload(&B->d_prog, blob)) || (rc = upload(&B->d_prog_off, poff))) return rc;
    B->prog_max = prog_max;
    B->warp_bytes = warp_bytes;
  }
  device_free(B->d_hbm_rec);
  B->d_hbm_rec = nullptr;
  if ((rc = upload(&B->d_hbm_rec, hrec))) return rc;
  B->n_hbm_rec = (int64_t)hrec.size();
  B->has_recipes = true;
  qtn::setmajor_destroy(B->sm);
  B->sm = nullptr;
  if (!B->smem_plans.empty() &&
      (rc = qtn::setmajor_build(&B->sm, B->smem_plans, B->smem_global, rec, offsets, B->n))) {
    // a structural limit of the set-major form (more than 8 operands in a
    // bucket, ...): the small networks keep the warp-resident executor
    B->sm = nullptr;
    if (rc != QTN_EINVAL) return rc;
  }
  return QTN_OK;
}

static int execute_angles_direct(qtn_batch* B, const double* angles, int32_t n_angles,
                                 int32_t n_sets, void* inputs_scratch, void* workspace,
                                 void* results, void* stream);

extern "C" int qtn_batch_execute_angles(qtn_batch* B, const double* angles, int32_t n_angles,
                                        int32_t n_sets, void* inputs_scratch, void* workspace,
                                        void* results, void* stream) {
  const char* gv = getenv("QTN_GRAPHS");
  int32_t n_launch = 0;
  if (B) qtn_batch_launches(B, n_sets, &n_launch);
  if (!B || (gv && gv[0] == '0') || n_launch <= 2)  // a single executor launch: nothing to save
    return execute_angles_direct(B, angles, n_angles, n_sets, inputs_scratch, workspace, results,
                                 stream);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const GraphKey key{angles, inputs_scratch, workspace, results, n_angles, n_sets,
                     use_setmajor(B, n_sets)};
  auto it = B->graphs.find(key);
  if (it == B->graphs.end()) {
    if (B->graphs.size() >= 16) {  // bounded cache
      for (auto& kv : B->graphs) cudaGraphExecDestroy(kv.second);
      B->graphs.clear();
    }
    if (!B->cap_stream && cudaStreamCreateWithFlags(&B->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
      return cuda_fail(cudaGetLastError(), "capture stream");
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(B->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "graph capture begin");
    int rc = execute_angles_direct(B, angles, n_angles, n_sets, inputs_scratch, workspace, results,
                                   B->cap_stream);
    e = cudaStreamEndCapture(B->cap_stream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "graph capture end");
    cudaGraphExec_t ex = nullptr;
    e = cudaGraphInstantiate(&ex, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
    it = B->graphs.emplace(key, ex).first;
  }
  cudaError_t e = cudaGraphLaunch(it->second, st);
  if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  return QTN_OK;
}

static int execute_angles_direct(qtn_batch* B, const double* angles, int32_t n_angles,
                                 int32_t n_sets, void* inputs_scratch, void* workspace,
                                 void* results, void* stream) {
  if (!B || !angles || !B->has_recipes) {
    set_error("qtn_batch_execute_angles: needs qtn_batch_set_recipes first");
    return QTN_EINVAL;
  }
  if (B->n_hbm && !inputs_scratch) {
    set_error("qtn_batch_execute_angles: HBM networks need an input scratch buffer");
    return QTN_EINVAL;
  }
  int rc;
  if (B->n_hbm_rec &&
      (rc = qtn_tensorgen(B->d_hbm_rec, B->n_hbm_rec, angles, n_angles, n_sets, B->set_elems,
                          inputs_scratch, stream)))
    return rc;
  if (use_setmajor(B, n_sets)) {
    // small networks: set-major streaming executor; HBM networks as usual
    char* smws = reinterpret_cast<char*>(workspace) + B->ws_per_set * n_sets;
    if ((rc = qtn::setmajor_run(B->sm, angles, n_angles, n_sets, smws, results, stream))) return rc;
    if (!B->n_hbm) return QTN_OK;
    const int n_smem = B->n_smem;
    B->n_smem = 0;  // skip the SMEM executor for this call
    rc = run_batch(B, inputs_scratch, B->set_elems, angles, n_angles, n_sets, workspace, results,
                   stream);
    B->n_smem = n_smem;
    return rc;
  }
  return run_batch(B, inputs_scratch, B->set_elems, angles, n_angles, n_sets, workspace, results,
                   stream);
}

static int run_batch(qtn_batch* B, const void* inputs, int64_t set_stride, const double* angles,
                     int32_t n_angles, int32_t n_sets, void* workspace, void* results,
                     void* stream) {
  if (!B || !results || n_sets < 1) {
    set_error("qtn_batch_execute: bad arguments");
    return QTN_EINVAL;
  }
  if (set_stride <= 0) set_stride = B->set_elems;
  if (B->n_hbm && B->ws_per_set > 0 && !workspace) {
    set_error("qtn_batch_execute: HBM networks need a workspace (qtn_batch_workspace_bytes)");
    return QTN_EINVAL;
  }
  if (!angles && !inputs) {
    set_error("qtn_batch_execute: no inputs");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (B->n_smem) {
    const uint32_t prog_max = (B->prog_max + 15) & ~15u;
    const uint32_t warp_bytes = (B->warp_bytes + 15) & ~15u;
    // lanes per set L (measured on B200, config 2 / config 3): 16 lanes per
    // set (2 sets per warp) for small per-set regions, 32 for large ones;
    // one lane per set (32 sets per warp, fully independent lanes) is
    // latency-bound at ~4 warps/SM and 4x slower
    static int env_l = -1;
    if (env_l < 0) {
      const char* v = getenv("QTN_LANES_PER_SET");
      env_l = v ? std::max(1, atoi(v)) : 0;
    }
    const size_t cap = 227u * 1024u;
    int L = env_l > 0 ? env_l : (warp_bytes <= 12 * 1024 ? 16 : 32);
    while (L < 32 && (size_t)prog_max + (size_t)(32 / L) * warp_bytes > cap) L *= 2;
    if ((size_t)prog_max + warp_bytes > cap) {
      set_error("smem executor: a network's shared-memory footprint exceeds 227 KiB");
      return QTN_EINVAL;
    }
    const int S = 32 / L;
    const size_t per_warp = (size_t)S * warp_bytes;
    const int warps_needed = (n_sets + S - 1) / S;
    int W = (int)std::min<size_t>(kNetWarps, (cap - prog_max) / std::max<size_t>(per_warp, 16));
    W = std::max(1, std::min(W, warps_needed));
    const size_t smem = (size_t)prog_max + (size_t)W * per_warp;
    static std::atomic<size_t> attr[64];  // per device ordinal
    int dev = 0;
    cudaGetDevice(&dev);
    if (smem > 48 * 1024 && smem > attr[dev & 63].load()) {
      cudaError_t e = cudaFuncSetAttribute(smem_net_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return cuda_fail(e, "smem_net_kernel attribute");
      attr[dev & 63].store(smem);
    }
    SmemArgs a;
    a.progs = B->d_prog;
    a.prog_off = B->d_prog_off;
    a.in_off = B->d_in_off;
    a.out_index = B->d_smem_index;
    a.inputs = reinterpret_cast<const double2*>(inputs);
    a.set_elems = set_stride;
    a.results = reinterpret_cast<double2*>(results);
    a.angles = (angles && B->has_recipes) ? angles : nullptr;
    a.n_angles = n_angles;
    a.n_sets = n_sets;
    a.n_total = B->n;
    a.prog_max = prog_max;
    a.set_bytes = warp_bytes;
    a.lanes_per_set = L;
    dim3 grid(B->n_smem, (warps_needed + W - 1) / W);
    smem_net_kernel<<<grid, 32 * W, smem, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "smem_net_kernel launch");
  }
  if (B->n_hbm) {
    // The launches of one level are independent (their buckets sit at the
    // same depth of the elimination trees, the arena never aliases buckets
    // of one level): run them concurrently on forked streams (QTN_LEVEL_STREAMS=0:
    // one stream, for A/B measurements).  A level's launches are joined
    // back before the next level starts.
    const char* lsv = getenv("QTN_LEVEL_STREAMS");
    const bool level_streams = !(lsv && lsv[0] == '0');
    const int G = B->n_groups;
    for (int g = 0; g < G; ++g) {
      if (level_streams && !B->gfork[g]) {
        cudaError_t e = cudaEventCreateWithFlags(&B->gfork[g], cudaEventDisableTiming);
        for (int k = 0; k < qtn_batch::kSide && e == cudaSuccess; ++k) {
          e = cudaStreamCreateWithFlags(&B->gside[g][k], cudaStreamNonBlocking);
          if (e == cudaSuccess) e = cudaEventCreateWithFlags(&B->gjoin[g][k], cudaEventDisableTiming);
        }
        if (e != cudaSuccess) return cuda_fail(e, "level streams");
      }
      if (g > 0 && !B->lane[g]) {
        cudaError_t e = cudaStreamCreateWithFlags(&B->lane[g], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&B->ev_lane_done[g], cudaEventDisableTiming);
        if (e == cudaSuccess && !B->ev_lanes) e = cudaEventCreateWithFlags(&B->ev_lanes, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "group lanes");
      }
    }
    if (G > 1) {  // the lanes start after everything before the evaluation
      cudaEventRecord(B->ev_lanes, st);
      for (int g = 1; g < G; ++g) cudaStreamWaitEvent(B->lane[g], B->ev_lanes, 0);
    }
    int cur_g = -1;
    cudaStream_t gst = st;       // the current group's lane
    void* gstream = stream;
    static int pdl_tiny_env = -1;
    if (pdl_tiny_env < 0) {
      const char* pv = getenv("QTN_PDL_TINY");
      pdl_tiny_env = (pv && pv[0] == '0') ? 0 : 1;
    }
    const bool pdl_tiny = pdl_tiny_env == 1;
    static int pdl_single_env = -1;
    if (pdl_single_env < 0) {
      const char* pv = getenv("QTN_PDL_SINGLE");
      pdl_single_env = (pv && pv[0] == '1') ? 1 : 0;
    }
    qtn::g_pdl_next = false;         // a clean state even after an earlier failed call
    bool prev_single_small = false;  // the previous level was one small_kernel launch
    bool prev_single = false;        // the previous level was one launch
    for (size_t lev = 0; lev < B->level_tiles.size(); ++lev) {
      const int g = B->lev_per_group ? (int)(lev / (size_t)B->lev_per_group) : 0;
      if (g != cur_g) {  // the next group: its own lane, a clean PDL state
        cur_g = g;
        gst = g ? B->lane[g] : st;
        gstream = reinterpret_cast<void*>(gst);
        prev_single_small = false;
        prev_single = false;
        qtn::g_pdl_next = false;
      }
      // launches of this level, in issue order: reduce, small, trace, expand, stream
      const uint32_t nsub = B->level_sub0[lev + 1] - B->level_sub0[lev];
      const int n_launch = (int)(B->level_fgroup0[lev + 1] - B->level_fgroup0[lev]) + (nsub ? 1 : 0) +
                           (B->level_red0[lev + 1] > B->level_red0[lev] ? 1 : 0) +
                           (B->level_sitem0[lev + 1] > B->level_sitem0[lev] ? 1 : 0) +
                           (B->level_r1chunks[lev] ? 1 : 0) + (B->level_xtiles[lev] ? 1 : 0) +
                           y_launches(B, lev) + (B->level_tiles[lev] ? 1 : 0) + (B->level_wsctas[lev] ? 1 : 0);
      const bool fork = level_streams && n_launch >= 2 && !B->chain_len[lev];
      // one launch after one launch: PDL for it (QTN_PDL_SINGLE=1; tiny
      // small_kernel levels take it by default below)
      qtn::g_pdl_next = pdl_single_env == 1 && n_launch == 1 && prev_single;
      int slot = 0;  // launch k of the level goes to stream k (0: the group's lane)
      auto next_stream = [&]() -> void* {
        if (!fork) return gstream;
        const int k = std::min(slot++, (int)qtn_batch::kSide);  // more launches than side streams: share the last
        if (k == 0) return gstream;
        cudaStreamWaitEvent(B->gside[g][k - 1], B->gfork[g], 0);
        return reinterpret_cast<void*>(B->gside[g][k - 1]);
      };
      if (fork) cudaEventRecord(B->gfork[g], gst);
      StreamLaunch L;
      std::memset(&L, 0, sizeof(L));
      L.descs = B->d_desc;
      L.n_sets = (uint32_t)n_sets;
      L.in_base = reinterpret_cast<const char*>(inputs);
      L.in_set_stride = 16 * set_stride;
      L.net_in_off = B->d_net_in_off;
      L.ws_base = reinterpret_cast<char*>(workspace);
      L.ws_set_stride = B->ws_per_set;
      L.net_ws_off = B->d_net_ws_off;
      if (B->chain_len[lev]) {
        StreamLaunch Lc = L;
        Lc.item_desc = B->d_sitem_desc;
        Lc.item_net = B->d_sitem_net;
        Lc.n_items = B->level_sitem0.back();
        if ((rc = qtn::launch_chain(Lc, B->d_level_sitem0 + lev, B->chain_len[lev], gstream)))
          return rc;
        lev += B->chain_len[lev] - 1;
        prev_single_small = false;
        prev_single = false;
        qtn::g_pdl_next = false;
        continue;
      }
      const uint32_t ns = B->level_sitem0[lev + 1] - B->level_sitem0[lev];
      // the level's launches (each on its own forked stream); issue order:
      // QTN_LEVEL_ORDER=1 (default) the bulk kernels first (stream, expand,
      // fused, trace, reduce, small, subtrees: config 3 default 3.08 -> 2.96
      // ms); 0: subtrees, fused, reduce, small, trace, expand, stream
      auto l_sub = [&]() -> int {
        if (nsub)
          return qtn::launch_subtree(L, B->d_sub_items + B->level_sub0[lev], nsub, B->d_sub_desc,
                                     B->level_sub_smem[lev], next_stream());
        return QTN_OK;
      };
      auto l_fused = [&]() -> int {
        for (uint32_t gi = B->level_fgroup0[lev]; gi < B->level_fgroup0[lev + 1]; ++gi) {
          const qtn_batch::FGroup& g = B->fgroups[gi];
          if (g.warp) {
            qtn::WLaunch W;
            std::memset(&W, 0, sizeof(W));
            W.blob = B->d_wblob;
            W.recs = B->d_wrecs + g.cta0;
            W.n_warps = (uint32_t)g.ctas;
            W.n_sets = (uint32_t)n_sets;
            W.f64 = g.f64;
            W.in_base = L.in_base;
            W.in_set_stride = L.in_set_stride;
            W.net_in_off = L.net_in_off;
            W.ws_base = L.ws_base;
            W.ws_set_stride = L.ws_set_stride;
            W.net_ws_off = L.net_ws_off;
            const int r2 = qtn::launch_fusedw(W, next_stream());
            if (r2) return r2;
            continue;
          }
          qtn::FLaunch F;
          std::memset(&F, 0, sizeof(F));
          F.descs = B->d_fdesc;
          F.tabs = B->d_ftab;
          F.ctas = B->d_fctas + g.cta0;
          F.blob = B->d_fblob;
          F.item_desc = B->d_fitem_desc + g.item0;
          F.item_net = B->d_fitem_net + g.item0;
          F.cta_prefix = B->d_fprefix + g.prefix0;
          F.n_items = g.n_items;
          F.n_sets = (uint32_t)n_sets;
          F.total_ctas = g.ctas;
          F.smem_bytes = g.smem;
          F.f64 = g.f64;
          F.in_base = L.in_base;
          F.in_set_stride = L.in_set_stride;
          F.net_in_off = L.net_in_off;
          F.ws_base = L.ws_base;
          F.ws_set_stride = L.ws_set_stride;
          F.net_ws_off = L.net_ws_off;
          void* fs = next_stream();
          int r2 = qtn::launch_fused(F, fs);
          if (r2) return r2;
          if (g.cctas) {  // split-K partial sums -> outputs, same stream
            F.cta_prefix = B->d_cprefix + g.prefix0;
            F.total_ctas = g.cctas;
            if ((r2 = qtn::launch_fused_combine(F, fs))) return r2;
          }
        }
        return QTN_OK;
      };
      auto l_red = [&]() -> int {
        const uint32_t nr = B->level_red0[lev + 1] - B->level_red0[lev];
        if (!nr) return QTN_OK;
        return qtn::launch_reduce(L, B->d_red + B->level_red0[lev], B->d_red_prefix + B->level_rprefix0[lev],
                                  nr, B->level_rchunks[lev], next_stream());
      };
      auto l_small = [&]() -> int {
        if (!ns) return QTN_OK;
        StreamLaunch Ls = L;
        Ls.item_desc = B->d_sitem_desc + B->level_sitem0[lev];
        Ls.item_net = B->d_sitem_net + B->level_sitem0[lev];
        Ls.n_items = ns;
        // a level made of this one small launch after a level that was too:
        // PDL (QTN_PDL_TINY=0 disables)
        const bool tiny_pdl = pdl_tiny && n_launch == 1 && prev_single_small;
        return qtn::launch_small(Ls, B->level_smax_r[lev], next_stream(), tiny_pdl);
      };
      auto l_trace = [&]() -> int {
        if (!B->level_r1chunks[lev]) return QTN_OK;
        return qtn::launch_trace(L, B->d_r1 + B->level_r1item0[lev], B->d_r1prefix + B->level_r1prefix0[lev],
                                 B->level_r1item0[lev + 1] - B->level_r1item0[lev], B->level_r1chunks[lev],
                                 next_stream(), B->d_r1chunk_item + B->level_r1chunk0[lev]);
      };
      auto l_expand = [&]() -> int {
        if (!B->level_xtiles[lev]) return QTN_OK;
        qtn::XLaunch X;
        std::memset(&X, 0, sizeof(X));
        X.descs = B->d_xdesc;
        X.item_desc = B->d_xitem_desc + B->level_xitem0[lev];
        X.item_net = B->d_xitem_net + B->level_xitem0[lev];
        X.tile_prefix = B->d_xprefix + B->level_xprefix0[lev];
        X.n_items = B->level_xitem0[lev + 1] - B->level_xitem0[lev];
        X.n_sets = (uint32_t)n_sets;
        X.total_tiles = B->level_xtiles[lev];
        X.stage_bytes = B->level_xstage[lev];
        X.in_base = L.in_base;
        X.in_set_stride = L.in_set_stride;
        X.net_in_off = L.net_in_off;
        X.ws_base = L.ws_base;
        X.ws_set_stride = L.ws_set_stride;
        X.net_ws_off = L.net_ws_off;
        return qtn::launch_expand(X, next_stream());
      };
      auto l_xt = [&]() -> int {
        for (int gq = qtn::kYMaxGB; gq >= 0; --gq) {  // the widest tiles first
          const size_t yi = lev * (qtn::kYMaxGB + 1) + gq;
          if (!B->level_ytiles[yi]) continue;
          qtn::YLaunch Y;
          std::memset(&Y, 0, sizeof(Y));
          Y.descs = B->d_ydesc;
          Y.item_desc = B->d_yitem_desc + B->level_yitem0[yi];
          Y.item_net = B->d_yitem_net + B->level_yitem0[yi];
          Y.tile_prefix = B->d_yprefix + B->level_yprefix0[yi];
          Y.n_items = B->level_yitem0[yi + 1] - B->level_yitem0[yi];
          Y.n_sets = (uint32_t)n_sets;
          Y.total_tiles = B->level_ytiles[yi];
          Y.stage_bytes = B->level_ystage[yi];
          Y.g = (uint32_t)gq;
          Y.in_base = L.in_base;
          Y.in_set_stride = L.in_set_stride;
          Y.net_in_off = L.net_in_off;
          Y.ws_base = L.ws_base;
          Y.ws_set_stride = L.ws_set_stride;
          Y.net_ws_off = L.net_ws_off;
          const int r2 = qtn::launch_xt(Y, next_stream());
          if (r2) return r2;
        }
        return QTN_OK;
      };
      auto l_ws = [&]() -> int {
        if (!B->level_wsctas[lev]) return QTN_OK;
        qtn::WsLaunch W;
        std::memset(&W, 0, sizeof(W));
        W.descs = B->d_wsdesc;
        W.item_desc = B->d_wsitem_desc + B->level_ws0[lev];
        W.item_net = B->d_wsitem_net + B->level_ws0[lev];
        W.cta_prefix = B->d_wsprefix + B->level_wsprefix0[lev];
        W.n_items = B->level_ws0[lev + 1] - B->level_ws0[lev];
        W.n_sets = (uint32_t)n_sets;
        W.total_ctas = B->level_wsctas[lev];
        W.in_base = L.in_base;
        W.in_set_stride = L.in_set_stride;
        W.net_in_off = L.net_in_off;
        W.ws_base = L.ws_base;
        W.ws_set_stride = L.ws_set_stride;
        W.net_ws_off = L.net_ws_off;
        return qtn::launch_wsum(W, next_stream());
      };
      auto l_stream = [&]() -> int {
        if (!B->level_tiles[lev]) return QTN_OK;
        StreamLaunch Lt = L;
        Lt.item_desc = B->d_item_desc + B->level_item0[lev];
        Lt.item_net = B->d_item_net + B->level_item0[lev];
        Lt.tile_prefix = B->d_tile_prefix + B->level_prefix0[lev];
        Lt.n_items = B->level_item0[lev + 1] - B->level_item0[lev];
        Lt.total_tiles = B->level_tiles[lev];
        // many items of few tiles each (per-item setup dominates): the
        // 16-consumer-warp build hides more latency (measured: config 3 default)
        const char* wv = getenv("QTN_WIDE_TPI");
        const uint64_t wide_tpi = wv ? strtoull(wv, nullptr, 10) : 32;
        const bool wide = Lt.total_tiles < wide_tpi * Lt.n_items;
        return launch_stream(Lt, next_stream(), wide);
      };
      static int lorder = -1;
      if (lorder < 0) {
        const char* ov = getenv("QTN_LEVEL_ORDER");
        lorder = ov ? atoi(ov) : 1;
      }
      if (lorder == 1) {
        if ((rc = l_stream()) || (rc = l_xt()) || (rc = l_ws()) || (rc = l_expand()) || (rc = l_fused()) || (rc = l_trace()) || (rc = l_red()) ||
            (rc = l_small()) || (rc = l_sub()))
          return rc;
      } else {
        if ((rc = l_sub()) || (rc = l_fused()) || (rc = l_red()) || (rc = l_small()) || (rc = l_trace()) ||
            (rc = l_expand()) || (rc = l_xt()) || (rc = l_ws()) || (rc = l_stream()))
          return rc;
      }
      // join: the next level (or the fold) waits for every branch
      for (int k = 1; k < std::min(slot, (int)qtn_batch::kSide + 1); ++k) {
        cudaEventRecord(B->gjoin[g][k - 1], B->gside[g][k - 1]);
        cudaStreamWaitEvent(gst, B->gjoin[g][k - 1], 0);
      }
      prev_single_small = n_launch == 1 && ns != 0;
      prev_single = n_launch == 1;
      qtn::g_pdl_next = false;
    }
    for (int g = 1; g < G; ++g) {  // join the lanes
      cudaEventRecord(B->ev_lane_done[g], B->lane[g]);
      cudaStreamWaitEvent(st, B->ev_lane_done[g], 0);
    }
    dim3 grid((B->n_hbm + 127) / 128, n_sets);
    cudaError_t e = launch_pdl<true>(
        hbm_fold_kernel, grid, dim3(128), 0, st, (const uint64_t*)B->d_fold_tags,
        (const uint8_t*)B->d_fold_c64, (const uint32_t*)B->d_fold_first,
        (const int32_t*)B->d_fold_pow2, (const int32_t*)B->d_hbm_index, B->n_hbm, B->n,
        reinterpret_cast<const char*>(inputs), (int64_t)(16 * set_stride),
        (const int64_t*)B->d_net_in_off, reinterpret_cast<const char*>(workspace),
        (int64_t)B->ws_per_set, (const int64_t*)B->d_net_ws_off,
        reinterpret_cast<double2*>(results));
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "hbm_fold_kernel launch");
  }
  return QTN_OK;
}

extern "C" int qtn_tensorgen(const qtn_tensor_recipe* recipes, int64_t n, const double* angles,
                             int32_t n_angles, int32_t n_sets, int64_t set_elems, void* out,
                             void* stream) {
  if (n < 0 || n_sets < 1 || n_sets > 65535 || (n > 0 && (!recipes || !out))) {
    set_error("qtn_tensorgen: bad arguments");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  if (n == 0) return QTN_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  dim3 grid((unsigned)((n + 127) / 128), n_sets);
  cudaError_t e = launch_pdl<true>(tensorgen_kernel, grid, dim3(128), 0, st, recipes, n, angles,
                             (int)n_angles, set_elems, reinterpret_cast<double2*>(out));
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "tensorgen launch");
  return QTN_OK;
}

extern "C" int qtn_energy_reduce(const void* values, const double* weights, int32_t n,
                                 int32_t n_sets, double* energies, void* zz_sum, void* stream) {
  if (!values || n < 0 || n_sets < 1) {
    set_error("qtn_energy_reduce: bad arguments");
    return QTN_EINVAL;
  }
  int rc = device_check();
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  energy_kernel<<<n_sets, 128, 0, st>>>(reinterpret_cast<const double2*>(values), weights, n,
                                       energies, reinterpret_cast<double2*>(zz_sum));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "energy launch");
  return QTN_OK;
}

extern "C" int qtn_batch_energies_host(qtn_batch* B, const double* angles_host, int32_t n_angles,
                                       int32_t n_sets, double* angles_dev, void* inputs_scratch,
                                       void* workspace, void* results, const double* weights_dev,
                                       double* energies_dev, double* energies_host, void* stream) {
  if (!B || !angles_host || !angles_dev || !energies_dev || !energies_host || n_sets < 1 ||
      n_angles < 1) {
    set_error("qtn_batch_energies_host: bad arguments");
    return QTN_EINVAL;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t na = (size_t)n_sets * n_angles, need = na + (size_t)n_sets;
  if (B->pin_doubles < need) {
    if (B->pin) cudaFreeHost(B->pin);
    B->pin = nullptr;
    B->pin_doubles = 0;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&B->pin), need * sizeof(double),
                                  cudaHostAllocDefault);
    if (e != cudaSuccess) return cuda_fail(e, "pinned staging");
    B->pin_doubles = need;
  }
  std::memcpy(B->pin, angles_host, na * sizeof(double));
  double* eh = B->pin + na;
  // the whole call as one graph: H2D, evaluation, reduction, D2H (QTN_GRAPHS=0:
  // stream-ordered calls)
  auto body = [&](cudaStream_t s2) -> int {
    cudaError_t e2 = cudaMemcpyAsync(angles_dev, B->pin, na * sizeof(double), cudaMemcpyHostToDevice, s2);
    if (e2 != cudaSuccess) return cuda_fail(e2, "angles H2D");
    int rc2 = execute_angles_direct(B, angles_dev, n_angles, n_sets, inputs_scratch, workspace, results, s2);
    if (rc2) return rc2;
    if ((rc2 = qtn_energy_reduce(results, weights_dev, B->n, n_sets, energies_dev, nullptr, s2))) return rc2;
    e2 = cudaMemcpyAsync(eh, energies_dev, (size_t)n_sets * sizeof(double), cudaMemcpyDeviceToHost, s2);
    if (e2 != cudaSuccess) return cuda_fail(e2, "energies D2H");
    return QTN_OK;
  };
  const char* gv = getenv("QTN_GRAPHS");
  cudaError_t e = cudaSuccess;
  if (gv && gv[0] == '0') {
    int rc = body(st);
    if (rc) return rc;
  } else {
    const std::vector<uintptr_t> key{(uintptr_t)angles_dev, (uintptr_t)inputs_scratch, (uintptr_t)workspace,
                                     (uintptr_t)results, (uintptr_t)weights_dev, (uintptr_t)energies_dev,
                                     (uintptr_t)B->pin, (uintptr_t)n_angles, (uintptr_t)n_sets};
    auto it = B->egraphs.find(key);
    if (it == B->egraphs.end()) {
      if (B->egraphs.size() >= 16) {
        for (auto& kv : B->egraphs) cudaGraphExecDestroy(kv.second);
        B->egraphs.clear();
      }
      if (!B->cap_stream && cudaStreamCreateWithFlags(&B->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "capture stream");
      cudaGraph_t g = nullptr;
      e = cudaStreamBeginCapture(B->cap_stream, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_fail(e, "graph capture begin");
      const int rc = body(B->cap_stream);
      e = cudaStreamEndCapture(B->cap_stream, &g);
      if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e != cudaSuccess) return cuda_fail(e, "graph capture end");
      cudaGraphExec_t ex = nullptr;
      e = cudaGraphInstantiate(&ex, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) return cuda_fail(e, "graph instantiate");
      it = B->egraphs.emplace(key, ex).first;
    }
    e = cudaGraphLaunch(it->second, st);
    if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  }
  e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "energies sync");
  std::memcpy(energies_host, eh, (size_t)n_sets * sizeof(double));
  return QTN_OK;
}
