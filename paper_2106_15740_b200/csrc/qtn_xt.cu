// Expanding bucket + its consumer in one pass (sm_100a).  An expanding
// bucket writes the widest tensor of a network (O1, e.g. rank 26 in config
// 4: 512 MB) and the next bucket reads it back once to eliminate one more
// variable (contraction.py:90-96, twice in a row).  Here
//   O2[o] = sum_{v2} W_{v2}(o) * sum_{v1} A_{v1,v2}(o) * B_{v1,v2}(o)
// is evaluated per O2 element, so O1 never exists in memory: the pair moves
// its small inputs and O2 only (qtn_stream.h YDesc for the index split).
//
// Persistent CTAs of 256 threads walk contiguous tile ranges; per tile
// (2^9 A positions x 2^h B positions):
//   1. B group -> shared memory Bst[x_b][x_c][v2][v1] (cp.async gather-copy
//      when it is one complex64 operand), W group -> Wst[x_b][x_w][v2];
//   2. per thread the A-type product for its 2 adjacent outputs x (v2, v1);
//   3. for each x_b: 4 (+2) 16-byte shared loads, 32 (+16) FMAs, one 16-byte
//      store (a warp writes 512 contiguous bytes).
// complex64 intermediates: operand products are formed in float64 and
// rounded once, the inner loop is float32 (the storage policy of the unfused
// buckets, whose O1 would have been rounded to complex64 as well).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

namespace qtn {
namespace {

__device__ __forceinline__ double2 ycmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ uint64_t ygather(uint64_t o, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((o >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}
__device__ __forceinline__ const char* yresolve(uint64_t tag, const char* in, char* ws) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return in + off;
  if (sel == 2) return ws + off;
  return reinterpret_cast<const char*>(off);
}
__device__ __forceinline__ double2 yld(const char* p, uint32_t i, uint32_t c64) {
  if (c64) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return make_double2(f.x, f.y);
  }
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
// a0 * (b.x, b.y) + a1 * (b.z, b.w)
__device__ __forceinline__ float2 mac2(float2 a0, float2 a1, float4 b) {
  float2 r;
  r.x = fmaf(a0.x, b.x, fmaf(-a0.y, b.y, fmaf(a1.x, b.z, -a1.y * b.w)));
  r.y = fmaf(a0.x, b.y, fmaf(a0.y, b.x, fmaf(a1.x, b.w, a1.y * b.z)));
  return r;
}

#ifndef XT_MINB1
#define XT_MINB1 4
#endif
#ifndef XT_UNROLL
#define XT_UNROLL 1
#endif
constexpr int kXtUnroll = XT_UNROLL;
constexpr int kYG = 2 * kYMaxG;  // staged operands (B group, then W group)
constexpr int kYMaxGroups = 1 << kYMaxGB;

// Per-item state in shared memory (rebuilt when a CTA moves to a new item):
// gathers are OR-linear over disjoint output bits, so a staged operand index
// is base(tile) + tb[x_b] + tc[x_c or x_w] + v strides.
struct YItemSmem {
  const char* ptr[kYOps];
  uint32_t base[kYOps];          // per tile
  uint32_t s1[kYOps], s2[kYOps]; // element strides of v1 / v2 (0: independent)
  uint32_t tb[kYG][1 << kYMaxH];
  uint32_t tc[kYG][512];
  uint32_t goff[kYMaxA][kYMaxGroups];  // A-type operand offset of group gi
  uint32_t gb[kYMaxGroups];            // x_c part of group gi
  uint32_t gw[kYMaxGroups];            // x_w part of group gi
  uint8_t c64[kYOps];
};

// Stage layout: the B group as two planes of float4 (v2 = 0 / 1), each
// [x_b][x_c] -> (v1 = 0, v1 = 1): a warp whose lanes differ in x_c reads
// consecutive 16-byte words (no bank conflicts); the W group [x_b][x_w] ->
// (v2 = 0, v2 = 1) after them.
// prev[0..3]: the operand bases the stages were last filled for (B group,
// W group); a tile whose bases are unchanged reuses them (the host orders the
// tile index so that consecutive tiles differ in bits a group does not see)
template <bool HASW, int G>
__device__ __forceinline__ void xt_tile(const YDesc& d, YItemSmem& X, const uint32_t* ea,
                                        const uint32_t* eb, uint32_t xc0, uint32_t xc1,
                                        uint32_t xw0, uint32_t xw1, uint64_t obase, float2* out,
                                        uint32_t bmask, unsigned char* smem, uint32_t* prev) {
  const uint32_t tid = threadIdx.x;
  const uint32_t c = d.c, cw = d.cw, h = d.h, nA = d.nA, nB = d.nB, nW = d.nW;
  const uint32_t nOps = nA + nB + nW;
  if (tid < nOps) X.base[tid] = (uint32_t)ygather(obase, d.ops[tid].runs, d.ops[tid].n_runs);
  __syncthreads();
  // 1. stages.  B entry i = (row << 2) | v2 << 1 | v1, row = x_b << c | x_c
  const uint32_t nBst = 4u << (h + c);
  float2* stB = reinterpret_cast<float2*>(smem);
  const uint32_t kYPlane = nBst * 4u, kYWOff = nBst * 8u;  // plane v2 = 1 and the W stage follow plane 0
  float2* stW = reinterpret_cast<float2*>(smem + kYWOff);
  bool async = false;
  bool fillB = false, fillW = false;
#ifdef XT_NOPREV
  fillB = fillW = true;
#endif
#pragma unroll
  for (uint32_t q = 0; q < kYMaxG; ++q) {  // (unrolled: prev stays in registers)
    if (q < nB) {
      const uint32_t bq = X.base[nA + q];
      fillB |= prev[q] != bq;
      prev[q] = bq;
    }
    if (q < nW) {
      const uint32_t bq = X.base[nA + nB + q];
      fillW |= prev[kYMaxG + q] != bq;
      prev[kYMaxG + q] = bq;
    }
  }
  if (!fillB) {
  } else if (nB == 1 && X.c64[nA]) {
    async = true;
    const float2* src = reinterpret_cast<const float2*>(X.ptr[nA]) + X.base[nA];
    const uint32_t s1 = X.s1[nA], s2 = X.s2[nA], cm = (1u << c) - 1u;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(stB));
    for (uint32_t i = tid; i < nBst; i += 256) {
      const uint32_t row = i >> 2, v2 = (i >> 1) & 1u, v1 = i & 1u;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + v2 * kYPlane + 8u * (2u * row + v1)),
                   "l"(src + X.tb[0][row >> c] + X.tc[0][row & cm] + v1 * s1 + v2 * s2)
                   : "memory");
    }
  } else {
    const uint32_t cm = (1u << c) - 1u;
    for (uint32_t i = tid; i < nBst; i += 256) {
      const uint32_t row = i >> 2, v2 = (i >> 1) & 1u, v1 = i & 1u;
      double2 pr = make_double2(1.0, 0.0);
      for (uint32_t q = 0; q < nB; ++q) {
        const uint32_t k = nA + q;
        pr = ycmul(pr, yld(X.ptr[k], X.base[k] + X.tb[q][row >> c] + X.tc[q][row & cm] + v1 * X.s1[k] +
                                         v2 * X.s2[k], X.c64[k]));
      }
      stB[v2 * (kYPlane / 8) + 2u * row + v1] = make_float2((float)pr.x, (float)pr.y);
    }
  }
  if (HASW && fillW) {
    const uint32_t nWst = 2u << (h + cw), cm = (1u << cw) - 1u, kW = nA + nB;
    if (nW == 1 && X.c64[kW]) {
      async = true;
      const float2* src = reinterpret_cast<const float2*>(X.ptr[kW]) + X.base[kW];
      const uint32_t s2 = X.s2[kW];
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(stW));
      for (uint32_t i = tid; i < nWst; i += 256)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * i),
                     "l"(src + X.tb[kYMaxG][i >> (cw + 1)] + X.tc[kYMaxG][(i >> 1) & cm] + (i & 1u) * s2)
                     : "memory");
    } else {
      for (uint32_t i = tid; i < nWst; i += 256) {
        const uint32_t xw = (i >> 1) & cm, xb = i >> (cw + 1);
        double2 pr = make_double2(1.0, 0.0);
        for (uint32_t q = 0; q < nW; ++q) {
          const uint32_t k = kW + q;
          pr = ycmul(pr, yld(X.ptr[k], X.base[k] + X.tb[kYMaxG + q][xb] + X.tc[kYMaxG + q][xw] +
                                           (i & 1u) * X.s2[k], X.c64[k]));
        }
        stW[i] = make_float2((float)pr.x, (float)pr.y);
      }
    }
  }
  if (async) asm volatile("cp.async.commit_group;\n" ::: "memory");
  // 2. A-type product of this thread's outputs: a[group][j][v2][v1], formed
  // in float (complex128 gate entries rounded once); the 8 loads of an
  // operand issue together
  float2 a[G][2][2][2];
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v2 = 0; v2 < 2; ++v2)
#pragma unroll
        for (int v1 = 0; v1 < 2; ++v1) a[gi][j][v2][v1] = make_float2(1.f, 0.f);
#pragma unroll
    for (uint32_t k = 0; k < kYMaxA; ++k) {
      if (k < nA) {
        const uint32_t i0 = X.base[k] + ea[k] + X.goff[k][gi], s1 = X.s1[k], s2 = X.s2[k];
        float2 v[2][2][2];
        if (X.c64[k]) {
          const float2* pk = reinterpret_cast<const float2*>(X.ptr[k]) + i0;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v2 = 0; v2 < 2; ++v2)
#pragma unroll
              for (int v1 = 0; v1 < 2; ++v1) v[j][v2][v1] = __ldg(pk + (j * eb[k] + v2 * s2 + v1 * s1));
        } else {
          const double2* pk = reinterpret_cast<const double2*>(X.ptr[k]) + i0;
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v2 = 0; v2 < 2; ++v2)
#pragma unroll
              for (int v1 = 0; v1 < 2; ++v1) {
                const double2 t = __ldg(pk + (j * eb[k] + v2 * s2 + v1 * s1));
                v[j][v2][v1] = make_float2((float)t.x, (float)t.y);
              }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int v2 = 0; v2 < 2; ++v2)
#pragma unroll
            for (int v1 = 0; v1 < 2; ++v1) {
              const float2 x = a[gi][j][v2][v1], y = v[j][v2][v1];
              a[gi][j][v2][v1] = make_float2(fmaf(x.x, y.x, -x.y * y.y), fmaf(x.x, y.y, x.y * y.x));
            }
      }
    }
  }
  if (async) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // 3. outputs.  x_b = kept << hs | summed: the shared-memory rows advance by
  // one stride per x_b; the hs summed loop bits and the 2^g groups accumulate
  // in registers, one 16-byte store per kept value (masked increment of the
  // output offset)
  const uint32_t nk = 1u << (h - d.hs), ns = 1u << d.hs;
  const bool pairb = xc0 == xc1;  // uniform per item: output bit 0 outside the B group
  const float4* pb0 = reinterpret_cast<const float4*>(smem) + xc0;
  const float4* pb1 = reinterpret_cast<const float4*>(smem) + xc1;
  const uint32_t plane = nBst >> 2;  // float4 words to plane v2 = 1
  const uint32_t strideB = 1u << c, strideW = 1u << cw;
  const float4* pw0 = reinterpret_cast<const float4*>(stW) + xw0;
  const float4* pw1 = reinterpret_cast<const float4*>(stW) + xw1;
  uint32_t gb[G], gw[G];
  bool gdepb = false;
#pragma unroll
  for (int gi = 0; gi < G; ++gi) {
    gb[gi] = X.gb[gi];
    gw[gi] = X.gw[gi];
    gdepb |= gb[gi] != 0u;
  }
  uint32_t ob = 0;
#pragma unroll 1
  for (uint32_t kept = 0; kept < nk; ++kept) {
    float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll 1
    for (uint32_t sv = 0; sv < ns; ++sv) {
      float4 b00, b01, b10, b11;
#pragma unroll
      for (int gi = 0; gi < G; ++gi) {
        if (gi == 0 || gdepb) {
          b00 = pb0[gb[gi]];
          b01 = pb0[gb[gi] + plane];
          b10 = b00;
          b11 = b01;
          if (!pairb) {
            b10 = pb1[gb[gi]];
            b11 = pb1[gb[gi] + plane];
          }
        }
        const float2 t00 = mac2(a[gi][0][0][0], a[gi][0][0][1], b00), t01 = mac2(a[gi][0][1][0], a[gi][0][1][1], b01);
        const float2 t10 = mac2(a[gi][1][0][0], a[gi][1][0][1], b10), t11 = mac2(a[gi][1][1][0], a[gi][1][1][1], b11);
        if (HASW) {
          const float4 w0 = pw0[gw[gi]], w1 = pw1[gw[gi]];
          const float2 r0 = mac2(t00, t01, w0), r1 = mac2(t10, t11, w1);
          acc0.x += r0.x;
          acc0.y += r0.y;
          acc1.x += r1.x;
          acc1.y += r1.y;
        } else {
          acc0.x += t00.x + t01.x;
          acc0.y += t00.y + t01.y;
          acc1.x += t10.x + t11.x;
          acc1.y += t10.y + t11.y;
        }
      }
      pb0 += strideB;
      pb1 += strideB;
      if (HASW) {
        pw0 += strideW;
        pw1 += strideW;
      }
    }
    __stcs(reinterpret_cast<float4*>(out + ob), make_float4(acc0.x, acc0.y, acc1.x, acc1.y));
    ob = ((ob | ~bmask) + 1u) & bmask;
  }
}

template <int G>
__device__ __forceinline__ void xt_body(const YLaunch& L, unsigned char* ysmem, YItemSmem& X, YDesc& SD) {
  const uint64_t per = (L.total_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = min(L.total_tiles, t0 + per);
  const uint32_t set = blockIdx.y, tid = threadIdx.x;
  uint64_t item_end = 0, first = 0;
  uint32_t bmask = 0;
  uint32_t prev[kYG];
  const YDesc* d = &SD;
  const char* in = nullptr;
  char* ws = nullptr;
  uint32_t ea[kYMaxA], eb[kYMaxA];
  uint32_t xc0 = 0, xc1 = 0, xw0 = 0, xw1 = 0;
  uint64_t oa = 0;
  for (uint64_t t = t0; t < t1; ++t) {
    if (t >= item_end) {
      uint32_t lo = 0, hi = L.n_items;  // last item whose first tile <= t
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (L.tile_prefix[mid] <= t) lo = mid;
        else hi = mid;
      }
      first = L.tile_prefix[lo];
      item_end = L.tile_prefix[lo + 1];
      const YDesc* gd = &L.descs[L.item_desc[lo]];
      const uint32_t net = L.item_net[lo];
      in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
      ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
      __syncthreads();  // the previous item's tables and descriptor are no longer read
      for (uint32_t i = tid; i < sizeof(YDesc) / 16; i += 256)
        reinterpret_cast<uint4*>(&SD)[i] = __ldg(reinterpret_cast<const uint4*>(gd) + i);
      __syncthreads();
      const uint32_t nA = d->nA, nB = d->nB, nW = d->nW, nOps = nA + nB + nW;
      if (tid < nOps) {
        const YOp& op = d->ops[tid];
        X.ptr[tid] = yresolve(op.ptr, in, ws);
        X.s1[tid] = op.vs1 == 0xff ? 0u : 1u << op.vs1;
        X.s2[tid] = op.vs2 == 0xff ? 0u : 1u << op.vs2;
        X.c64[tid] = op.c64;
      }
      if (tid < kYMaxGroups) {  // group gi = element bits 9.. (0 beyond 2^g)
        const uint32_t e = (tid < (1u << d->g)) ? tid << kXABits : 0u;
        const uint64_t o = ygather(e, d->arun, d->n_arun);  // extended bits of the group's summed variables
        X.gb[tid] = (uint32_t)ygather(e, d->acrun, d->n_acrun);
        X.gw[tid] = (uint32_t)ygather(e, d->awrun, d->n_awrun);
        for (uint32_t k = 0; k < nA; ++k)
          X.goff[k][tid] = (uint32_t)ygather(o, d->ops[k].runs, d->ops[k].n_runs);
      }
      for (uint32_t q = 0; q < nB + nW; ++q) {
        const bool isw = q >= nB;
        const YOp& op = d->ops[nA + q];
        const uint32_t slot = isw ? kYMaxG + (q - nB) : q;
        for (uint32_t i = tid; i < (1u << d->h); i += 256)
          X.tb[slot][i] = (uint32_t)ygather(ygather(i, d->brun, d->n_brun), op.runs, op.n_runs);
        const uint32_t nc = 1u << (isw ? d->cw : d->c);
        for (uint32_t i = tid; i < nc; i += 256)
          X.tc[slot][i] = (uint32_t)ygather(
              isw ? ygather(i, d->wrun, d->n_wrun) : ygather(i, d->crun, d->n_crun), op.runs, op.n_runs);
      }
      const uint32_t e0 = 2u * tid;
      oa = ygather(e0, d->arun, d->n_arun);
#pragma unroll
      for (uint32_t k = 0; k < kYMaxA; ++k) {
        ea[k] = 0;
        eb[k] = 0;
        if (k < nA) {
          ea[k] = (uint32_t)ygather(oa, d->ops[k].runs, d->ops[k].n_runs);
          eb[k] = (uint32_t)ygather(1u, d->ops[k].runs, d->ops[k].n_runs);  // output bit 0
        }
      }
      xc0 = (uint32_t)ygather(e0, d->acrun, d->n_acrun);
      xc1 = (uint32_t)ygather(e0 + 1u, d->acrun, d->n_acrun);
      xw0 = (uint32_t)ygather(e0, d->awrun, d->n_awrun);
      xw1 = (uint32_t)ygather(e0 + 1u, d->awrun, d->n_awrun);
      // output bits of the kept loop bits (output rank <= 32, host check: 32-bit element offsets)
      bmask = (uint32_t)ygather(((1u << d->h) - 1u) ^ ((1u << d->hs) - 1u), d->brun, d->n_brun);
#pragma unroll
      for (int q = 0; q < kYG; ++q) prev[q] = 0xffffffffu;  // no stage of this item yet
    } else {
      __syncthreads();  // stage reuse
    }
    const uint64_t obase = ygather(t - first, d->trun, d->n_trun);
    float2* outp = reinterpret_cast<float2*>(const_cast<char*>(yresolve(d->out, in, ws))) + (obase | oa);
    if (d->nW)
      xt_tile<true, G>(*d, X, ea, eb, xc0, xc1, xw0, xw1, obase, outp, bmask, ysmem, prev);
    else
      xt_tile<false, G>(*d, X, ea, eb, xc0, xc1, xw0, xw1, obase, outp, bmask, ysmem, prev);
  }
}

// One launch holds items of one group count (the executor launches per g).
template <int G, int MINB>
__global__ void __launch_bounds__(256, MINB) xt_kernel(const __grid_constant__ YLaunch L) {
  extern __shared__ __align__(16) unsigned char ysmem[];
  __shared__ YItemSmem X;
  __shared__ __align__(16) YDesc SD;
  pdl_trigger();
  pdl_wait();
  xt_body<G>(L, ysmem, X, SD);
}

}  // namespace

template <int G, int MINB>
static int xt_ctas_per_sm(uint32_t stage_bytes) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, xt_kernel<G, MINB>, 256, stage_bytes) !=
      cudaSuccess)
    per_sm = MINB;
  return std::max(1, per_sm);
}

template <int G, int MINB>
static int launch_xt_g(const YLaunch& L, void* stream) {
  static std::atomic<uint64_t> attr{0};
  if (needs_setup(attr)) {
    cudaError_t e = cudaFuncSetAttribute(xt_kernel<G, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (kYStageB + kYStageW) * 8);
    if (e != cudaSuccess) {
      set_error(std::string("xt_kernel attribute: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    mark_setup(attr);
  }
  int n_sm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (n_sm <= 0) n_sm = 148;
  int per_sm = 0;
  const char* xc = getenv("QTN_XT_CTAS");
  if (xc) per_sm = atoi(xc);
  if (per_sm <= 0) per_sm = xt_ctas_per_sm<G, MINB>(L.stage_bytes);
  const uint64_t ctas = std::min<uint64_t>(L.total_tiles, (uint64_t)n_sm * (uint64_t)per_sm);
  dim3 grid((uint32_t)ctas, L.n_sets);
  cudaError_t e = launch_pdl<true>(xt_kernel<G, MINB>, grid, dim3(256), L.stage_bytes,
                                   reinterpret_cast<cudaStream_t>(stream), L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("xt_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

// The register bound follows the shared-memory bound: a launch whose stages
// leave room for fewer CTAs per SM than the default build's register budget
// targets runs the build compiled for that CTA count (more registers, no
// spills).  QTN_XT_REGS=0: always the default builds.
template <int G, int MINB>
static int launch_xt_fit(const YLaunch& L, void* stream) {
  static const bool fit = [] {
    const char* e = getenv("QTN_XT_REGS");
    return !e || atoi(e) != 0;
  }();
  if (fit && MINB > 2 && xt_ctas_per_sm<G, MINB>(L.stage_bytes) < MINB)
    return launch_xt_g<G, MINB - 1>(L, stream);
  return launch_xt_g<G, MINB>(L, stream);
}

int launch_xt(const YLaunch& L, void* stream) {
  if (!L.n_items || !L.n_sets || !L.total_tiles) return QTN_OK;
  if (L.n_sets > 65535 || L.total_tiles > 0x7fffffffull) {
    set_error("xt_kernel: grid too large");
    return QTN_EINVAL;
  }
  // the launch's items share one group count (level lists are built per g)
  switch (L.g) {
    case 0: return launch_xt_fit<1, XT_MINB1>(L, stream);
    case 1: return launch_xt_fit<2, 3>(L, stream);
    default: return launch_xt_g<4, 2>(L, stream);
  }
}

}  // namespace qtn
