// Expanding-bucket kernel (sm_100a): buckets whose output is wider than
// their primary operand, e.g. two rank-17 operands -> a rank-25 output in
// config 4 (contraction.py:42-54 `_product` + :94-96 `.sum`).  Such a bucket
// is an outer product summed over the eliminated variable v:
//   out[o] = sum_v A_v(o) * B_v(o)
// with A_v the product of the operands that live on the primary's variables
// and B_v the product of the others.  It moves few input bytes and many
// output bytes, so it is bound by the output write stream when each output
// costs a handful of instructions; the streaming tile kernel (which gathers
// every non-primary operand per output element) spends ~60 there.
//
// Persistent CTAs of 256 threads walk contiguous tile ranges; per tile
// (2^9 A positions x 2^h B positions):
//   1. the B-side product over (x_b, x_c, v) into shared memory, x_c = the
//      tile-local A bits a B-side operand depends on (host keeps it small);
//   2. per thread A_v for its two adjacent outputs (primary: coalesced);
//   3. for each x_b: two 16-byte shared loads, the v-sum, one 16-byte store
//      (a warp writes 512 contiguous bytes).
// Products of the staged/A factors are formed in float64; the inner loop is
// float32 for complex64 outputs (the complex64 storage policy), float64 for
// complex128 outputs.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

namespace qtn {
namespace {

__device__ __forceinline__ double2 xcmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ uint64_t xgather(uint64_t o, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((o >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}
__device__ __forceinline__ const char* xresolve(uint64_t tag, const char* in, char* ws) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return in + off;
  if (sel == 2) return ws + off;
  return reinterpret_cast<const char*>(off);
}

__device__ __forceinline__ float4 f4mac(float2 a0, float2 a1, float4 b) {
  // a0 * (b.x, b.y) + a1 * (b.z, b.w) for one output, packed as float2 in .xy
  float2 r;
  r.x = fmaf(a0.x, b.x, fmaf(-a0.y, b.y, fmaf(a1.x, b.z, -a1.y * b.w)));
  r.y = fmaf(a0.x, b.y, fmaf(a0.y, b.x, fmaf(a1.x, b.w, a1.y * b.z)));
  return make_float4(r.x, r.y, 0.f, 0.f);
}

// Per-item state in shared memory (rebuilt when a CTA moves to a new item):
// gathers are OR-linear over disjoint output bits, so an operand index is
// base(tile) + tb[x_b] + tc[x_c] (B side) or base(tile) + ea(e) (A side),
// with the tile-independent parts tabulated once per item.
struct XItemSmem {
  const char* ptr[2 * kXMaxOps];
  uint32_t base[2 * kXMaxOps];         // per tile
  uint32_t tb[kXMaxOps][256];          // B ops: x_b -> operand offset
  uint32_t tc[kXMaxOps][512];          // B ops: x_c -> operand offset
  uint8_t vs[2 * kXMaxOps], c64[2 * kXMaxOps];
};

__device__ __forceinline__ double2 xld32(const char* p, uint32_t i, uint32_t c64) {
  if (c64) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return make_double2(f.x, f.y);
  }
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}

template <bool F32>
__device__ __forceinline__ void expand_tile(const XDesc& d, XItemSmem& X, const uint32_t* ea,
                                            const uint32_t* eb, uint64_t obase, char* outp,
                                            unsigned char* smem) {
  const uint32_t tid = threadIdx.x;
  const uint32_t c = d.c, h = d.h, nA = d.nA, nAB = d.nA + d.nB;
  // per-tile operand bases
  if (tid < nAB) X.base[tid] = (uint32_t)xgather(obase, d.ops[tid].runs, d.ops[tid].n_runs);
  __syncthreads();
  // 1. B-side stage: entry ((x_b << c) | x_c) * 2 + v
  const uint32_t n_st = 2u << (h + c);
  const bool async_stage = F32 && d.nB == 1 && X.c64[nA];
  if (async_stage) {
    // one complex64 B operand (all of configs 3-4): the stage is a
    // gather-copy, issued as cp.async (every copy of the thread in flight at
    // once, no register round trip); the A-side loads below overlap it
    const float2* src = reinterpret_cast<const float2*>(X.ptr[nA]) + X.base[nA];
    const uint32_t vs = X.vs[nA], cm = (1u << c) - 1u;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    for (uint32_t i = tid; i < n_st; i += 256)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 8u * i),
                   "l"(src + X.tb[0][i >> (c + 1)] + X.tc[0][(i >> 1) & cm] + ((i & 1u) << vs))
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  } else
  for (uint32_t i = tid; i < n_st; i += 256) {
    const uint32_t v = i & 1u, xc = (i >> 1) & ((1u << c) - 1u), xb = i >> (c + 1);
    double2 pr = make_double2(1.0, 0.0);
    for (uint32_t k = nA; k < nAB; ++k) {
      const uint32_t q = k - nA;
      const uint32_t idx = X.base[k] + X.tb[q][xb] + X.tc[q][xc] + (v << X.vs[k]);
      pr = xcmul(pr, xld32(X.ptr[k], idx, X.c64[k]));
    }
    if (F32)
      reinterpret_cast<float2*>(smem)[i] = make_float2((float)pr.x, (float)pr.y);
    else
      reinterpret_cast<double2*>(smem)[i] = pr;
  }
  // 2. A-side factors of this thread's two adjacent outputs
  double2 a00 = make_double2(1.0, 0.0), a01 = a00, a10 = a00, a11 = a00;
#pragma unroll
  for (uint32_t k = 0; k < kXMaxOps; ++k) {
    if (k < nA) {
      const uint32_t i0 = X.base[k] + ea[k], i1 = i0 + eb[k], vb = 1u << X.vs[k];
      a00 = xcmul(a00, xld32(X.ptr[k], i0, X.c64[k]));
      a01 = xcmul(a01, xld32(X.ptr[k], i0 + vb, X.c64[k]));
      a10 = xcmul(a10, xld32(X.ptr[k], i1, X.c64[k]));
      a11 = xcmul(a11, xld32(X.ptr[k], i1 + vb, X.c64[k]));
    }
  }
  const uint32_t cx0 = ea[kXMaxOps] << 1, cx1 = eb[kXMaxOps] << 1;
  if (async_stage) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // x_b -> output offset by a masked increment (pdep of a counter)
  uint64_t bmask = 0;
  for (uint32_t r = 0; r < d.n_brun; ++r) {
    const uint32_t w = d.brun[r];
    bmask |= ((1ull << ((w >> 16) & 0xff)) - 1) << ((w >> 8) & 0xff);
  }
  const uint32_t nb = 1u << h;
  if (F32) {
    const float2 A00 = make_float2((float)a00.x, (float)a00.y), A01 = make_float2((float)a01.x, (float)a01.y);
    const float2 A10 = make_float2((float)a10.x, (float)a10.y), A11 = make_float2((float)a11.x, (float)a11.y);
    const float4* st = reinterpret_cast<const float4*>(smem);
    float2* out = reinterpret_cast<float2*>(outp);
    uint64_t ob = 0;
#pragma unroll 4
    for (uint32_t xb = 0; xb < nb; ++xb) {
      const uint32_t sb = xb << (c + 1);
      const float4 b0 = st[(sb | cx0) >> 1], b1 = st[(sb | cx1) >> 1];
      const float4 r0 = f4mac(A00, A01, b0), r1 = f4mac(A10, A11, b1);
      __stcs(reinterpret_cast<float4*>(out + ob), make_float4(r0.x, r0.y, r1.x, r1.y));
      ob = ((ob | ~bmask) + 1) & bmask;
    }
  } else {
    const double2* st = reinterpret_cast<const double2*>(smem);
    double2* out = reinterpret_cast<double2*>(outp);
    uint64_t ob = 0;
#pragma unroll 2
    for (uint32_t xb = 0; xb < nb; ++xb) {
      const uint32_t sb = xb << (c + 1);
      const double2 b00 = st[sb | cx0], b01 = st[sb | cx0 | 1u];
      const double2 b10 = st[sb | cx1], b11 = st[sb | cx1 | 1u];
      const double2 p0 = xcmul(a00, b00), q0 = xcmul(a01, b01);
      const double2 p1 = xcmul(a10, b10), q1 = xcmul(a11, b11);
      __stcs(out + ob, make_double2(p0.x + q0.x, p0.y + q0.y));
      __stcs(out + ob + 1, make_double2(p1.x + q1.x, p1.y + q1.y));
      ob = ((ob | ~bmask) + 1) & bmask;
    }
  }
}

// Persistent: CTA b of grid.x takes a contiguous range of the launch's tiles
// (all items, one set = blockIdx.y), rebuilding the per-item tables only
// when the item changes.
__global__ void __launch_bounds__(256, 5) expand_kernel(const __grid_constant__ XLaunch L) {
  extern __shared__ __align__(16) unsigned char xsmem[];
  __shared__ XItemSmem X;
  __shared__ __align__(16) XDesc SD;
  pdl_trigger();
  pdl_wait();
  const uint64_t per = (L.total_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = min(L.total_tiles, t0 + per);
  const uint32_t set = blockIdx.y, tid = threadIdx.x;
  uint64_t item_end = 0, first = 0;
  const XDesc* d = nullptr;
  const char* in = nullptr;
  char* ws = nullptr;
  uint32_t ea[kXMaxOps + 1], eb[kXMaxOps + 1];  // [kXMaxOps]: x_c of the two outputs
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
      const XDesc* gd = &L.descs[L.item_desc[lo]];
      const uint32_t net = L.item_net[lo];
      in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
      ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
      __syncthreads();  // the previous item's tables and descriptor are no longer read
      // the descriptor into shared memory (one 16-byte load per thread): every
      // run list below is read from there instead of through L1/L2
      for (uint32_t i = tid; i < sizeof(XDesc) / 16; i += 256)
        reinterpret_cast<uint4*>(&SD)[i] = __ldg(reinterpret_cast<const uint4*>(gd) + i);
      __syncthreads();
      d = &SD;
      const uint32_t nA = d->nA, nAB = d->nA + d->nB;
      if (tid < nAB) {
        X.ptr[tid] = xresolve(d->ops[tid].ptr, in, ws);
        X.vs[tid] = d->ops[tid].vshift;
        X.c64[tid] = d->ops[tid].c64;
      }
      for (uint32_t k = nA; k < nAB; ++k) {
        const XOp& op = d->ops[k];
        for (uint32_t i = tid; i < (1u << d->h); i += 256)
          X.tb[k - nA][i] = (uint32_t)xgather(xgather(i, d->brun, d->n_brun), op.runs, op.n_runs);
        for (uint32_t i = tid; i < (1u << d->c); i += 256)
          X.tc[k - nA][i] = (uint32_t)xgather(xgather(i, d->crun, d->n_crun), op.runs, op.n_runs);
      }
      const uint32_t e0 = 2u * tid;
      const uint64_t oe = xgather(e0, d->arun, d->n_arun);
#pragma unroll
      for (uint32_t k = 0; k < kXMaxOps; ++k) {
        ea[k] = 0;
        eb[k] = 0;
        if (k < nA) {
          ea[k] = (uint32_t)xgather(oe, d->ops[k].runs, d->ops[k].n_runs);
          eb[k] = (uint32_t)xgather(1u, d->ops[k].runs, d->ops[k].n_runs);  // output bit 0
        }
      }
      ea[kXMaxOps] = (uint32_t)xgather(e0, d->acrun, d->n_acrun);
      eb[kXMaxOps] = (uint32_t)xgather(e0 + 1u, d->acrun, d->n_acrun);
    } else {
      __syncthreads();  // stage reuse
    }
    const uint64_t obase = xgather(t - first, d->trun, d->n_trun);
    char* outp = const_cast<char*>(xresolve(d->out, in, ws)) +
                 (obase | xgather(2u * tid, d->arun, d->n_arun)) * (d->out_c64 ? 8u : 16u);
    if (d->out_c64)
      expand_tile<true>(*d, X, ea, eb, obase, outp, xsmem);
    else
      expand_tile<false>(*d, X, ea, eb, obase, outp, xsmem);
  }
}

}  // namespace

int launch_expand(const XLaunch& L, void* stream) {
  if (!L.n_items || !L.n_sets || !L.total_tiles) return QTN_OK;
  if (L.n_sets > 65535 || L.total_tiles > 0x7fffffffull) {
    set_error("expand_kernel: grid too large");
    return QTN_EINVAL;
  }
  // dynamic stage (<= kXStageMax complex128 entries) + the static per-item
  // tables exceed the default 48 KiB: opt in once for the largest stage
  static std::atomic<uint64_t> attr{0};
  if (needs_setup(attr)) {
    cudaError_t e = cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kXStageMax * 16);
    if (e != cudaSuccess) {
      set_error(std::string("expand_kernel attribute: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    mark_setup(attr);
  }
  // persistent CTAs (several resident per SM), contiguous tile ranges
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (n_sm <= 0) n_sm = 148;
  }
  // as many resident CTAs per SM as registers and this launch's stage allow
  // (QTN_EXPAND_CTAS: a fixed count per SM, for experiments)
  int per_sm = 0;
  const char* xc = getenv("QTN_EXPAND_CTAS");
  if (xc) per_sm = atoi(xc);
  if (per_sm <= 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, expand_kernel, 256, L.stage_bytes) != cudaSuccess)
    per_sm = 4;
  per_sm = std::max(1, per_sm);
  const uint64_t ctas = std::min<uint64_t>(L.total_tiles, (uint64_t)n_sm * (uint64_t)per_sm);
  dim3 grid((uint32_t)ctas, L.n_sets);
  cudaError_t e = launch_pdl<true>(expand_kernel, grid, dim3(256), L.stage_bytes,
                             reinterpret_cast<cudaStream_t>(stream), L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("expand_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

}  // namespace qtn
