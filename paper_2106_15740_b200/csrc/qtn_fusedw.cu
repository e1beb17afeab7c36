// Warp-granular fused product chains (sm_100a), qtn_stream.h WHdr/WOpRec.
//
// The contraction of a product bucket and the partial traces of its result
// (contraction.py:42-54 `_product` chain, then k+1 times the `.sum` of
// :94-96) as one sum over the chain's summed variables:
//   out[o] = sum_{s in 2^K} prod_t T_t[idx_t(o, s)]
// evaluated by one warp per 32 * NI outputs.  Lanes take output bits 0..4
// (coalesced stores), each lane accumulates NI outputs (in-lane slots over
// 3 more output bits, chosen by the host among the bits the widest operand
// does not depend on, so that operand is loaded once per s for all slots).
// Every index map is OR-linear over disjoint bits, so an operand index is
//   chunk_t(chunk) + lane_t[lane] + slot_t[i] + hs_t[s]
// with the lane / slot / summed tables built on the host.  Operand entries
// are read straight from L1/L2 (chain operands are small and were written by
// the previous level); nothing is staged, so a warp's setup is a handful of
// loads instead of the CTA kernel's descriptor/table copies and cp.async
// stages.  Products in float when the chain's head product is a complex64
// intermediate (the unfused buckets' storage policy), partial sums of 8
// terms in that type, accumulated across blocks in double.
#include <cuda_runtime.h>

#include <string>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

namespace qtn {
namespace {

template <typename C> struct WE;
template <> struct WE<float2> { using T = float; };
template <> struct WE<double2> { using T = double; };

__device__ __forceinline__ float2 wcm(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 wcm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a * b
__device__ __forceinline__ float2 wcfma(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, fmaf(-a.y, b.y, c.x)), fmaf(a.x, b.y, fmaf(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 wcfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}

__device__ __forceinline__ uint64_t wgather(uint64_t x, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = __ldg(runs + r);
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((x >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}
__device__ __forceinline__ const char* wresolve(uint64_t tag, const char* in, char* ws) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return in + off;
  if (sel == 2) return ws + off;
  return reinterpret_cast<const char*>(off);
}
// operand entry in the math type; MATCH: stored in the math type
template <typename C, bool MATCH>
__device__ __forceinline__ C wld(const char* p, uint32_t i, bool c64) {
  using E = typename WE<C>::T;
  if (MATCH) return __ldg(reinterpret_cast<const C*>(p) + i);
  if (c64) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return C{(E)f.x, (E)f.y};
  }
  const double2 d = __ldg(reinterpret_cast<const double2*>(p) + i);
  return C{(E)d.x, (E)d.y};
}

// One operand's factor of the NI terms of summed value s: FIRST starts the
// products, LAST multiplies into the partial sums, else multiplies in.
template <typename C, int NI, bool MATCH, int MODE>  // MODE 0 first, 1 middle, 2 last
__device__ __forceinline__ void wfactor(const char* p, uint32_t h, const uint32_t (&sl)[NI], bool inv,
                                        bool c64, C (&pr)[NI], C (&part)[NI]) {
  if (inv) {
    const C v = wld<C, MATCH>(p, h, c64);
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (MODE == 0) pr[i] = v;
      else if (MODE == 1) pr[i] = wcm(pr[i], v);
      else part[i] = wcfma(pr[i], v, part[i]);
    }
  } else {
    C v[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) v[i] = wld<C, MATCH>(p, h + sl[i], c64);
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (MODE == 0) pr[i] = v[i];
      else if (MODE == 1) pr[i] = wcm(pr[i], v[i]);
      else part[i] = wcfma(pr[i], v[i], part[i]);
    }
  }
}

template <typename C, int NI, bool MATCH>
__device__ __forceinline__ void wbody(const uint8_t* blob, const char* in, char* ws, uint32_t chunk,
                                      uint32_t lane) {
  const WHdr* hp = reinterpret_cast<const WHdr*>(blob);
  const WOpRec* ops = reinterpret_cast<const WOpRec*>(blob + sizeof(WHdr));
  const uint32_t* tw = reinterpret_cast<const uint32_t*>(blob);
  const uint32_t n = hp->n_ops, K = hp->K;
  const char* p[kWMaxOps];
  uint32_t base[kWMaxOps];
  uint32_t sl[kWMaxOps][NI];
  const uint32_t* hs[kWMaxOps];
  bool inv[kWMaxOps], c64[kWMaxOps];
#pragma unroll
  for (int t = 0; t < kWMaxOps; ++t) {
    p[t] = nullptr;
    base[t] = 0;
    hs[t] = tw;
    inv[t] = true;
    c64[t] = true;
#pragma unroll
    for (int i = 0; i < NI; ++i) sl[t][i] = 0;
    if ((uint32_t)t < n) {
      const WOpRec& o = ops[t];
      p[t] = wresolve(o.ptr, in, ws);
      base[t] = (uint32_t)wgather(chunk, o.crun, o.n_crun) + __ldg(tw + o.lane_off + lane);
      inv[t] = o.inv != 0;
      c64[t] = o.c64 != 0;
      if (!inv[t]) {
#pragma unroll
        for (int i = 0; i < NI; ++i) sl[t][i] = __ldg(tw + o.slot_off + i);
      }
      hs[t] = tw + o.hs_off;
    }
  }
  double2 acc[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) acc[i] = make_double2(0.0, 0.0);
  const uint32_t ns = 1u << K, blk = ns < 8u ? ns : 8u;
  for (uint32_t s0 = 0; s0 < ns; s0 += blk) {
    C part[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) part[i] = C{0, 0};
#pragma unroll 2
    for (uint32_t s = s0; s < s0 + blk; ++s) {
      C pr[NI];
      wfactor<C, NI, MATCH, 0>(p[0], base[0] + __ldg(hs[0] + s), sl[0], inv[0], c64[0], pr, part);
      if (n == 2) {
        wfactor<C, NI, MATCH, 2>(p[1], base[1] + __ldg(hs[1] + s), sl[1], inv[1], c64[1], pr, part);
      } else if (n == 3) {
        wfactor<C, NI, MATCH, 1>(p[1], base[1] + __ldg(hs[1] + s), sl[1], inv[1], c64[1], pr, part);
        wfactor<C, NI, MATCH, 2>(p[2], base[2] + __ldg(hs[2] + s), sl[2], inv[2], c64[2], pr, part);
      } else {
        wfactor<C, NI, MATCH, 1>(p[1], base[1] + __ldg(hs[1] + s), sl[1], inv[1], c64[1], pr, part);
        wfactor<C, NI, MATCH, 1>(p[2], base[2] + __ldg(hs[2] + s), sl[2], inv[2], c64[2], pr, part);
        wfactor<C, NI, MATCH, 2>(p[3], base[3] + __ldg(hs[3] + s), sl[3], inv[3], c64[3], pr, part);
      }
    }
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      acc[i].x += (double)part[i].x;
      acc[i].y += (double)part[i].y;
    }
  }
  char* outp = const_cast<char*>(wresolve(hp->out, in, ws));
  const uint64_t ob = wgather(chunk, hp->ocrun, hp->n_ocrun) + lane;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const uint64_t o = ob + (NI > 1 ? __ldg(&hp->slot_out[i]) : 0u);
    if (hp->out_c64)
      reinterpret_cast<float2*>(outp)[o] = make_float2((float)acc[i].x, (float)acc[i].y);
    else
      reinterpret_cast<double2*>(outp)[o] = acc[i];
  }
}

template <typename C>
__global__ void __launch_bounds__(256, 2) fusedw_kernel(const __grid_constant__ WLaunch L) {
  pdl_trigger();
  const uint32_t w = blockIdx.x * 8u + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
  if (w >= L.n_warps) return;
  const WRec r = L.recs[w];
  const uint8_t* blob = L.blob + 16ull * r.blob16;
  const char* in = L.in_base + (int64_t)blockIdx.y * L.in_set_stride + L.net_in_off[r.net];
  char* ws = L.ws_base + (int64_t)blockIdx.y * L.ws_set_stride + L.net_ws_off[r.net];
  const WHdr* hp = reinterpret_cast<const WHdr*>(blob);
  const bool ni4 = hp->ni_log2 == 2, match = hp->match != 0;
  pdl_wait();
  if (ni4) {
    if (match) wbody<C, 4, true>(blob, in, ws, r.chunk, lane);
    else wbody<C, 4, false>(blob, in, ws, r.chunk, lane);
  } else {
    if (match) wbody<C, 1, true>(blob, in, ws, r.chunk, lane);
    else wbody<C, 1, false>(blob, in, ws, r.chunk, lane);
  }
}

}  // namespace

int launch_fusedw(const WLaunch& L, void* stream) {
  if (!L.n_warps || !L.n_sets) return QTN_OK;
  if (L.n_sets > 65535) {
    set_error("fusedw_kernel: grid too large");
    return QTN_EINVAL;
  }
  const dim3 grid((L.n_warps + 7u) / 8u, L.n_sets);
  cudaError_t e = L.f64 ? launch_pdl<true>(fusedw_kernel<double2>, grid, dim3(256), 0,
                                           reinterpret_cast<cudaStream_t>(stream), L)
                        : launch_pdl<true>(fusedw_kernel<float2>, grid, dim3(256), 0,
                                           reinterpret_cast<cudaStream_t>(stream), L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("fusedw_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

}  // namespace qtn
