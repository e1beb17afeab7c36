// Weighted full sums (sm_100a): the tail of an elimination order as one pass.
// After the widest buckets the reference's loop (contraction.py:75-106) walks
// a linear chain: each bucket multiplies the previous result by a few
// rank-1/2 gates and sums one more variable (contraction.py:90-96), down to
// the scalar — R launches over tensors of 2^R, 2^(R-1), ... entries.  The
// chain is the single sum
//   Z = sum_x T[x] * prod_k g_k(x[vars_k])
// so T is read once and none of the chain's intermediates exists.
//
// wsum_kernel: a warp per tile of 2^kWsL consecutive entries of T.  Gates on
// tile bits only are folded into a per-CTA lookup table (built level by level
// over the bits: 2^(b+1) entries at bit b), gates on high bits into one
// factor per tile, gates across both are multiplied per entry.  float64 math
// (T is complex64, the gates complex128).  Every CTA writes one partial sum;
// wsum_fin_kernel adds an item's partials in a fixed order (bitwise
// repeatable) and writes the scalar.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

namespace qtn {
namespace {

__device__ __forceinline__ double2 wcmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ const char* wresolve(uint64_t tag, const char* in, char* ws) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return in + off;
  if (sel == 2) return ws + off;
  return reinterpret_cast<const char*>(off);
}
// entry index of gate g at the index x (x: bits of T's index, shifted right by sh)
__device__ __forceinline__ uint32_t gidx(const WsGate& g, uint64_t x, uint32_t sh) {
  const uint32_t a = (uint32_t)(x >> (g.b0 - sh)) & 1u;
  if (g.rank == 1) return a;
  return (a << 1) | ((uint32_t)(x >> (g.b1 - sh)) & 1u);
}

__device__ __forceinline__ uint32_t find_item(const uint32_t* prefix, uint32_t n_items, uint32_t cb) {
  uint32_t lo = 0, hi = n_items;  // last item whose first CTA <= cb
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= cb) lo = mid;
    else hi = mid;
  }
  return lo;
}

// A warp's tiles (R >= kWsL: a tile is 2^kWsL entries = 4 batches of 8 x
// 16-byte loads per lane); v holds the first batch of the first tile.  NST:
// upper bound of the gates across the tile boundary (exact for 0..2).
template <int NST>
__device__ __forceinline__ double2 ws_tiles(const WsDesc& D, const double2 (*gv)[4], const double2* tab,
                                            const float4* src4, float4 (&v)[8], uint64_t h0, uint32_t nw,
                                            uint32_t lane) {
  const uint32_t n_lo = D.n_lo, n_hi = D.n_hi, n_st = D.n_st;
  double2 acc = make_double2(0.0, 0.0);
  for (uint64_t h = h0; h < D.n_tiles; h += nw) {
    double2 hw = make_double2(1.0, 0.0);
    for (uint32_t k = n_lo; k < n_lo + n_hi; ++k) hw = wcmul(hw, gv[k][gidx(D.g[k], h, kWsL)]);
    // gates across the tile boundary: b0 is the tile bit, b1 the high bit
    // (the encoder orders them so); the pair (x[b0] = 0, 1) for this tile
    const double2* sp[NST > 0 ? NST : 1];
    uint32_t sb[NST > 0 ? NST : 1], ss[NST > 0 ? NST : 1];
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      sp[s] = &gv[0][0];
      sb[s] = 0;
      ss[s] = 0;
      if ((uint32_t)s < n_st) {
        const WsGate& g = D.g[n_lo + n_hi + s];
        const uint32_t hb = (uint32_t)(h >> (g.b1 - kWsL)) & 1u;
        // pad = 1: the tile bit is the entry index's high bit (entry = t << 1 | hb), else entry = hb << 1 | t
        sp[s] = &gv[n_lo + n_hi + s][g.pad ? hb : (hb << 1)];
        ss[s] = g.pad ? 2u : 1u;
        sb[s] = g.b0;
      }
    }
    double2 ts = make_double2(0.0, 0.0);
    const float4* t4 = src4 + (h << (kWsL - 1)) + lane;
#pragma unroll 1
    for (uint32_t bt = 0; bt < (1u << kWsL) / 512u; ++bt) {
      if (bt != 0 || h != h0) {
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) v[q] = __ldg(t4 + 256u * bt + 32u * q);
      }
#pragma unroll
      for (uint32_t q = 0; q < 8; ++q) {
        const uint32_t e = 2u * lane + 64u * q + 512u * bt;
        double2 w0 = tab[e], w1 = tab[e + 1];
#pragma unroll
        for (int s = 0; s < NST; ++s)
          if (NST <= 2 || (uint32_t)s < n_st) {
            w0 = wcmul(w0, sp[s][((e >> sb[s]) & 1u) * ss[s]]);
            w1 = wcmul(w1, sp[s][(((e + 1u) >> sb[s]) & 1u) * ss[s]]);
          }
        ts.x = fma((double)v[q].x, w0.x, fma(-(double)v[q].y, w0.y, ts.x));
        ts.y = fma((double)v[q].x, w0.y, fma((double)v[q].y, w0.x, ts.y));
        ts.x = fma((double)v[q].z, w1.x, fma(-(double)v[q].w, w1.y, ts.x));
        ts.y = fma((double)v[q].z, w1.y, fma((double)v[q].w, w1.x, ts.y));
      }
    }
    const double2 t = wcmul(hw, ts);
    acc.x += t.x;
    acc.y += t.y;
  }
  return acc;
}

__global__ void __launch_bounds__(256, 3) wsum_kernel(const __grid_constant__ WsLaunch L) {
  __shared__ __align__(16) WsDesc D;
  __shared__ double2 gv[kWsMaxGates][4];
  __shared__ double2 tab[1 << kWsL];
  __shared__ double2 wpart[8];
  pdl_trigger();
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t item = find_item(L.cta_prefix, L.n_items, blockIdx.x);
  const uint32_t c = blockIdx.x - L.cta_prefix[item];
  const WsDesc* gd = L.descs + L.item_desc[item];
  for (uint32_t i = tid; i < sizeof(WsDesc) / 16; i += 256)
    reinterpret_cast<uint4*>(&D)[i] = __ldg(reinterpret_cast<const uint4*>(gd) + i);
  const uint32_t net = L.item_net[item], set = blockIdx.y;
  const char* in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
  char* ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
  __syncthreads();
  pdl_wait();  // the gates (tensorgen) and T are written by earlier launches
  const uint32_t n_lo = D.n_lo, n_hi = D.n_hi, n_st = D.n_st, n_g = n_lo + n_hi + n_st;
  // the first batch of this warp's first tile is in flight during the table build
  const float4* src4 = reinterpret_cast<const float4*>(wresolve(D.src, in, ws));
  const uint32_t nw = D.n_ctas * 8u;
  const uint64_t h0 = (uint64_t)c * 8u + warp;
  float4 v[8];
  if (h0 < D.n_tiles) {
#pragma unroll
    for (uint32_t q = 0; q < 8; ++q) v[q] = __ldg(src4 + (h0 << (kWsL - 1)) + lane + 32u * q);
  }
  for (uint32_t i = tid; i < 4u * n_g; i += 256) {
    const WsGate& g = D.g[i >> 2];
    const uint32_t e = i & 3u;
    double2 v = make_double2(0.0, 0.0);
    if (e < (1u << g.rank)) {
      const char* p = wresolve(g.ptr, in, ws);
      if (g.c64) {
        const float2 f = __ldg(reinterpret_cast<const float2*>(p) + e);
        v = make_double2(f.x, f.y);
      } else {
        v = __ldg(reinterpret_cast<const double2*>(p) + e);
      }
    }
    gv[i >> 2][e] = v;
  }
  __syncthreads();
  // table over the tile bits: entry x = tid + 256 q is the product of the lo
  // gates at x; a gate on bits < 8 only has one value per thread
  {
    double2 wt = make_double2(1.0, 0.0);
    for (uint32_t k = 0; k < n_lo; ++k) {
      const WsGate g = D.g[k];
      const uint32_t top = g.rank == 2 ? max((uint32_t)g.b0, (uint32_t)g.b1) : (uint32_t)g.b0;
      if (top < 8u) wt = wcmul(wt, gv[k][gidx(g, tid, 0)]);
    }
#pragma unroll 1
    for (uint32_t q0 = 0; q0 < (1u << kWsL) / 256u; q0 += 4) {
      double2 wq[4];
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) wq[q] = wt;
      for (uint32_t k = 0; k < n_lo; ++k) {
        const WsGate g = D.g[k];
        const uint32_t top = g.rank == 2 ? max((uint32_t)g.b0, (uint32_t)g.b1) : (uint32_t)g.b0;
        if (top >= 8u) {
#pragma unroll
          for (uint32_t q = 0; q < 4; ++q) wq[q] = wcmul(wq[q], gv[k][gidx(g, tid + 256u * (q0 + q), 0)]);
        }
      }
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) tab[tid + 256u * (q0 + q)] = wq[q];
    }
  }
  __syncthreads();
  // tiles: warp wi of the item's n_ctas * 8 takes tiles wi, wi + nw, ...
  double2 acc;
  if (n_st == 0) acc = ws_tiles<0>(D, gv, tab, src4, v, h0, nw, lane);
  else if (n_st == 1) acc = ws_tiles<1>(D, gv, tab, src4, v, h0, nw, lane);
  else if (n_st == 2) acc = ws_tiles<2>(D, gv, tab, src4, v, h0, nw, lane);
  else acc = ws_tiles<kWsMaxSt>(D, gv, tab, src4, v, h0, nw, lane);
#pragma unroll
  for (uint32_t m = 16; m >= 1; m >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, m);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, m);
  }
  if (lane == 0) wpart[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double2 z = wpart[0];
#pragma unroll
    for (uint32_t w = 1; w < 8; ++w) {
      z.x += wpart[w].x;
      z.y += wpart[w].y;
    }
    reinterpret_cast<double2*>(const_cast<char*>(wresolve(D.part, in, ws)))[c] = z;
  }
}

// one warp per item: the CTA partials in a fixed order -> the scalar
__global__ void __launch_bounds__(32) wsum_fin_kernel(const __grid_constant__ WsLaunch L) {
  pdl_trigger();
  const uint32_t item = blockIdx.x, lane = threadIdx.x;
  const WsDesc* d = L.descs + L.item_desc[item];
  const uint32_t net = L.item_net[item], set = blockIdx.y;
  const char* in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
  char* ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
  const uint32_t n = d->n_ctas;
  const uint64_t part = d->part, outt = d->out;
  const uint32_t oc64 = d->out_c64;
  pdl_wait();
  const double2* p = reinterpret_cast<const double2*>(wresolve(part, in, ws));
  double2 z = make_double2(0.0, 0.0);
  for (uint32_t i = lane; i < n; i += 32) {
    const double2 v = __ldcg(p + i);
    z.x += v.x;
    z.y += v.y;
  }
#pragma unroll
  for (uint32_t m = 16; m >= 1; m >>= 1) {
    z.x += __shfl_xor_sync(0xffffffffu, z.x, m);
    z.y += __shfl_xor_sync(0xffffffffu, z.y, m);
  }
  if (lane == 0) {
    char* o = const_cast<char*>(wresolve(outt, in, ws));
    if (oc64) *reinterpret_cast<float2*>(o) = make_float2((float)z.x, (float)z.y);
    else *reinterpret_cast<double2*>(o) = z;
  }
}

}  // namespace

bool encode_wsum_desc(const WsSpec& s, WsDesc& d) {
  const int R = (int)s.src_vars.size();
  if (R < kWsL || R > 40 || s.gate_vars.size() > (size_t)kWsMaxGates) return false;
  std::memset(&d, 0, sizeof(d));
  auto bit_of = [&](int32_t u) -> int {
    for (int i = 0; i < R; ++i)
      if (s.src_vars[i] == u) return R - 1 - i;
    return -1;
  };
  const int Lb = std::min(R, kWsL);
  struct G {
    WsGate g;
    int hi;  // highest bit
  };
  std::vector<G> lo, hi, st;
  for (size_t k = 0; k < s.gate_vars.size(); ++k) {
    const auto& gvars = s.gate_vars[k];
    if (gvars.empty() || gvars.size() > 2) return false;
    WsGate g{};
    g.ptr = s.gate_tag[k];
    g.rank = (uint8_t)gvars.size();
    g.c64 = s.gate_c64[k];
    const int b0 = bit_of(gvars[0]), b1 = g.rank == 2 ? bit_of(gvars[1]) : -1;
    if (b0 < 0 || (g.rank == 2 && (b1 < 0 || b1 == b0))) return false;
    g.b0 = (uint8_t)b0;
    g.b1 = (uint8_t)(g.rank == 2 ? b1 : 0);
    const int top = std::max(b0, b1), bot = g.rank == 2 ? std::min(b0, b1) : b0;
    if (top < Lb) lo.push_back({g, top});
    else if (bot >= Lb) hi.push_back({g, top});
    else {
      // across: b0 := the tile bit, b1 := the high bit; pad = 1 when the
      // tile bit is the entry index's high bit (variable 0)
      g.pad = b0 < Lb ? 1u : 0u;
      g.b0 = (uint8_t)bot;
      g.b1 = (uint8_t)top;
      st.push_back({g, top});
    }
  }
  if (st.size() > (size_t)kWsMaxSt) return false;
  std::stable_sort(lo.begin(), lo.end(), [](const G& a, const G& b) { return a.hi < b.hi; });
  size_t q = 0;
  for (int b = 0; b <= kWsL; ++b) {
    while (q < lo.size() && lo[q].hi < b) ++q;
    d.lo_first[b] = (uint8_t)q;
  }
  size_t k = 0;
  for (auto& x : lo) d.g[k++] = x.g;
  for (auto& x : hi) d.g[k++] = x.g;
  for (auto& x : st) d.g[k++] = x.g;
  d.n_lo = (uint8_t)lo.size();
  d.n_hi = (uint8_t)hi.size();
  d.n_st = (uint8_t)st.size();
  d.R = (uint8_t)R;
  d.out_c64 = s.out_c64 ? 1 : 0;
  d.src = s.src_tag;
  d.out = s.out_tag;
  d.n_tiles = 1ull << (R - Lb);
  d.n_ctas = (uint32_t)std::min<uint64_t>((d.n_tiles + 7) / 8, (uint64_t)kWsMaxCtas);
  return true;
}

int launch_wsum(const WsLaunch& L, void* stream) {
  if (!L.n_items || !L.n_sets || !L.total_ctas) return QTN_OK;
  if (L.n_sets > 65535) {
    set_error("wsum_kernel: grid too large");
    return QTN_EINVAL;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = launch_pdl<true>(wsum_kernel, dim3(L.total_ctas, L.n_sets), dim3(256), 0, st, L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess)
    e = launch_pdl_if<true>(true, wsum_fin_kernel, dim3(L.n_items, L.n_sets), dim3(32), 0, st, L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("wsum_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

}  // namespace qtn
