// Tile pipeline of the streaming bucket kernel (sm_100a), compiled once per
// consumer-thread count: qtn_stream.cu (256 consumers, namespace s256) and
// qtn_stream512.cu (512 consumers, namespace s512).  See qtn_stream.cu for
// the design.  Included, not compiled on its own.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

#ifndef QTN_STREAM_NS
#error "define QTN_STREAM_NS before including qtn_stream_tile.cuh"
#endif

namespace qtn {
namespace QTN_STREAM_NS {


#ifndef QTN_STREAM_COMPUTE
#define QTN_STREAM_COMPUTE 256
#endif
constexpr int kCompute = QTN_STREAM_COMPUTE;  // 8 consumer warps (9 warps/block
                                            // leave 168 registers per thread)
constexpr int kWarps = kCompute / 32;
constexpr bool kPrecomp = kCompute <= 256;
constexpr int kThreads = kCompute + 32;     // + 1 producer warp
constexpr int kStages = kStreamStages;
constexpr int kChunkBytes = kStreamChunk;     // primary slice per stage
constexpr int kJ = (1 << kTileBitsC64) / kCompute;  // elements per consumer thread per tile
constexpr int kTabEntries = kSMaxT * 512;    // complex128 entries
constexpr int kDescSlot = (kSDescMax + 127) / 128 * 128;

struct __align__(128) Smem {
  uint8_t chunk[kStages][kChunkBytes];
  uint8_t desc[kStages][kDescSlot];
  double2 tab[kTabEntries];   // lookup tables (complex64 in the F32 fast path)
  double2 gslice[kStages][2 << kStageMaxK];  // staged tile slice of gathered operand 0
                                             // (raw complex64 or complex128 entries)
  uint64_t gjj[kSMaxG][kJ];   // thread-independent gather parts (per descriptor)
  uint32_t tjj[kSMaxT][kJ];
  uint32_t tjs[kJ];           // ... of the staged slice index
  __align__(16) uint8_t pdesc[sizeof(SHdr) + sizeof(SGRec)];  // producer's descriptor cache
  uint64_t full[kStages];
  uint64_t empty[kStages];
};

struct InlineDesc {
  uint8_t bytes[kDescSlot];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async(void* dst, const void* src, uint32_t bytes) {
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
// consumer-warps-only barrier (the producer warp never joins)
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 ldg_c(const void* p, uint64_t i, uint32_t c64) {
  if (c64) {
    float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return make_double2(f.x, f.y);
  }
  return __ldg(reinterpret_cast<const double2*>(p) + i);
}
__device__ __forceinline__ uint64_t gather(uint64_t o, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((o >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}

struct Bases {
  const char* in;
  char* ws;
  char* sm = nullptr;  // shared memory of a tiny-subtree CTA (tag selector 3)
};

__device__ __forceinline__ const char* resolve(uint64_t tag, const Bases& b) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return b.in + off;
  if (sel == 2) return b.ws + off;
  if (sel == 3) return b.sm + off;
  return reinterpret_cast<const char*>(off);
}

struct Loc {
  uint32_t item, set;
  uint64_t tile;
};

// Output base of a tile: the tile index enumerates the output bits that are
// not tile-local (primary bits [ta, rP-1), then new bits [rP-1+tn, R)).
__device__ __forceinline__ uint64_t tile_base(const SHdr& h, uint64_t t) {
  const uint32_t r1 = h.p_rank - 1u, a = h.ta;
  const uint64_t low = t & ((1ull << (r1 - a)) - 1);
  return (low << a) | ((t >> (r1 - a)) << (r1 + h.tn));
}
// Tile-local element e -> output offset within the tile.
__device__ __forceinline__ uint64_t tile_off(uint32_t e, uint32_t a, uint32_t r1) {
  return (uint64_t)(e & ((1u << a) - 1u)) | ((uint64_t)(e >> a) << r1);
}

// Cached item range of the last lookup (tiles of one block are contiguous,
// so consecutive tiles almost always hit the same item).
struct LocCache {
  uint32_t item = 0;
  uint64_t lo = 1, hi = 0;  // empty
  uint32_t set = 0;
  uint64_t set_lo = 1, set_hi = 0;  // tile range of the cached set (no 64-bit divide per tile)
};

__device__ __forceinline__ Loc locate(const StreamLaunch& L, uint64_t t, LocCache& c) {
  Loc r;
  if (!L.item_desc) {
    r.item = 0;
    r.set = 0;
    r.tile = t;
    return r;
  }
  if (!(t >= c.set_lo && t < c.set_hi)) {
    c.set = (uint32_t)(t / L.total_tiles);
    c.set_lo = (uint64_t)c.set * L.total_tiles;
    c.set_hi = c.set_lo + L.total_tiles;
  }
  r.set = c.set;
  const uint64_t tt = t - c.set_lo;
  if (!(tt >= c.lo && tt < c.hi)) {
    uint32_t it = c.item < L.n_items ? c.item : 0;
    if (L.tile_prefix[it] > tt) it = 0;
    if (L.tile_prefix[it + 1] <= tt) {
      uint32_t lo = it, hi = L.n_items;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (L.tile_prefix[mid] <= tt) lo = mid;
        else hi = mid;
      }
      it = lo;
    }
    c.item = it;
    c.lo = L.tile_prefix[it];
    c.hi = L.tile_prefix[it + 1];
  }
  r.item = c.item;
  r.tile = tt - c.lo;
  return r;
}

__device__ __forceinline__ Bases bases_of(const StreamLaunch& L, const Loc& l) {
  Bases b{nullptr, nullptr, nullptr};
  if (!L.item_desc) return b;
  const uint32_t net = L.item_net[l.item];
  b.in = L.in_base + (int64_t)l.set * L.in_set_stride + L.net_in_off[net];
  b.ws = L.ws_base + (int64_t)l.set * L.ws_set_stride + L.net_ws_off[net];
  return b;
}

// Producer: the primary slice of one tile (+ the descriptor in work-list
// mode) into stage `s`, completing on full[s].
__device__ void issue_tile(const StreamLaunch& L, const uint8_t* dsc, const SHdr& h, Smem& S,
                           const Loc& l, int s) {
  const Bases b = bases_of(L, l);
  const uint32_t esz = h.p_c64 ? 8u : 16u;
  const uint32_t tb = h.tb;
  const uint32_t ptb = h.ta;
  const uint64_t op = tile_base(h, l.tile) & ((1ull << (h.p_rank - 1)) - 1);
  const uint64_t pidx = (op & ((1ull << h.p_k) - 1)) | ((op >> h.p_k) << (h.p_k + 1));
  const char* P = resolve(h.p, b);
  const bool split = ptb >= 1 && h.p_k >= ptb;
  const uint32_t dbytes = L.item_desc ? h.desc_bytes : 0u;
  const uint32_t cbytes = (2u << ptb) * esz;
  uint64_t* bar = &S.full[s];
  mbar_expect_tx(bar, cbytes + dbytes);
  if (dbytes) bulk_g2s(S.desc[s], dsc, dbytes, bar);
  if (split) {
    const uint32_t half = cbytes / 2;
    const char* a = P + pidx * esz;
    const char* c = P + (pidx + (1ull << h.p_k)) * esz;
    for (uint32_t o = 0; o < half; o += 8192) {
      const uint32_t n = min(8192u, half - o);
      bulk_g2s(S.chunk[s] + o, a + o, n, bar);
      bulk_g2s(S.chunk[s] + half + o, c + o, n, bar);
    }
  } else {
    const char* a = P + pidx * esz;
    for (uint32_t o = 0; o < cbytes; o += 8192)
      bulk_g2s(S.chunk[s] + o, a + o, min(8192u, cbytes - o), bar);
  }
}

// Per-thread state valid for one (descriptor, network, set).
struct ThreadState {
  uint32_t tt[kSMaxT];                // table index bits from this thread's lane part
  uint32_t toff[kSMaxT];
  uint64_t gt[kSMaxG];                // gathered-operand index, lane part
  const char* gptr[kSMaxG];
  uint32_t gvs[kSMaxG], gc64[kSMaxG];
  char* out;
  uint32_t ng, nt, tile_elems, tb, pmask, pk, split, pstep;
  uint32_t ts;                        // staged slice index, lane part
  uint32_t ta, r1;                    // tile-local primary bits, primary rank - 1
  uint32_t stage_k;                   // 0xff: operand 0 not staged
  // per element j: primary index (v = 0) in the chunk and output offset in
  // the tile, precomputed per descriptor (256-consumer build; the
  // 512-consumer build recomputes them to stay within 96 registers)
  uint32_t pi0[kPrecomp ? kJ : 1];
  uint64_t ooff[kPrecomp ? kJ : 1];
};

// Generic tile: any dtypes, any operand counts, partial tiles.  Inlined
// with constant-index (guarded, unrolled) operand loops so ThreadState stays
// in registers.
__device__ __forceinline__ void tile_generic(const ThreadState& T, const uint8_t* chunk,
                                             const Smem& S, const SGRec* gr, const STRec* tr,
                                             uint64_t obase, uint32_t tid, uint32_t pc64,
                                             uint32_t oc64) {
#pragma unroll 1
  for (uint32_t e = tid; e < T.tile_elems; e += kCompute) {
    const uint32_t j = e / kCompute;
    const uint32_t pe = e & T.pmask;
    const uint32_t i0 = T.split ? pe : ((pe & ((1u << T.pk) - 1u)) | ((pe >> T.pk) << (T.pk + 1)));
    const uint32_t i1 = i0 + T.pstep;
    double2 a0, a1;
    if (pc64) {
      const float2 x = reinterpret_cast<const float2*>(chunk)[i0];
      const float2 y = reinterpret_cast<const float2*>(chunk)[i1];
      a0 = make_double2(x.x, x.y);
      a1 = make_double2(y.x, y.y);
    } else {
      a0 = reinterpret_cast<const double2*>(chunk)[i0];
      a1 = reinterpret_cast<const double2*>(chunk)[i1];
    }
#pragma unroll
    for (int q = 0; q < kSMaxT; ++q) {
      if (q < (int)T.nt) {
        const uint32_t ti = (uint32_t)gather(obase, tr[q].runs, tr[q].n_runs) | T.tt[q] | S.tjj[q][j];
        const double2* tp = S.tab + tr[q].smem_off + (ti << 1);
        a0 = cmul(a0, tp[0]);
        a1 = cmul(a1, tp[1]);
      }
    }
#pragma unroll
    for (int g = 0; g < kSMaxG; ++g) {
      if (g < (int)T.ng) {
        const uint64_t idx = gather(obase, gr[g].runs, gr[g].n_runs) | T.gt[g] | S.gjj[g][j];
        const uint32_t gc = gr[g].c64, vs = gr[g].vshift;
        a0 = cmul(a0, ldg_c(T.gptr[g], idx, gc));
        a1 = cmul(a1, ldg_c(T.gptr[g], idx + (1ull << vs), gc));
      }
    }
    const double2 r = make_double2(a0.x + a1.x, a0.y + a1.y);
    if (oc64)
      reinterpret_cast<float2*>(T.out)[obase + tile_off(e, T.ta, T.r1)] = make_float2((float)r.x, (float)r.y);
    else
      reinterpret_cast<double2*>(T.out)[obase + tile_off(e, T.ta, T.r1)] = r;
  }
}

__device__ __forceinline__ float2 cmulf(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}

// Full tile, operand counts known at compile time.  F32: complex64 primary
// and output, float32 arithmetic with complex64 lookup tables (the tables
// themselves are products formed in float64); otherwise complex128 / float64.
template <bool F32, int NT, int NG, bool STAGED = false>
__device__ __forceinline__ void tile_fast(const ThreadState& T, const uint8_t* chunk, Smem& S,
                                          const SGRec* gr, const STRec* tr, uint64_t obase,
                                          uint32_t tid, const double2* gsl) {
  // STAGED: the producer warp already gathered the 2^(k+1) entries of
  // operand 0 this tile touches into gsl (raw storage type)
  uint64_t gb[NG > 0 ? NG : 1];
  uint32_t tbs[NT > 0 ? NT : 1];
#pragma unroll
  for (int g = 0; g < NG; ++g) gb[g] = gather(obase, gr[g].runs, gr[g].n_runs) | T.gt[g];
#pragma unroll
  for (int q = 0; q < NT; ++q)
    tbs[q] = (uint32_t)gather(obase, tr[q].runs, tr[q].n_runs) | T.tt[q];
#pragma unroll
  for (int j = 0; j < kJ; ++j) {
    uint32_t i0;
    uint64_t oo;
    if constexpr (kPrecomp) {
      i0 = T.pi0[j];
      oo = T.ooff[j];
    } else {
      const uint32_t e = tid + (uint32_t)j * kCompute;
      const uint32_t pe = e & T.pmask;
      i0 = T.split ? pe : ((pe & ((1u << T.pk) - 1u)) | ((pe >> T.pk) << (T.pk + 1)));
      oo = tile_off(e, T.ta, T.r1);
    }
    const uint32_t i1 = i0 + T.pstep;
    if constexpr (F32) {
      float2 a0 = reinterpret_cast<const float2*>(chunk)[i0];
      float2 a1 = reinterpret_cast<const float2*>(chunk)[i1];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const float4 tv = *reinterpret_cast<const float4*>(
            reinterpret_cast<const float2*>(S.tab) + T.toff[q] + ((tbs[q] | S.tjj[q][j]) << 1));
        a0 = cmulf(a0, make_float2(tv.x, tv.y));
        a1 = cmulf(a1, make_float2(tv.z, tv.w));
      }
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        float2 x, y;
        if (STAGED && g == 0) {
          const uint32_t si = (T.ts | S.tjs[j]) << 1;
          if (T.gc64[0]) {
            x = reinterpret_cast<const float2*>(gsl)[si];
            y = reinterpret_cast<const float2*>(gsl)[si + 1];
          } else {
            x = make_float2((float)gsl[si].x, (float)gsl[si].y);
            y = make_float2((float)gsl[si + 1].x, (float)gsl[si + 1].y);
          }
        } else {
          const uint64_t idx = gb[g] | S.gjj[g][j];
          if (T.gc64[g]) {
            x = __ldg(reinterpret_cast<const float2*>(T.gptr[g]) + idx);
            y = __ldg(reinterpret_cast<const float2*>(T.gptr[g]) + idx + (1ull << T.gvs[g]));
          } else {
            const double2 xd = ldg_c(T.gptr[g], idx, 0);
            const double2 yd = ldg_c(T.gptr[g], idx + (1ull << T.gvs[g]), 0);
            x = make_float2((float)xd.x, (float)xd.y);
            y = make_float2((float)yd.x, (float)yd.y);
          }
        }
        a0 = cmulf(a0, x);
        a1 = cmulf(a1, y);
      }
      reinterpret_cast<float2*>(T.out)[obase + oo] = make_float2(a0.x + a1.x, a0.y + a1.y);
    } else {
      double2 a0 = reinterpret_cast<const double2*>(chunk)[i0];
      double2 a1 = reinterpret_cast<const double2*>(chunk)[i1];
#pragma unroll
      for (int q = 0; q < NT; ++q) {
        const double2* tp = S.tab + T.toff[q] + ((tbs[q] | S.tjj[q][j]) << 1);
        a0 = cmul(a0, tp[0]);
        a1 = cmul(a1, tp[1]);
      }
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        if (STAGED && g == 0) {
          const uint32_t si = (T.ts | S.tjs[j]) << 1;
          double2 x, y;
          if (T.gc64[0]) {
            const float2 xf = reinterpret_cast<const float2*>(gsl)[si];
            const float2 yf = reinterpret_cast<const float2*>(gsl)[si + 1];
            x = make_double2(xf.x, xf.y);
            y = make_double2(yf.x, yf.y);
          } else {
            x = gsl[si];
            y = gsl[si + 1];
          }
          a0 = cmul(a0, x);
          a1 = cmul(a1, y);
        } else {
          const uint64_t idx = gb[g] | S.gjj[g][j];
          a0 = cmul(a0, ldg_c(T.gptr[g], idx, T.gc64[g]));
          a1 = cmul(a1, ldg_c(T.gptr[g], idx + (1ull << T.gvs[g]), T.gc64[g]));
        }
      }
      reinterpret_cast<double2*>(T.out)[obase + oo] = make_double2(a0.x + a1.x, a0.y + a1.y);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    stream_kernel(const __grid_constant__ StreamLaunch L, const __grid_constant__ InlineDesc D) {
  extern __shared__ __align__(128) uint8_t smraw[];
  Smem& S = *reinterpret_cast<Smem*>(smraw);
  const uint32_t tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();  // operands written by the previous level
  uint64_t total;
  if (L.item_desc) total = L.total_tiles * L.n_sets;
  else total = reinterpret_cast<const SHdr*>(D.bytes)->n_tiles;
  const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * per;
  const uint64_t t1 = min(total, t0 + per);
  if (t0 >= t1) return;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1 + 32);
      mbar_init(&S.empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid >= kCompute) {
    // ---------------- producer warp
    // lane 0 issues the bulk copies; all 32 lanes gather the staged slice
    // of gathered operand 0 with cp.async and arrive on full[s] when their
    // copies land (full[s] expects 1 + 32 arrivals per phase)
    const uint32_t lane = tid & 31;
    LocCache lc;
    uint32_t pitem = 0xffffffffu;
    const uint8_t* dsc = D.bytes;
    uint64_t i = 0;
    for (uint64_t t = t0; t < t1; ++t, ++i) {
      const int s = (int)(i % kStages);
      if (i >= (uint64_t)kStages) mbar_wait(&S.empty[s], (uint32_t)(((i / kStages) - 1) & 1));
      const Loc l = locate(L, t, lc);
      if (l.item != pitem) {
        // cache the header + first gather record of the new descriptor
        if (L.item_desc) {
          dsc = L.descs + L.item_desc[l.item];
          const uint4* src = reinterpret_cast<const uint4*>(dsc);
          uint4* dst = reinterpret_cast<uint4*>(S.pdesc);
          for (uint32_t w = lane; w < sizeof(S.pdesc) / 16; w += 32) dst[w] = __ldg(src + w);
        } else {
          for (uint32_t w = lane; w < sizeof(S.pdesc) / 16; w += 32)
            reinterpret_cast<uint4*>(S.pdesc)[w] = reinterpret_cast<const uint4*>(D.bytes)[w];
        }
        __syncwarp();
        pitem = l.item;
      }
      const SHdr* h = reinterpret_cast<const SHdr*>(S.pdesc);
      const SGRec* G = reinterpret_cast<const SGRec*>(S.pdesc + sizeof(SHdr));
      if (lane == 0) issue_tile(L, dsc, *h, S, l, s);
      if (h->ng >= 1 && G->stage_k != 0xff) {
        const Bases b = bases_of(L, l);
        const char* gp = resolve(G->ptr, b);
        const uint32_t esz = G->c64 ? 8u : 16u;
        const uint64_t gbh = gather(tile_base(*h, l.tile), G->runs, G->n_runs);
        const uint32_t n = 2u << G->stage_k;
        char* dst = reinterpret_cast<char*>(S.gslice[s]);
        for (uint32_t j = lane; j < n; j += 32) {
          const uint64_t gi = gbh | gather(j >> 1, G->grun, G->n_grun) |
                              ((uint64_t)(j & 1) << G->vshift);
          cp_async(dst + j * esz, gp + gi * esz, esz);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_u32(&S.full[s]))
                     : "memory");
      } else {
        mbar_arrive(&S.full[s]);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }

  // ---------------- consumer warps
  ThreadState T;
  uint32_t cur_item = 0xffffffffu, cur_set = 0xffffffffu;
  LocCache lc;
  uint32_t variant = 0, pc64 = 0, oc64 = 0;
  uint64_t i = 0;
  for (uint64_t t = t0; t < t1; ++t, ++i) {
    const int s = (int)(i % kStages);
    const Loc l = locate(L, t, lc);
    mbar_wait(&S.full[s], (uint32_t)((i / kStages) & 1));
    const uint8_t* dsc = L.item_desc ? S.desc[s] : D.bytes;
    const SHdr* h = reinterpret_cast<const SHdr*>(dsc);
    const SGRec* gr = reinterpret_cast<const SGRec*>(dsc + sizeof(SHdr));
    const STRec* tr = reinterpret_cast<const STRec*>(dsc + sizeof(SHdr) + h->ng * sizeof(SGRec));
    if (l.item != cur_item || l.set != cur_set) {
      consumers_sync();  // everyone is done with the previous tables
      const Bases b = bases_of(L, l);
      const SORec* orr = reinterpret_cast<const SORec*>(dsc + sizeof(SHdr) + h->ng * sizeof(SGRec) +
                                                        h->nt * sizeof(STRec));
      const bool full_tile = (1u << h->tb) == (uint32_t)(kJ * kCompute);
      const bool tab_f32 = full_tile && h->nt <= 2 && h->ng <= 1 && h->p_c64 && h->out_c64;
      for (uint32_t q = 0; q < h->nt; ++q) {
        const STRec& TR = tr[q];
        const uint32_t n = 2u << TR.nbits;
        for (uint32_t e = tid; e < n; e += kCompute) {
          const uint32_t bits = e >> 1, v = e & 1;
          // operand loads issued 4 at a time (independent L2 round trips)
          double2 acc = make_double2(1.0, 0.0);
          for (uint32_t k0 = 0; k0 < TR.n_ops; k0 += 4) {
            double2 x[4];
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) {
              x[u] = make_double2(1.0, 0.0);
              if (k0 + u < TR.n_ops) {
                const SORec& O = orr[TR.first_op + k0 + u];
                const uint64_t idx = gather(bits, O.runs, O.n_runs) | ((uint64_t)v << O.vshift);
                x[u] = ldg_c(resolve(O.ptr, b), idx, O.c64);
              }
            }
#pragma unroll
            for (uint32_t u = 0; u < 4; ++u) acc = cmul(acc, x[u]);
          }
          if (tab_f32)
            reinterpret_cast<float2*>(S.tab)[TR.smem_off + e] = make_float2((float)acc.x, (float)acc.y);
          else
            S.tab[TR.smem_off + e] = acc;
        }
      }
      T.ng = h->ng;
      T.nt = h->nt;
      T.tb = h->tb;
      T.tile_elems = 1u << h->tb;
      T.out = const_cast<char*>(resolve(h->out, b));
      const uint32_t ptb = h->ta;
      T.ta = h->ta;
      T.r1 = h->p_rank - 1u;
      T.pk = h->p_k;
      T.split = (ptb >= 1 && T.pk >= ptb) ? 1u : 0u;
      T.pmask = (1u << ptb) - 1u;
      T.pstep = T.split ? (1u << ptb) : (1u << T.pk);
      const uint32_t lane_e = tid & (T.tile_elems - 1);
#pragma unroll
      for (int q = 0; q < kSMaxT; ++q) {
        if (q < (int)T.nt) {
          T.toff[q] = tr[q].smem_off;
          T.tt[q] = (uint32_t)gather(lane_e, tr[q].erun, tr[q].n_erun);
        }
      }
#pragma unroll
      for (int g = 0; g < kSMaxG; ++g) {
        if (g < (int)T.ng) {
          T.gptr[g] = resolve(gr[g].ptr, b);
          T.gvs[g] = gr[g].vshift;
          T.gc64[g] = gr[g].c64;
          T.gt[g] = gather(lane_e, gr[g].erun, gr[g].n_erun);
        }
      }
      T.stage_k = (T.ng >= 1) ? gr[0].stage_k : 0xffu;
      if (T.stage_k != 0xffu) T.ts = (uint32_t)gather(lane_e, gr[0].srun, gr[0].n_srun);
      if (tid < kJ) {
        const uint64_t ej = ((uint64_t)tid * kCompute) & (T.tile_elems - 1);
        if (T.stage_k != 0xffu) S.tjs[tid] = (uint32_t)gather(ej, gr[0].srun, gr[0].n_srun);
        for (uint32_t q = 0; q < T.nt; ++q) S.tjj[q][tid] = (uint32_t)gather(ej, tr[q].erun, tr[q].n_erun);
        for (uint32_t g = 0; g < T.ng; ++g) S.gjj[g][tid] = gather(ej, gr[g].erun, gr[g].n_erun);
      }
      // fast path: full tiles, <= 2 tables, <= 1 gathered operand, matching
      // dtypes; variant = 1 + F32*6 + NT*2 + NG, 0 = generic
      pc64 = h->p_c64;
      oc64 = h->out_c64;
      variant = 0;
      if (T.tile_elems == (uint32_t)(kJ * kCompute) && T.nt <= 2 && T.ng <= 1 && pc64 == oc64) {
        variant = 1 + (pc64 ? 6u : 0u) + T.nt * 2 + T.ng;
        if (T.ng == 1 && T.stage_k != 0xffu) variant = 13 + (pc64 ? 3u : 0u) + T.nt;
      }
      // per-element primary index and output offset of the fast paths
      if (kPrecomp && variant != 0) {
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
          const uint32_t e = tid + (uint32_t)j * kCompute;
          const uint32_t pe = e & T.pmask;
          T.pi0[j] = T.split ? pe : ((pe & ((1u << T.pk) - 1u)) | ((pe >> T.pk) << (T.pk + 1)));
          T.ooff[j] = tile_off(e, T.ta, T.r1);
        }
      }
      cur_item = l.item;
      cur_set = l.set;
      consumers_sync();  // tables visible
    }
    const uint64_t obase = tile_base(*h, l.tile);
    const uint8_t* chunk = S.chunk[s];
    switch (variant) {
      case 1: tile_fast<false, 0, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 2: tile_fast<false, 0, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 3: tile_fast<false, 1, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 4: tile_fast<false, 1, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 5: tile_fast<false, 2, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 6: tile_fast<false, 2, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 7: tile_fast<true, 0, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 8: tile_fast<true, 0, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 9: tile_fast<true, 1, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 10: tile_fast<true, 1, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 11: tile_fast<true, 2, 0>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 12: tile_fast<true, 2, 1>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 13: tile_fast<false, 0, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 14: tile_fast<false, 1, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 15: tile_fast<false, 2, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 16: tile_fast<true, 0, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 17: tile_fast<true, 1, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      case 18: tile_fast<true, 2, 1, true>(T, chunk, S, gr, tr, obase, tid, S.gslice[s]); break;
      default: tile_generic(T, chunk, S, gr, tr, obase, tid, pc64, oc64); break;
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&S.empty[s]);
  }
}

int g_sms = 0;

int prep() {
  static std::atomic<uint64_t> done{0};
  if (needs_setup(done)) {
    cudaError_t e = cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sizeof(Smem));
    if (e != cudaSuccess) {
      set_error(std::string("stream_kernel attribute: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
    mark_setup(done);
  }
  return QTN_OK;
}

int launch(const StreamLaunch& L, const InlineDesc& D, uint64_t total, void* stream) {
  const unsigned grid = (unsigned)std::min<uint64_t>(total, (uint64_t)g_sms);
  cudaError_t e = launch_pdl<true>(stream_kernel, dim3(grid), dim3(kThreads), sizeof(Smem),
                             reinterpret_cast<cudaStream_t>(stream), L, D);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("stream_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}


int launch_list(const StreamLaunch& L, void* stream) {
  int rc = device_check();
  if (rc || (rc = prep())) return rc;
  const uint64_t total = L.total_tiles * L.n_sets;
  if (total == 0) return QTN_OK;
  InlineDesc D;
  std::memset(&D, 0, sizeof(D));
  return launch(L, D, total, stream);
}

int launch_one(const std::vector<uint8_t>& desc, void* stream) {
  int rc = device_check();
  if (rc || (rc = prep())) return rc;
  InlineDesc D;
  std::memset(&D, 0, sizeof(D));
  std::memcpy(D.bytes, desc.data(), std::min<size_t>(desc.size(), sizeof(D.bytes)));
  StreamLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.n_sets = 1;
  L.total_tiles = reinterpret_cast<const SHdr*>(D.bytes)->n_tiles;
  return launch(L, D, L.total_tiles, stream);
}


}  // namespace QTN_STREAM_NS
}  // namespace qtn
