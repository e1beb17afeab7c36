// Fused product-chain kernel (sm_100a).
//
// A bucket of >= 2 operands followed by k single-operand buckets that sum
// away variables of its result (contraction.py:42-54 `_product` chain, then
// k+1 times the `.sum` of :94-96) is evaluated as ONE contraction
//   out[o] = sum_{s in 2^K} prod_t T_t[idx_t(o, s)]
// i.e. a batched GEMM out[b,m,n] = sum_k A[b,m,k] B[b,n,k] with the small
// gate operands folded into its sides.  The reference materialises the
// union-size product and every partial trace; here neither is written: the
// HBM traffic is the operands once plus the final output.
//
// Index space U = output bits + summed bits (qtn_stream.h FDesc).  A CTA
// (256 threads) takes `upc` grid units (output bits outside the tile); per
// unit it loops over the loop bits (summed bits outside the tile).  Each
// (unit, loop value) is one stage: every operand's entries touched by the
// tile are copied into shared memory with cp.async (double buffered: the
// next stage's copies are in flight while the current one is multiplied),
// then each thread accumulates its <= 4 outputs over the tile's summed bits:
// thread = the tile's low 8 bits, the rest looped in registers.  Products in
// float when the chain's head product is a complex64 intermediate (the
// storage policy of the unfused buckets), double otherwise; every sum across
// stages in double.  A tile with fewer than 8 output bits spreads summed
// bits over the threads; their partial sums meet in shared memory in a fixed
// order (deterministic).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "qtn_internal.h"
#include "qtn_stream.h"
#include "qtn_pdl.cuh"

namespace qtn {
namespace {

constexpr int kAcc = 1 << kFMaxAcc;  // output accumulators per thread

__device__ __forceinline__ float2 cm(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c2d(float2 a) { return make_double2(a.x, a.y); }
__device__ __forceinline__ double2 c2d(double2 a) { return a; }

__device__ __forceinline__ uint64_t fgather(uint64_t x, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((x >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}
// out-of-line form for the per-CTA setup (keeps the kernel's code small:
// a cold kernel fetches its instructions from L2/DRAM)
__device__ __noinline__ uint64_t fgather_ol(uint64_t x, const uint32_t* runs, uint32_t n) {
  return fgather(x, runs, n);
}
__device__ __forceinline__ const char* fresolve(uint64_t tag, const char* in, char* ws) {
  const uint64_t sel = tag >> kSelShift, off = tag & kOffMask;
  if (sel == 1) return in + off;
  if (sel == 2) return ws + off;
  return reinterpret_cast<const char*>(off);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float2 lds_c(uint32_t a, float2*) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_c(uint32_t a, double2*) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
template <typename C> struct Elem;
template <> struct Elem<float2> { using T = float; };
template <> struct Elem<double2> { using T = double; };
template <typename C> __device__ __forceinline__ C ld_conv(const char* p, uint64_t i, uint32_t c64) {
  using E = typename Elem<C>::T;
  if (c64) {
    const float2 f = __ldg(reinterpret_cast<const float2*>(p) + i);
    return C{(E)f.x, (E)f.y};
  }
  const double2 f = __ldg(reinterpret_cast<const double2*>(p) + i);
  return C{(E)f.x, (E)f.y};
}

// Per-operand copy record, built per CTA (pointers resolved for its item/set).
struct OpIssue {
  const char* src;     // operand base
  uint32_t dst;        // raw region (conversion side: side region) byte offset in a buffer
  uint16_t n;          // copies: elements (pairs for mode 1)
  uint8_t mode;        // 0: c64 8-byte, 1: c64 pairs 16-byte, 2: c128 16-byte, 3: conversion (register)
  uint8_t c64;
};
static_assert(sizeof(OpIssue) == 16, "OpIssue");

// Shared-memory layout of a CTA (dynamic part):
//   buf[2]  two stage buffers of d.buf_bytes
//   red     256 x 16 B: cross-thread reduction of summed thread bits
//   issue   per operand OpIssue (pointers resolved for the CTA's item/set)
//   tab     the descriptor's lookup tables, built on the host
//           (fused_build_tables) and copied in with the descriptor:
//     os    4 u64: output offset of the in-thread output bits
//     on    2 x 16 u64: output offset of the thread index (low / high nibble)
//     per operand: kt  gather(k << 8) (pairs: k << 9) of its compact index
//                  lt  2^nl loop-index offsets (nl <= kFLTabBits)
//                  tn  2 x 16: element offset of the thread index (nibbles)
//     per side:    js  njs byte offsets of the summed in-thread bits
//                  ja  4 byte offsets of the in-thread output bits
//                  cn  2 x 16: byte offset of the thread's entry (nibbles)
// Gathers are OR-linear over disjoint bits, so a thread index's offset is
// lo[tid & 15] + hi[tid >> 4].
struct FLayout {
  uint32_t bstride, red, issue, tab, total;  // bytes
  uint32_t os, on, words;                    // words within tab
  uint32_t kt[kFMaxOps], lt[kFMaxOps], tn[kFMaxOps];
  uint32_t js[kFMaxOps], ja[kFMaxOps], cn[kFMaxOps];
};
__host__ __device__ inline FLayout fused_layout(const FDesc& d) {
  FLayout L{};
  const uint32_t nthr = d.nq < kFThreadBits ? d.nq : kFThreadBits;
  const uint32_t jn = d.nq - nthr, na = d.nto > nthr ? d.nto - nthr : 0u;
  const uint32_t njs = 1u << (jn - na);
  const uint32_t nlt = d.nl <= kFLTabBits ? 1u << d.nl : 0u;
  uint32_t w = 0;
  L.os = w;
  w += 2u * kAcc;
  L.on = w;
  w += 2u * 32u;
  for (uint32_t t = 0; t < d.n_ops; ++t) {
    const uint32_t nst = d.ops[t].nst, sh = d.ops[t].pairs ? 9u : 8u;
    L.kt[t] = w;
    w += nst > sh ? 1u << (nst - sh) : 1u;
    L.lt[t] = w;
    w += nlt;
    L.tn[t] = w;
    w += 32u;
  }
  for (uint32_t s = 0; s < d.n_sides; ++s) {
    L.js[s] = w;
    w += njs;
    L.ja[s] = w;
    w += kAcc;
    L.cn[s] = w;
    w += 32u;
  }
  L.words = (w + 3u) & ~3u;
  // the tables first (offset 0: the CTA copies them in before it has read
  // its descriptor), then the stage buffers
  L.tab = 0;
  uint32_t off = 4u * L.words;
  L.bstride = (d.buf_bytes + 15u) & ~15u;
  L.red = off + 2u * L.bstride;
  L.issue = L.red + 256u * 16u;
  off = L.issue + 16u * d.n_ops;
  L.total = (off + 15u) & ~15u;
  return L;
}

// One stage's contribution of the in-thread terms to a thread's per-slot
// partial sums: for each summed in-thread value js and output slot a < 2^NA,
// the product of one staged entry per varying side (32-bit shared addresses:
// thread base + js part + slot part).
// (side tables: sj[s * sstr + js] = summed part, sj[s * sstr + njs + a] = slot part)
// G0: side 0 is streamed from global memory (element offsets, base g0);
// A0: side 0 does not depend on the in-thread output slots
template <typename C, int NS, int NA, bool G0, bool A0 = false>
__device__ __forceinline__ void stage_terms(const uint32_t* sj, uint32_t sstr, const uint32_t* cb,
                                            uint32_t njs, C (&ps)[kAcc], const C* g0) {
  uint32_t jta[NS][1 << NA];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int a = 0; a < (1 << NA); ++a) jta[s][a] = sj[s * sstr + njs + a];
#pragma unroll 2
  for (uint32_t js = 0; js < njs; ++js) {
    uint32_t off[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) off[s] = cb[s] + sj[s * sstr + js];
    C v0[1 << NA];
    if (!G0 && A0) {  // side 0 does not depend on the slot bits: one load for every slot
      const C v = lds_c(off[0], (C*)nullptr);
#pragma unroll
      for (int a = 0; a < (1 << NA); ++a) v0[a] = v;
    } else {
#pragma unroll
      for (int a = 0; a < (1 << NA); ++a)  // the streamed loads of all slots first
        v0[a] = G0 ? __ldg(g0 + off[0] + jta[0][a]) : lds_c(off[0] + jta[0][a], (C*)nullptr);
    }
#pragma unroll
    for (int a = 0; a < (1 << NA); ++a) {
      C p = v0[a];
#pragma unroll
      for (int s = 1; s < NS; ++s) p = cm(p, lds_c(off[s] + jta[s][a], (C*)nullptr));
      ps[a] = cadd(ps[a], p);
    }
  }
}
template <typename C, int NS, bool G0>
__device__ __forceinline__ void stage_terms_na(uint32_t na, const uint32_t* sj, uint32_t sstr,
                                               const uint32_t* cb, uint32_t njs, C (&ps)[kAcc],
                                               const C* g0, bool a0 = false) {
  if (!G0 && a0 && NS == 2) {  // the common GEMM shape: side 0 shared by every slot
    switch (na) {
      case 0: stage_terms<C, NS, 0, false, true>(sj, sstr, cb, njs, ps, g0); break;
      case 1: stage_terms<C, NS, 1, false, true>(sj, sstr, cb, njs, ps, g0); break;
      default: stage_terms<C, NS, 2, false, true>(sj, sstr, cb, njs, ps, g0); break;
    }
    return;
  }
  switch (na) {
    case 0: stage_terms<C, NS, 0, G0>(sj, sstr, cb, njs, ps, g0); break;
    case 1: stage_terms<C, NS, 1, G0>(sj, sstr, cb, njs, ps, g0); break;
    default: stage_terms<C, NS, 2, G0>(sj, sstr, cb, njs, ps, g0); break;
  }
}
// more than 4 varying sides: slot offsets from shared memory
template <typename C>
__device__ __forceinline__ void stage_terms_any(uint32_t nv, uint32_t na, const uint32_t* sj, uint32_t sstr,
                                                const uint32_t* cb, uint32_t njs, C (&ps)[kAcc]) {
  for (uint32_t js = 0; js < njs; ++js) {
#pragma unroll
    for (uint32_t a = 0; a < (uint32_t)kAcc; ++a) {
      if (a < (1u << na)) {
        C p = lds_c(cb[0] + sj[js] + sj[njs + a], (C*)nullptr);
        for (uint32_t s = 1; s < nv; ++s)
          p = cm(p, lds_c(cb[s] + sj[s * sstr + js] + sj[s * sstr + njs + a], (C*)nullptr));
        ps[a] = cadd(ps[a], p);
      }
    }
  }
}

template <typename C>
__device__ __forceinline__ void fused_body(const FDesc& d, const uint32_t* tabs, const char* in, char* ws,
                                           uint64_t u0, uint64_t u1, uint32_t l0, uint32_t l1,
                                           uint32_t split, unsigned char* smem) {
  using E = typename Elem<C>::T;
  const FLayout Lo = fused_layout(d);
  const uint32_t tid = threadIdx.x, n = d.n_ops, ns = d.n_sides, nv = d.n_var;
  const uint32_t nq = d.nq, nto = d.nto;
  const uint32_t nthr = nq < (uint32_t)kFThreadBits ? nq : (uint32_t)kFThreadBits;
  const uint32_t jn = nq - nthr;                           // in-thread tile bits
  const uint32_t na = nto > nthr ? nto - nthr : 0u;        // in-thread output bits
  const uint32_t njs = 1u << (jn - na);
  const bool active = tid < (1u << nthr);
  unsigned char* bufs = smem + 4u * Lo.words;             // stage buffers (after the tables)
  const uint32_t sbase = smem_u32(bufs);                   // stage buffer 0
  const bool ltab_on = d.nl <= kFLTabBits;
  // ---- per-CTA tables: the host-built tables with the descriptor (one
  // 16-byte copy per thread), the copy records with resolved pointers
  const uint32_t* tw = reinterpret_cast<const uint32_t*>(smem + Lo.tab);  // copied in by the entry
  (void)tabs;
  {
    if (tid < n) {
      const FOp& o = d.ops[tid];
      const FSide& S = d.sides[o.side];
      OpIssue r;
      r.src = fresolve(o.ptr, in, ws);
      r.c64 = o.c64;
      if (S.kind == kFSideStream) {
        r.mode = 4;  // read by the terms from global memory: no copies
        r.dst = 0;
        r.n = 0;
      } else if (S.kind == kFSideConv) {
        r.mode = 3;
        r.dst = S.st_off;
        r.n = (uint16_t)(1u << o.nst);
      } else {
        r.mode = o.pairs ? 1 : (o.c64 ? 0 : 2);
        r.dst = o.raw_off;
        r.n = (uint16_t)(o.pairs ? (1u << o.nst) >> 1 : 1u << o.nst);
      }
      reinterpret_cast<OpIssue*>(smem + Lo.issue)[tid] = r;
    }
  }
  __syncthreads();
  // per-thread parts: operand element offsets (copies), side entry addresses (terms)
  const uint32_t tlo = tid & 15u, thi = tid >> 4;
  uint32_t thr[kFMaxOps], cth[kFMaxOps];
  for (uint32_t t = 0; t < kFMaxOps; ++t) {
    thr[t] = t < n ? tw[Lo.tn[t] + tlo] + tw[Lo.tn[t] + 16u + thi] : 0u;
    // shared byte address of the thread's entry of side t in buffer 0
    // (streamed side 0: the thread's element offset in the operand)
    const uint32_t tpart = active && t < ns ? tw[Lo.cn[t] + tlo] + tw[Lo.cn[t] + 16u + thi] : 0u;
    cth[t] = t < ns ? (d.sides[t].kind == kFSideStream ? tpart : sbase + d.sides[t].st_off + tpart) : 0u;
  }
  char* outp = const_cast<char*>(fresolve(d.out, in, ws));
  double2* part = d.sk ? reinterpret_cast<double2*>(const_cast<char*>(fresolve(d.part, in, ws))) : nullptr;
  const uint64_t* tw64 = reinterpret_cast<const uint64_t*>(tw);
  const uint64_t othr = tw64[Lo.on / 2u + tlo] + tw64[Lo.on / 2u + 16u + thi];
  const OpIssue* iss = reinterpret_cast<const OpIssue*>(smem + Lo.issue);
  const uint64_t* oslot = tw64 + Lo.os / 2u;
  const uint32_t* sj = tw + Lo.js[0];
  const uint32_t sstr = njs + (uint32_t)kAcc + 32u;  // side table stride (fused_layout)
  const uint32_t nlr = l1 - l0;  // a power of two
  const uint32_t lsh = 31u - __clz(nlr), lmask = nlr - 1u;
  const uint32_t nit = (uint32_t)(u1 - u0) * nlr;
  uint64_t gbu[kFMaxOps];
  uint64_t gunit = ~0ull;
  C pend[kFMaxOps];  // conversion sides: this thread's element of the next stage (few live)
  // issue the copies of iteration `it` into buffer `buf` (shared byte address);
  // conversion sides load into `pend` (stored after the current stage's terms)
  auto issue = [&](uint32_t it, uint32_t buf) {
    const uint64_t unit = u0 + (it >> lsh);
    const uint32_t l = l0 + (it & lmask);
    if (unit != gunit) {  // unit part + thread part of every operand index
      for (uint32_t t = 0; t < n; ++t) gbu[t] = fgather_ol(unit, d.ops[t].grun, d.ops[t].n_grun) + thr[t];
      gunit = unit;
    }
#pragma unroll 1
    for (uint32_t t = 0; t < n; ++t) {
      const OpIssue r = iss[t];
      const uint64_t base =
          gbu[t] + (ltab_on ? tw[Lo.lt[t] + l] : fgather(l, d.ops[t].lrun, d.ops[t].n_lrun));
      const uint32_t* kt = tw + Lo.kt[t];
      if (r.mode == 4) continue;  // streamed side: no copies
      if (r.mode == 3) {
        if (tid < r.n) pend[t] = ld_conv<C>(r.src, base, r.c64);
        continue;
      }
      const uint32_t elt = r.mode == 2 ? 16u : 8u;  // bytes per operand element
      const char* src = r.src + (uint64_t)elt * base;
      if (r.mode == 0) {
        const uint32_t dst = buf + r.dst + 8u * tid;
        for (uint32_t k = 0, i = tid; i < r.n; ++k, i += 256u)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst + 2048u * k),
                       "l"(src + 8ull * kt[k]) : "memory");
      } else {
        const uint32_t dst = buf + r.dst + 16u * tid;
        for (uint32_t k = 0, i = tid; i < r.n; ++k, i += 256u)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 4096u * k),
                       "l"(src + (uint64_t)elt * kt[k]) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto store_pend = [&](uint32_t bufoff) {
    for (uint32_t t = 0; t < n; ++t) {
      const OpIssue r = iss[t];
      if (r.mode == 3 && tid < r.n) reinterpret_cast<C*>(bufs + bufoff + r.dst)[tid] = pend[t];
    }
  };
  // product sides: their math-type region from the operands' raw regions
  auto finish = [&](uint32_t bufoff) {
    for (uint32_t si = 0; si < ns; ++si) {
      const FSide& S = d.sides[si];
      if (S.kind != kFSideProd) continue;
      C* dst = reinterpret_cast<C*>(bufs + bufoff + S.st_off);
      for (uint32_t c = tid; c < (1u << S.nst); c += 256u) {
        C v = C{1, 0};
        for (uint32_t t = S.first_op; t < S.first_op + S.n_ops; ++t) {
          const FOp& o = d.ops[t];
          const uint32_t j = (uint32_t)fgather(c, o.ocrun, o.n_ocrun);
          C x;
          if (o.c64) {
            const float2 f = reinterpret_cast<const float2*>(bufs + bufoff + o.raw_off)[j];
            x = C{(E)f.x, (E)f.y};
          } else {
            const double2 f = reinterpret_cast<const double2*>(bufs + bufoff + o.raw_off)[j];
            x = C{(E)f.x, (E)f.y};
          }
          v = t == S.first_op ? x : cm(v, x);
        }
        dst[c] = v;
      }
    }
  };
  // a streamed side 0 (kFSideStream) is read by the terms from global memory
  const bool stream0 = ns > 0 && d.sides[0].kind == kFSideStream && nv >= 1 && nv <= 4;
  uint64_t sunit = ~0ull, sgb = 0;
  issue(0, sbase);
  store_pend(0);
  double2 acc[kAcc];
#pragma unroll
  for (int a = 0; a < kAcc; ++a) acc[a] = make_double2(0.0, 0.0);
  for (uint32_t it = 0; it < nit; ++it) {
    const uint32_t cur = it & 1u, boff = cur * Lo.bstride, noff = (cur ^ 1u) * Lo.bstride;
    const bool more = it + 1 < nit;
    if (more) {  // the next stage's copies fly while this one is multiplied
      issue(it + 1, sbase + noff);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    if (d.has_finish) {
      finish(boff);
      __syncthreads();
    }
    if (active) {
      uint32_t cb[kFMaxOps];
#pragma unroll
      for (uint32_t t = 0; t < kFMaxOps; ++t) cb[t] = cth[t] + boff;
      C ps[kAcc];
#pragma unroll
      for (int a = 0; a < kAcc; ++a) ps[a] = C{0, 0};
      if (stream0) {
        // side 0 from global memory at this iteration's operand base
        cb[0] = cth[0];
        const uint64_t unit = u0 + (it >> lsh);
        const uint32_t l = l0 + (it & lmask);
        const uint32_t t0 = d.sides[0].first_op;
        if (unit != sunit) {
          sgb = fgather_ol(unit, d.ops[t0].grun, d.ops[t0].n_grun);
          sunit = unit;
        }
        const C* g0 = reinterpret_cast<const C*>(iss[t0].src) + sgb +
                      (ltab_on ? tw[Lo.lt[t0] + l] : fgather(l, d.ops[t0].lrun, d.ops[t0].n_lrun));
        switch (nv) {
          case 1: stage_terms_na<C, 1, true>(na, sj, sstr, cb, njs, ps, g0); break;
          case 2: stage_terms_na<C, 2, true>(na, sj, sstr, cb, njs, ps, g0); break;
          case 3: stage_terms_na<C, 3, true>(na, sj, sstr, cb, njs, ps, g0); break;
          default: stage_terms_na<C, 4, true>(na, sj, sstr, cb, njs, ps, g0); break;
        }
      } else {
        switch (nv) {
          case 0: ps[0] = C{1, 0}; break;
          case 1: stage_terms_na<C, 1, false>(na, sj, sstr, cb, njs, ps, nullptr); break;
          case 2: stage_terms_na<C, 2, false>(na, sj, sstr, cb, njs, ps, nullptr, d.sides[0].aind != 0); break;
          case 3: stage_terms_na<C, 3, false>(na, sj, sstr, cb, njs, ps, nullptr); break;
          case 4: stage_terms_na<C, 4, false>(na, sj, sstr, cb, njs, ps, nullptr); break;
          default: stage_terms_any<C>(nv, na, sj, sstr, cb, njs, ps); break;
        }
      }
      // sides constant over the in-thread bits multiply the stage's sums once
      C tc = C{1, 0};
      for (uint32_t s = nv; s < ns; ++s) tc = cm(tc, lds_c(cb[s], (C*)nullptr));
#pragma unroll
      for (int a = 0; a < kAcc; ++a) acc[a] = cadd(acc[a], c2d(cm(ps[a], tc)));
    }
    if (more) store_pend(noff);
    if (((it + 1) & lmask) == 0) {  // last loop value of this unit: write its outputs
      const uint64_t unit = u0 + (it >> lsh);
      const uint64_t og = part ? 0ull : fgather_ol(unit, d.ogrun, d.n_ogrun);
      auto emit = [&](uint32_t e, uint32_t a, double2 v) {
        if (part) {
          part[(((unit << d.sk) | split) << nto) | e] = v;
        } else {
          const uint64_t o = og | othr | oslot[a];
          if (d.out_c64)
            reinterpret_cast<float2*>(outp)[o] = make_float2((float)v.x, (float)v.y);
          else
            reinterpret_cast<double2*>(outp)[o] = v;
        }
      };
      if (nto >= nthr) {
        if (active) {
#pragma unroll
          for (uint32_t a = 0; a < (uint32_t)kAcc; ++a)
            if (a < (1u << na)) emit(tid | (a << nthr), a, acc[a]);
        }
      } else {
        // thread bits [nto, nthr) are summed: combine in shared memory, fixed order
        double2* red = reinterpret_cast<double2*>(smem + Lo.red);
        if (active) red[tid] = acc[0];
        __syncthreads();
        if (tid < (1u << nto)) {
          double2 r = red[tid];
          for (uint32_t s2 = 1; s2 < (1u << (nthr - nto)); ++s2) r = cadd(r, red[tid | (s2 << nto)]);
          emit(tid, 0, r);
        }
      }
#pragma unroll
      for (int a = 0; a < kAcc; ++a) acc[a] = make_double2(0.0, 0.0);
    }
    __syncthreads();  // buffer `cur` is free for the copies of it + 2
  }
}

// 3 CTAs per SM (80 registers; the complex128-math variant spills ~260 bytes,
// measured equal to 2 CTAs per SM without spills)
template <typename C>
__global__ void __launch_bounds__(256, 3) fused_kernel(const __grid_constant__ FLaunch L) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ __align__(16) FDesc SD;
  pdl_trigger();
  pdl_wait();
  // the CTA's record, then its descriptor and tables in one pass (both
  // copies in flight together: the tables sit at offset 0 of the dynamic
  // shared memory whatever the descriptor says)
  const FCta rec = L.ctas[blockIdx.x];
  {
    const uint4* src = reinterpret_cast<const uint4*>(L.blob + rec.blob);
    uint4* dsd = reinterpret_cast<uint4*>(&SD);
    uint4* dtab = reinterpret_cast<uint4*>(fsm);
    const uint32_t nd = rec.desc16, nt = rec.tab16;
    for (uint32_t i = threadIdx.x; i < nd + nt; i += 256u) {
      const uint4 v = __ldg(src + i);
      if (i < nd) dsd[i] = v;
      else dtab[i - nd] = v;
    }
  }
  __syncthreads();
  const uint32_t net = rec.net, set = blockIdx.y;
  const char* in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
  char* ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
  const uint64_t c = rec.c;
  uint64_t u0, u1;
  uint32_t l0 = 0, l1 = 1u << SD.nl, split = 0;
  if (SD.sk) {  // split-K: CTA = (unit, split), a contiguous range of loop values
    u0 = c >> SD.sk;
    u1 = u0 + 1;
    split = (uint32_t)(c & ((1u << SD.sk) - 1u));
    l0 = split << (SD.nl - SD.sk);
    l1 = l0 + (1u << (SD.nl - SD.sk));
  } else {
    u0 = c << SD.upc_log2;
    u1 = min((uint64_t)SD.n_units, (uint64_t)(u0 + (1ull << SD.upc_log2)));
  }
  fused_body<C>(SD, L.tabs, in, ws, u0, u1, l0, l1, split, fsm);
}

// Split-K combine: one CTA per (split item, unit); thread e sums its output's
// 2^sk partials (complex128) in split order and stores the output element.
__global__ void __launch_bounds__(256) fused_combine_kernel(const __grid_constant__ FLaunch L) {
  pdl_trigger();
  pdl_wait();
  const uint64_t cb = blockIdx.x;
  uint32_t lo = 0, hi = L.n_items;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (L.cta_prefix[mid] <= cb) lo = mid;
    else hi = mid;
  }
  const FDesc& d = L.descs[L.item_desc[lo]];
  const uint32_t net = L.item_net[lo], set = blockIdx.y;
  const char* in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[net];
  char* ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[net];
  const uint64_t unit = cb - L.cta_prefix[lo];
  const uint32_t nto = d.nto, sk = d.sk;
  const uint64_t og = fgather(unit, d.ogrun, d.n_ogrun);
  char* outp = const_cast<char*>(fresolve(d.out, in, ws));
  const double2* part = reinterpret_cast<const double2*>(fresolve(d.part, in, ws));
  for (uint32_t e = threadIdx.x; e < (1u << nto); e += 256u) {
    const uint64_t o = og | fgather(e, d.oqrun, d.n_oqrun);
    const double2* p = part + ((unit << (sk + nto)) | e);
    // 4 partial sums in flight (sk >= 1 when split); combined in split order
    const uint32_t ns = 1u << sk;
    double2 r = make_double2(0.0, 0.0);
    uint32_t s = 0;
    for (; s + 4u <= ns; s += 4u) {
      const double2 a = __ldcg(p + ((uint64_t)s << nto)), b = __ldcg(p + ((uint64_t)(s + 1) << nto));
      const double2 c = __ldcg(p + ((uint64_t)(s + 2) << nto)), e2 = __ldcg(p + ((uint64_t)(s + 3) << nto));
      r = cadd(cadd(cadd(cadd(r, a), b), c), e2);
    }
    for (; s < ns; ++s) r = cadd(r, __ldcg(p + ((uint64_t)s << nto)));
    if (d.out_c64)
      reinterpret_cast<float2*>(outp)[o] = make_float2((float)r.x, (float)r.y);
    else
      reinterpret_cast<double2*>(outp)[o] = r;
  }
}

}  // namespace

uint32_t fused_smem_bytes(const FDesc& d) { return fused_layout(d).total; }

static uint64_t hgather(uint64_t x, const uint32_t* runs, uint32_t n) {
  uint64_t idx = 0;
  for (uint32_t r = 0; r < n; ++r) {
    const uint32_t w = runs[r];
    const uint32_t s = w & 0xff, d = (w >> 8) & 0xff, l = (w >> 16) & 0xff;
    idx |= ((x >> s) & ((1ull << l) - 1)) << d;
  }
  return idx;
}

void fused_build_tables(FDesc& d, std::vector<uint32_t>& blob) {
  const FLayout L = fused_layout(d);
  std::vector<uint32_t> w(L.words, 0u);
  const uint32_t nthr = d.nq < kFThreadBits ? d.nq : kFThreadBits;
  const uint32_t jn = d.nq - nthr, na = d.nto > nthr ? d.nto - nthr : 0u;
  const uint32_t njs = 1u << (jn - na);
  const uint32_t esz = d.math_f32 ? 8u : 16u;
  auto put64 = [&](uint32_t at, uint64_t v) {
    w[at] = (uint32_t)v;
    w[at + 1] = (uint32_t)(v >> 32);
  };
  for (uint32_t a = 0; a < (uint32_t)kAcc; ++a)
    put64(L.os + 2 * a, a < (1u << na) ? hgather((uint64_t)a << nthr, d.oqrun, d.n_oqrun) : 0ull);
  for (uint32_t i = 0; i < 16; ++i) {
    put64(L.on + 2 * i, hgather(i, d.oqrun, d.n_oqrun));
    put64(L.on + 32 + 2 * i, hgather((uint64_t)i << 4, d.oqrun, d.n_oqrun));
  }
  for (uint32_t t = 0; t < d.n_ops; ++t) {
    const FOp& o = d.ops[t];
    const uint32_t sh = o.pairs ? 9u : 8u;
    const uint32_t nk = o.nst > sh ? 1u << (o.nst - sh) : 1u;
    for (uint32_t k = 0; k < nk; ++k) w[L.kt[t] + k] = (uint32_t)hgather((uint64_t)k << sh, o.srun, o.n_srun);
    if (d.nl <= kFLTabBits)
      for (uint32_t l = 0; l < (1u << d.nl); ++l) w[L.lt[t] + l] = (uint32_t)hgather(l, o.lrun, o.n_lrun);
    const uint32_t m = o.pairs ? 2u : 1u;  // copy index of thread tid: tid (pairs: 2 tid)
    for (uint32_t i = 0; i < 16; ++i) {
      w[L.tn[t] + i] = (uint32_t)hgather(m * i, o.srun, o.n_srun);
      w[L.tn[t] + 16 + i] = (uint32_t)hgather((uint64_t)m * (i << 4), o.srun, o.n_srun);
    }
  }
  for (uint32_t s = 0; s < d.n_sides; ++s) {
    const FSide& S = d.sides[s];
    // offset of tile index q: shared byte offset of the side's compact
    // entry, or (streamed side) the element offset in the operand
    const FOp& o0 = d.ops[S.first_op];
    auto off = [&](uint64_t q) -> uint32_t {
      const uint64_t c = hgather(q, S.qrun, S.n_qrun);
      return S.kind == kFSideStream ? (uint32_t)hgather(c, o0.srun, o0.n_srun) : esz * (uint32_t)c;
    };
    for (uint32_t js = 0; js < njs; ++js) w[L.js[s] + js] = off((uint64_t)(js << na) << nthr);
    for (uint32_t a = 0; a < (uint32_t)kAcc; ++a) w[L.ja[s] + a] = a < (1u << na) ? off((uint64_t)a << nthr) : 0u;
    for (uint32_t i = 0; i < 16; ++i) {
      w[L.cn[s] + i] = off(i);
      w[L.cn[s] + 16 + i] = off((uint64_t)i << 4);
    }
  }
  d.tab_words = L.words;
  blob.insert(blob.end(), w.begin(), w.end());
}

int launch_fused(const FLaunch& L, void* stream) {
  if (!L.n_items || !L.n_sets || !L.total_ctas) return QTN_OK;
  if (L.n_sets > 65535 || L.total_ctas > 0x7fffffffull) {
    set_error("fused_kernel: grid too large");
    return QTN_EINVAL;
  }
  static std::atomic<uint64_t> attr{0};
  if (needs_setup(attr)) {
    cudaError_t e = cudaFuncSetAttribute(fused_kernel<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(2 * kFBufBytes + 32768));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fused_kernel<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(2 * kFBufBytes + 32768));
    if (e != cudaSuccess) {
      set_error(std::string("fused_kernel attribute: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    mark_setup(attr);
  }
  dim3 grid((uint32_t)L.total_ctas, L.n_sets);
  cudaError_t e = L.f64 ? launch_pdl<true>(fused_kernel<double2>, grid, dim3(256), L.smem_bytes,
                                           reinterpret_cast<cudaStream_t>(stream), L)
                        : launch_pdl<true>(fused_kernel<float2>, grid, dim3(256), L.smem_bytes,
                                           reinterpret_cast<cudaStream_t>(stream), L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("fused_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

int launch_fused_combine(const FLaunch& L, void* stream) {
  if (!L.n_items || !L.n_sets || !L.total_ctas) return QTN_OK;
  if (L.n_sets > 65535 || L.total_ctas > 0x7fffffffull) {
    set_error("fused_combine_kernel: grid too large");
    return QTN_EINVAL;
  }
  dim3 grid((uint32_t)L.total_ctas, L.n_sets);
  cudaError_t e = launch_pdl<true>(fused_combine_kernel, grid, dim3(256), 0,
                                   reinterpret_cast<cudaStream_t>(stream), L);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("fused_combine_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

}  // namespace qtn
