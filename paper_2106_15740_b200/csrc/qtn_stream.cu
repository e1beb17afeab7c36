// Streaming bucket kernel (sm_100a): the HBM-bound hot op.
//
// One bucket  out[o] = sum_{v in {0,1}} prod_t T_t[idx_t(o, v)]
// (contraction.py:42-54 `_product` chain + contraction.py:94-96 `.sum`) is
// cut into tiles of 2^tb consecutive outputs.  The output layout keeps the
// primary (largest) operand's variables on the low bits, so a tile's slice
// of the primary is one or two contiguous chunks.  A dedicated producer warp
// moves them into shared memory with cp.async.bulk (the bulk-copy/TMA
// engine; SASS UBLKCP) through a 2-stage full/empty mbarrier pipeline of
// 2^12-element tiles; 8 (or 16, `s512`) consumer warps combine them with
//   * small operands pre-multiplied into shared-memory lookup tables over
//     groups of <= 8 output bits (the diagonal rank-1/2 tensors), and
//   * wider non-primary operands gathered from global memory (L2),
// sum over v in registers, float64 arithmetic, complex64/complex128
// storage.  Every per-element index is precomputed per thread when the
// descriptor changes (gathers are OR-linear over output bits), so the inner
// loop is loads, FMAs and one store.
//
// The same persistent kernel executes one bucket (qtn_bucket_contract) or a
// whole level of an elimination tree across many networks and angle sets
// (level-synchronous HBM executor): items = (descriptor, network), tiles
// flattened, each block takes a contiguous range of tiles.
#define QTN_STREAM_NS s256
#include "qtn_stream_tile.cuh"

#include <type_traits>
#include "qtn_pdl.cuh"

namespace qtn {
using s256::Bases;
using s256::Loc;
using s256::bases_of;
using s256::cmul;
using s256::gather;
using s256::ldg_c;
using s256::resolve;

// ---- small buckets: `tpi` threads (32 or 256) per (item, set), threads over
// output elements.
// out[o] = sum_v P[o | v] * prod_tables prod_ops Op[..] * prod_gathered G[..]
// with the same index maps as the tile kernel applied to the full output
// index o (every run list covers all output bits).
// CTA mode (tpi = 256): blockIdx.y selects a chunk of kSmallChunk elements,
// so a few wide buckets (tail levels of one network) still spread over SMs.
// Elements o = o_begin, o_begin + o_step, ... < o_end of one bucket, every
// operand gathered: out[o] = sum_v P[o | v] * prod_tables prod_ops Op[..] *
// prod_gathered G[..].  CG: operand loads through L2 only (coherent with
// writes of other CTAs ordered by a cluster barrier, chain_kernel).
// CG: 0 read-only path (__ldg), 1 L2 (__ldcg, coherent with writes of other
// CTAs), 2 generic loads (operands in shared or global memory: subtrees)
template <int CG>
__device__ __forceinline__ double2 ld_op(const void* p, uint64_t i, uint32_t c64) {
  if (CG == 2) {
    if (c64) {
      const float2 f = reinterpret_cast<const float2*>(p)[i];
      return make_double2(f.x, f.y);
    }
    return reinterpret_cast<const double2*>(p)[i];
  }
  if (!CG) return ldg_c(p, i, c64);
  if (c64) {
    const float2 f = __ldcg(reinterpret_cast<const float2*>(p) + i);
    return make_double2(f.x, f.y);
  }
  return __ldcg(reinterpret_cast<const double2*>(p) + i);
}
template <int CG>
__device__ __forceinline__ void small_eval(const uint8_t* dsc, const Bases& b, uint64_t o_begin,
                                           uint64_t o_end, uint64_t o_step) {
  const SHdr& h = *reinterpret_cast<const SHdr*>(dsc);
  const SGRec* gr = reinterpret_cast<const SGRec*>(dsc + sizeof(SHdr));
  const STRec* tr = reinterpret_cast<const STRec*>(dsc + sizeof(SHdr) + h.ng * sizeof(SGRec));
  const SORec* orr =
      reinterpret_cast<const SORec*>(dsc + sizeof(SHdr) + h.ng * sizeof(SGRec) + h.nt * sizeof(STRec));
  const char* P = resolve(h.p, b);
  char* out = const_cast<char*>(resolve(h.out, b));
  const uint32_t r1 = h.p_rank - 1u, pk = h.p_k;
  for (uint64_t o = o_begin; o < o_end; o += o_step) {
    const uint64_t op = o & ((1ull << r1) - 1);
    const uint64_t p0 = (op & ((1ull << pk) - 1)) | ((op >> pk) << (pk + 1));
    double2 a0 = ld_op<CG>(P, p0, h.p_c64), a1 = ld_op<CG>(P, p0 | (1ull << pk), h.p_c64);
    for (uint32_t q = 0; q < h.nt; ++q) {
      const uint64_t bits = gather(o, tr[q].runs, tr[q].n_runs);
      for (uint32_t k = 0; k < tr[q].n_ops; ++k) {
        const SORec& O = orr[tr[q].first_op + k];
        const char* op_p = resolve(O.ptr, b);
        const uint64_t idx = gather(bits, O.runs, O.n_runs);
        a0 = cmul(a0, ld_op<CG>(op_p, idx, O.c64));
        a1 = cmul(a1, ld_op<CG>(op_p, idx | (1ull << O.vshift), O.c64));
      }
    }
    for (uint32_t g = 0; g < h.ng; ++g) {
      const char* gp = resolve(gr[g].ptr, b);
      const uint64_t idx = gather(o, gr[g].runs, gr[g].n_runs);
      a0 = cmul(a0, ld_op<CG>(gp, idx, gr[g].c64));
      a1 = cmul(a1, ld_op<CG>(gp, idx | (1ull << gr[g].vshift), gr[g].c64));
    }
    const double2 r = make_double2(a0.x + a1.x, a0.y + a1.y);
    if (h.out_c64)
      reinterpret_cast<float2*>(out)[o] = make_float2((float)r.x, (float)r.y);
    else
      reinterpret_cast<double2*>(out)[o] = r;
  }
}

constexpr uint32_t kSmallChunk = 1024;
constexpr uint32_t kSmallCtaBudget = 2400;  // measured: config 4 0.510 -> 0.479 ms, config 3 default unchanged
__global__ void __launch_bounds__(256) small_kernel(const __grid_constant__ StreamLaunch L,
                                                    uint32_t tpi_log2, uint32_t chunk) {
  pdl_trigger();
  const uint32_t tpi = 1u << tpi_log2;
  const uint32_t item = blockIdx.x * (256u >> tpi_log2) + (threadIdx.x >> tpi_log2);
  if (item >= L.n_items) return;
  const uint32_t lane = threadIdx.x & (tpi - 1);
  Loc l;
  l.item = item;
  l.set = blockIdx.z;
  l.tile = 0;
  const Bases b = bases_of(L, l);
  // the item's descriptor into shared memory (its run lists are read per
  // element; from L1/L2 they were a chain of dependent loads)
  __shared__ uint4 sdesc[8][(kSDescMax + 15) / 16];
  const uint8_t* gdsc = L.descs + L.item_desc[item];
  // CTA mode: chunks beyond the bucket's 2^R elements leave before staging
  if (tpi == 256 && ((uint64_t)blockIdx.y * chunk >> reinterpret_cast<const SHdr*>(gdsc)->R)) return;
  uint4* slot = sdesc[tpi == 256 ? 0 : (threadIdx.x >> 5)];
  {
    const uint32_t n16 = (reinterpret_cast<const SHdr*>(gdsc)->desc_bytes + 15u) / 16u;
    for (uint32_t i = lane; i < n16; i += tpi) slot[i] = __ldg(reinterpret_cast<const uint4*>(gdsc) + i);
    if (tpi == 256) __syncthreads();
    else __syncwarp();
  }
  const uint8_t* dsc = reinterpret_cast<const uint8_t*>(slot);
  // the item lookup and descriptor staging above read static data only: with
  // PDL they overlap the previous level's tail; tensors are read after this
  pdl_wait();
  const uint64_t n_all = 1ull << reinterpret_cast<const SHdr*>(dsc)->R;
  const uint64_t o0 = tpi == 256 ? (uint64_t)blockIdx.y * chunk : 0;
  if (o0 >= n_all) return;
  const uint64_t n_out = tpi == 256 ? min(n_all, o0 + chunk) : n_all;
  small_eval<0>(dsc, b, o0 + lane, n_out, tpi);
}

// ---- tiny subtrees (qtn_stream.h SubItem): one CTA per (subtree, set)
// evaluates the member buckets in order, each with the small-bucket routine
// (threads over output elements), intermediates in shared memory.
__global__ void __launch_bounds__(256) subtree_kernel(const __grid_constant__ StreamLaunch L,
                                                      const SubItem* __restrict__ items,
                                                      const uint64_t* __restrict__ sub_desc) {
  extern __shared__ __align__(16) unsigned char ssm[];
  __shared__ uint4 sdesc[(kSDescMax + 15) / 16];
  pdl_trigger();
  const SubItem it = items[blockIdx.x];
  Bases b;
  b.in = L.in_base + (int64_t)blockIdx.y * L.in_set_stride + L.net_in_off[it.net];
  b.ws = L.ws_base + (int64_t)blockIdx.y * L.ws_set_stride + L.net_ws_off[it.net];
  b.sm = reinterpret_cast<char*>(ssm);
  pdl_wait();
  for (uint32_t k = 0; k < it.count; ++k) {
    const uint8_t* gdsc = L.descs + sub_desc[it.first + k];
    const uint32_t n16 = (reinterpret_cast<const SHdr*>(gdsc)->desc_bytes + 15u) / 16u;
    __syncthreads();  // previous member done (its output visible, descriptor free)
    for (uint32_t i = threadIdx.x; i < n16; i += 256u) sdesc[i] = __ldg(reinterpret_cast<const uint4*>(gdsc) + i);
    __syncthreads();
    const uint8_t* dsc = reinterpret_cast<const uint8_t*>(sdesc);
    small_eval<2>(dsc, b, threadIdx.x, 1ull << reinterpret_cast<const SHdr*>(dsc)->R, 256);
  }
}

int launch_subtree(const StreamLaunch& L, const SubItem* items, uint32_t n_items,
                   const uint64_t* sub_desc, uint32_t smem_bytes, void* stream) {
  if (!n_items || !L.n_sets) return QTN_OK;
  static std::atomic<uint64_t> attr{0};
  if (needs_setup(attr)) {
    cudaError_t e = cudaFuncSetAttribute(subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         96 * 1024);
    if (e != cudaSuccess) {
      set_error(std::string("subtree_kernel attribute: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    mark_setup(attr);
  }
  cudaError_t e = launch_pdl<true>(subtree_kernel, dim3(n_items, L.n_sets), dim3(256), smem_bytes,
                                   reinterpret_cast<cudaStream_t>(stream), L, items, sub_desc);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("subtree_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

int launch_small(const StreamLaunch& L, uint32_t max_r, void* stream, bool pdl) {
  if (L.n_items == 0 || L.n_sets == 0) return QTN_OK;
  // many items: a warp each; few items (tails of one network): CTAs of
  // kSmallChunk elements each
  const uint32_t tpi_log2 = (uint64_t)L.n_items * L.n_sets >= 4u * 148u * 8u ? 5u : 8u;
  const uint32_t per_block = 256u >> tpi_log2;
  // CTA mode: the fewest elements per thread (each a chain of dependent
  // operand round trips) that keeps the launch within ~kSmallCtaBudget CTAs
  static const uint32_t fixed = [] {
    const char* e = getenv("QTN_SMALL_CHUNK");
    const uint32_t v = e ? (uint32_t)atoi(e) : 0u;
    return v >= 256u ? v : 0u;
  }();
  static const uint64_t budget = [] {
    const char* e = getenv("QTN_SMALL_CTAS");
    const uint64_t v = e ? (uint64_t)atoll(e) : 0u;
    return v ? v : (uint64_t)kSmallCtaBudget;
  }();
  uint32_t chunk = kSmallChunk;
  if (fixed) chunk = fixed;
  else if (tpi_log2 == 8u)
    while (chunk > 256u &&
           (uint64_t)L.n_items * L.n_sets * (((1ull << max_r) + chunk / 2 - 1) / (chunk / 2)) <= budget)
      chunk >>= 1;
  const uint32_t chunks = tpi_log2 == 8u ? (uint32_t)(((1ull << max_r) + chunk - 1) / chunk) : 1u;
  dim3 grid((L.n_items + per_block - 1) / per_block, chunks, L.n_sets);
  cudaError_t e = launch_pdl_if<true>(pdl, small_kernel, grid, dim3(256), 0,
                                      reinterpret_cast<cudaStream_t>(stream), L, tpi_log2, chunk);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("small_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

// ---- chains of tiny levels (head and tail of the elimination trees):
// one cluster of kChainCTAs CTAs per angle set runs every level of the chain
// in order, the level's buckets spread over the cluster's threads, a
// cluster barrier (release/acquire) between levels instead of a kernel
// launch per level.  Operands are read through L2 (ld.global.cg).
constexpr uint32_t kChainCTAs = 8;
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__global__ void __launch_bounds__(256) chain_kernel(const __grid_constant__ StreamLaunch L,
                                                    const uint32_t* __restrict__ level_item0,
                                                    uint32_t n_levels) {
  pdl_trigger();
  pdl_wait();
  // a warp per bucket (buckets of a level round-robin over the cluster's
  // warps), its descriptor staged in the warp's shared-memory slot
  __shared__ uint4 sdesc[8][(kSDescMax + 15) / 16];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gwarp = rank * 8u + warp, n_warps = 8u * kChainCTAs;
  uint4* slot = sdesc[warp];
  Loc l;
  l.set = blockIdx.y;
  l.tile = 0;
  for (uint32_t lv = 0; lv < n_levels; ++lv) {
    for (uint32_t it = level_item0[lv] + gwarp; it < level_item0[lv + 1]; it += n_warps) {
      l.item = it;
      const Bases b = bases_of(L, l);
      const uint8_t* gdsc = L.descs + L.item_desc[it];
      const uint32_t n16 = (reinterpret_cast<const SHdr*>(gdsc)->desc_bytes + 15u) / 16u;
      __syncwarp();  // the warp's previous descriptor is no longer read
      for (uint32_t i = lane; i < n16; i += 32) slot[i] = __ldg(reinterpret_cast<const uint4*>(gdsc) + i);
      __syncwarp();
      const uint8_t* dsc = reinterpret_cast<const uint8_t*>(slot);
      small_eval<1>(dsc, b, lane, 1ull << reinterpret_cast<const SHdr*>(dsc)->R, 32);
    }
    cluster_sync_all();
  }
}

int launch_chain(const StreamLaunch& L, const uint32_t* level_item0_dev, uint32_t n_levels,
                 void* stream) {
  if (!n_levels || !L.n_sets) return QTN_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kChainCTAs, L.n_sets);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = reinterpret_cast<cudaStream_t>(stream);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kChainCTAs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, chain_kernel, L, level_item0_dev, n_levels);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("chain_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

// ---- single-operand buckets (partial traces), see qtn_stream.h
// Staged-operand path of trace_kernel: 1-2 operands depending on <= 7 of
// the output's 12 low bits are gathered into shared memory per CTA as
// (v0, v1) pairs; the primary is read at the output's low pr bits (so the
// output may be wider: its new bits come from the staged operands).  PC64 /
// OC64: primary / output element types; float32 math for complex64 outputs,
// float64 for complex128 outputs.
constexpr uint32_t kTraceSmem = kR1MaxS * (2u << kR1StageBits) * 16u + kR1MaxS * 8u * 4u;
template <bool PC64, bool OC64>
__device__ __forceinline__ void trace_staged(const R1Dev& r, const Bases& b, const char* src,
                                             char* out, uint64_t o0, uint64_t o1, double2 w0,
                                             double2 w1, unsigned char* sm) {
  using C = typename std::conditional<OC64, float2, double2>::type;
  // [op][2l + v] staged entries, then the l bits of e = 512 j
  C (*stg)[2 << kR1StageBits] = reinterpret_cast<C (*)[2 << kR1StageBits]>(sm);
  uint32_t (*lj)[8] = reinterpret_cast<uint32_t (*)[8]>(sm + kR1MaxS * (2u << kR1StageBits) * 16u);
  const uint32_t ns = r.ns, pk = r.pk;
  const uint64_t vstep = 1ull << pk, pmask = (1ull << r.pr) - 1;
  for (uint32_t g = 0; g < ns; ++g) {
    const R1Stage& S = r.st[g];
    const char* gp = resolve(S.ptr, b);
    const uint64_t base = gather(o0, S.hrun, S.n_hrun);
    const uint32_t ne = 2u << S.kl;
    for (uint32_t i = threadIdx.x; i < ne; i += 256) {
      const uint64_t idx = base | gather(i >> 1, S.lrun, S.n_lrun) | ((uint64_t)(i & 1u) << S.vshift);
      const double2 a = ldg_c(gp, idx, S.c64);
      stg[g][i] = C{(decltype(C::x))a.x, (decltype(C::x))a.y};
    }
    if (threadIdx.x < 8) lj[g][threadIdx.x] = (uint32_t)gather(512ull * threadIdx.x, S.erun, S.n_erun);
  }
  __syncthreads();
  uint32_t lt[kR1MaxS], lb[kR1MaxS];
#pragma unroll
  for (uint32_t g = 0; g < kR1MaxS; ++g) {
    lt[g] = g < ns ? (uint32_t)gather(2u * threadIdx.x, r.st[g].erun, r.st[g].n_erun) : 0u;
    lb[g] = g < ns ? (uint32_t)gather(1u, r.st[g].erun, r.st[g].n_erun) : 0u;
  }
  auto cm = [](C a, C c) {
    if constexpr (OC64) return C{fmaf(a.x, c.x, -a.y * c.y), fmaf(a.x, c.y, a.y * c.x)};
    else return C{fma(a.x, c.x, -a.y * c.y), fma(a.x, c.y, a.y * c.x)};
  };
  const C W0{(decltype(C::x))w0.x, (decltype(C::x))w0.y}, W1{(decltype(C::x))w1.x, (decltype(C::x))w1.y};
  auto ld = [&](uint64_t i) -> C {  // primary entry i
    if (PC64) {
      const float2 f = __ldg(reinterpret_cast<const float2*>(src) + i);
      return C{f.x, f.y};
    }
    const double2 d = __ldg(reinterpret_cast<const double2*>(src) + i);
    return C{(decltype(C::x))d.x, (decltype(C::x))d.y};
  };
#pragma unroll 2
  for (uint32_t j = 0; j < 8; ++j) {
    const uint64_t p = o0 + 2u * threadIdx.x + 512u * j;
    if (p >= o1) break;
    const uint64_t po = p & pmask;  // even: bit 0 is a primary bit (pr >= 1)
    C a00, a01, a10, a11;  // [output p / p+1][v]
    if (pk >= 1) {
      const uint64_t i0 = (po & (vstep - 1)) | ((po >> pk) << (pk + 1));
      if (PC64) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src) + (i0 >> 1));
        const float4 y = __ldg(reinterpret_cast<const float4*>(src) + ((i0 + vstep) >> 1));
        a00 = C{x.x, x.y}; a10 = C{x.z, x.w}; a01 = C{y.x, y.y}; a11 = C{y.z, y.w};
      } else {
        a00 = ld(i0); a10 = ld(i0 + 1); a01 = ld(i0 + vstep); a11 = ld(i0 + vstep + 1);
      }
    } else {
      a00 = ld(2 * po); a01 = ld(2 * po + 1); a10 = ld(2 * po + 2); a11 = ld(2 * po + 3);
    }
#pragma unroll
    for (uint32_t g = 0; g < kR1MaxS; ++g) {
      if (g < ns) {
        const uint32_t l0 = lt[g] | lj[g][j], l1 = l0 | lb[g];
        a00 = cm(a00, stg[g][2 * l0]);
        a01 = cm(a01, stg[g][2 * l0 + 1]);
        a10 = cm(a10, stg[g][2 * l1]);
        a11 = cm(a11, stg[g][2 * l1 + 1]);
      }
    }
    const C r0 = cm(W0, a00), r0b = cm(W1, a01), r1 = cm(W0, a10), r1b = cm(W1, a11);
    C* oc = reinterpret_cast<C*>(out) + p;
    oc[0] = C{r0.x + r0b.x, r0.y + r0b.y};
    oc[1] = C{r1.x + r1b.x, r1.y + r1b.y};
  }
}

__global__ void __launch_bounds__(256, 8) trace_kernel(const __grid_constant__ StreamLaunch L,
                                                    const R1Dev* __restrict__ items,
                                                    const uint64_t* __restrict__ prefix,
                                                    uint32_t n_items,
                                                    const uint32_t* __restrict__ chunk_item) {
  pdl_trigger();
  pdl_wait();
  const uint64_t cb = blockIdx.x;
  uint32_t lo = 0;
  if (chunk_item) {
    lo = chunk_item[cb];
  } else {
    uint32_t hi = n_items;  // last item whose first chunk <= cb
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (prefix[mid] <= cb) lo = mid;
      else hi = mid;
    }
  }
  const R1Dev& r = items[lo];
  const uint32_t set = blockIdx.y;
  Bases b;
  b.in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[r.net];
  b.ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[r.net];
  const char* src = resolve(r.src, b);
  char* out = const_cast<char*>(resolve(r.out, b));
  const uint64_t n = 1ull << r.R;
  const uint64_t o0 = (cb - prefix[lo]) * kTraceChunk;
  const uint64_t o1 = min(n, o0 + kTraceChunk);
  const uint32_t pk = r.pk;
  const uint64_t vstep = 1ull << pk;
  // per-v weights: product of the v-only operands (float64)
  double2 w0 = make_double2(1.0, 0.0), w1 = w0;
  for (uint32_t k = 0; k < r.nw; ++k) {
    const char* wp = resolve(r.w[k], b);
    w0 = cmul(w0, ldg_c(wp, 0, r.w_c64[k]));
    w1 = cmul(w1, ldg_c(wp, 1, r.w_c64[k]));
  }
  if (r.ns) {
    __shared__ __align__(16) unsigned char tsm[kTraceSmem];
    if (r.src_c64 && r.out_c64)
      trace_staged<true, true>(r, b, src, out, o0, o1, w0, w1, tsm);
    else if (r.out_c64)
      trace_staged<false, true>(r, b, src, out, o0, o1, w0, w1, tsm);
    else if (r.src_c64)
      trace_staged<true, false>(r, b, src, out, o0, o1, w0, w1, tsm);
    else
      trace_staged<false, false>(r, b, src, out, o0, o1, w0, w1, tsm);
    return;
  }
  if (r.src_c64 && r.out_c64 && r.R >= 1 && r.nw) {
    const float2 W0 = make_float2((float)w0.x, (float)w0.y), W1 = make_float2((float)w1.x, (float)w1.y);
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* out4 = reinterpret_cast<float4*>(out);
    // out = W0 * a + W1 * b for one complex64 pair
    auto wsum = [&](float ax, float ay, float bx, float by, float& rx, float& ry) {
      rx = fmaf(W0.x, ax, fmaf(-W0.y, ay, fmaf(W1.x, bx, -W1.y * by)));
      ry = fmaf(W0.x, ay, fmaf(W0.y, ax, fmaf(W1.x, by, W1.y * bx)));
    };
#pragma unroll 8
    for (uint64_t p = o0 + 2u * threadIdx.x; p < o1; p += 512) {
      float4 x, y, z;
      if (pk >= 1) {
        const uint64_t i0 = (p & (vstep - 1)) | ((p >> pk) << (pk + 1));
        x = __ldg(s4 + (i0 >> 1));
        y = __ldg(s4 + ((i0 + vstep) >> 1));
        wsum(x.x, x.y, y.x, y.y, z.x, z.y);
        wsum(x.z, x.w, y.z, y.w, z.z, z.w);
      } else {
        x = __ldg(s4 + p);
        y = __ldg(s4 + p + 1);
        wsum(x.x, x.y, x.z, x.w, z.x, z.y);
        wsum(y.x, y.y, y.z, y.w, z.z, z.w);
      }
      out4[p >> 1] = z;
    }
    return;
  }
  if (r.src_c64 && r.out_c64 && r.R >= 1) {
    // two adjacent outputs per thread and step, 16-byte loads and stores
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* out4 = reinterpret_cast<float4*>(out);
#pragma unroll 8
    for (uint64_t p = o0 + 2u * threadIdx.x; p < o1; p += 512) {
      float4 x, y;
      if (pk >= 1) {
        const uint64_t i0 = (p & (vstep - 1)) | ((p >> pk) << (pk + 1));  // even
        x = __ldg(s4 + (i0 >> 1));
        y = __ldg(s4 + ((i0 + vstep) >> 1));
        out4[p >> 1] = make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
      } else {
        x = __ldg(s4 + p);       // entries 2p, 2p+1
        y = __ldg(s4 + p + 1);   // entries 2p+2, 2p+3
        out4[p >> 1] = make_float4(x.x + x.z, x.y + x.w, y.x + y.z, y.y + y.w);
      }
    }
    return;
  }
  for (uint64_t o = o0 + threadIdx.x; o < o1; o += 256) {
    const uint64_t i0 = (o & (vstep - 1)) | ((o >> pk) << (pk + 1));
    const double2 x = cmul(w0, ldg_c(src, i0, r.src_c64)), y = cmul(w1, ldg_c(src, i0 + vstep, r.src_c64));
    const double2 z = make_double2(x.x + y.x, x.y + y.y);
    if (r.out_c64)
      reinterpret_cast<float2*>(out)[o] = make_float2((float)z.x, (float)z.y);
    else
      reinterpret_cast<double2*>(out)[o] = z;
  }
}

int launch_trace(const StreamLaunch& L, const R1Dev* items, const uint64_t* prefix,
                 uint32_t n_items, uint64_t total_chunks, void* stream, const uint32_t* chunk_item) {
  if (!n_items || !total_chunks || !L.n_sets) return QTN_OK;
  if (total_chunks > 0x7fffffffull || L.n_sets > 65535) {
    set_error("trace_kernel: grid too large");
    return QTN_EINVAL;
  }
  cudaError_t e = launch_pdl<true>(trace_kernel, dim3((uint32_t)total_chunks, L.n_sets), dim3(256), 0,
                                   reinterpret_cast<cudaStream_t>(stream), L, items, prefix, n_items,
                                   chunk_item);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("trace_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

// ---- fused single-operand chains (multi-variable partial traces)
// out[o] = sum over the 2^k source entries spread(o) | offs[m].  A CTA of 8
// warps covers 32 * (8 / G) consecutive outputs: lanes = outputs (32
// consecutive outputs read 32 consecutive source entries for a given m:
// coalesced), G = min(8, 2^k) warps split the m range, each lane keeping 4
// loads in flight; the G partial sums meet in shared memory.  Every source
// entry is read once and no intermediate of the chain is stored.
__global__ void __launch_bounds__(256) reduce_kernel(const __grid_constant__ StreamLaunch L,
                                                     const RedDev* __restrict__ items,
                                                     const uint32_t* __restrict__ prefix,
                                                     uint32_t n_items) {
  pdl_trigger();
  pdl_wait();
  __shared__ uint64_t offs[256];
  const uint32_t cb = blockIdx.x;
  uint32_t lo = 0, hi = n_items;  // last item with prefix <= cb
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= cb) lo = mid;
    else hi = mid;
  }
  const RedDev& r = items[lo];
  const uint32_t k = r.k, nm = 1u << k;
  for (uint32_t m = threadIdx.x; m < nm; m += 256) {
    uint64_t o = 0;
    for (uint32_t q = 0; q < k; ++q) o |= (uint64_t)((m >> q) & 1u) << r.pos[q];
    offs[m] = o;
  }
  __syncthreads();
  const uint64_t n_out = 1ull << r.R;
  const uint32_t set = blockIdx.y;
  Bases b;
  b.in = L.in_base + (int64_t)set * L.in_set_stride + L.net_in_off[r.net];
  b.ws = L.ws_base + (int64_t)set * L.ws_set_stride + L.net_ws_off[r.net];
  const char* src = resolve(r.src, b);
  char* out = const_cast<char*>(resolve(r.out, b));
  const uint32_t chunk = red_chunk(k);
  const uint64_t o0 = (uint64_t)(cb - prefix[lo]) * chunk, o1 = min(n_out, o0 + chunk);
  auto spread = [&](uint64_t o) {
    for (uint32_t q = 0; q < k; ++q) {
      const uint32_t p = r.pos[q];
      o = (o & ((1ull << p) - 1)) | ((o >> p) << (p + 1));
    }
    return o;
  };
  if (r.src_c64 && r.out_c64 && r.R >= 1) {
    // two adjacent outputs per thread and step; bit 0 kept: one 16-byte load
    // per m covers both outputs; bit 0 summed: one 16-byte load covers the
    // (m, m+1) pair of one output
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* out4 = reinterpret_cast<float4*>(out);
    const bool b0 = r.pos[0] == 0;
    const uint64_t d1 = spread(1);
    for (uint64_t p = o0 + 2u * threadIdx.x; p < o1; p += 512) {
      const uint64_t i0 = spread(p);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!b0) {
        uint32_t m = 0;
        for (; m + 4 <= nm; m += 4) {
          float4 x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) x[u] = __ldg(s4 + ((i0 | offs[m + u]) >> 1));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w;
          }
        }
        for (; m < nm; ++m) {
          const float4 x = __ldg(s4 + ((i0 | offs[m]) >> 1));
          acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
        }
      } else {
        for (uint32_t m = 0; m < nm; m += 2) {
          const float4 x = __ldg(s4 + ((i0 | offs[m]) >> 1));
          const float4 y = __ldg(s4 + (((i0 + d1) | offs[m]) >> 1));
          acc.x += x.x + x.z; acc.y += x.y + x.w;
          acc.z += y.x + y.z; acc.w += y.y + y.w;
        }
      }
      out4[p >> 1] = acc;
    }
    return;
  }
  for (uint64_t o = o0 + threadIdx.x; o < o1; o += 256) {
    const uint64_t i0 = spread(o);
    double2 acc = make_double2(0.0, 0.0);
    for (uint32_t m = 0; m < nm; ++m) {
      const double2 x = ldg_c(src, i0 | offs[m], r.src_c64);
      acc.x += x.x;
      acc.y += x.y;
    }
    if (r.out_c64)
      reinterpret_cast<float2*>(out)[o] = make_float2((float)acc.x, (float)acc.y);
    else
      reinterpret_cast<double2*>(out)[o] = acc;
  }
}

int launch_reduce(const StreamLaunch& L, const RedDev* items, const uint32_t* prefix,
                  uint32_t n_items, uint32_t total_chunks, void* stream) {
  if (!n_items || !total_chunks || !L.n_sets) return QTN_OK;
  dim3 grid(total_chunks, L.n_sets);
  cudaError_t e = launch_pdl<true>(reduce_kernel, grid, dim3(256), 0,
                             reinterpret_cast<cudaStream_t>(stream), L, items, prefix, n_items);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("reduce_kernel launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

int launch_stream(const StreamLaunch& L, void* stream, bool wide) {
  return wide ? s512::launch_list(L, stream) : s256::launch_list(L, stream);
}

int launch_stream_single(const std::vector<uint8_t>& desc, void* stream) {
  return s256::launch_one(desc, stream);
}

}  // namespace qtn
