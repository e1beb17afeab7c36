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
constexpr uint32_t kSmallChunk = 1024;
__global__ void __launch_bounds__(256) small_kernel(const __grid_constant__ StreamLaunch L,
                                                    uint32_t tpi_log2) {
  const uint32_t tpi = 1u << tpi_log2;
  const uint32_t item = blockIdx.x * (256u >> tpi_log2) + (threadIdx.x >> tpi_log2);
  if (item >= L.n_items) return;
  const uint32_t lane = threadIdx.x & (tpi - 1);
  Loc l;
  l.item = item;
  l.set = blockIdx.z;
  l.tile = 0;
  const Bases b = bases_of(L, l);
  const uint8_t* dsc = L.descs + L.item_desc[item];
  const SHdr& h = *reinterpret_cast<const SHdr*>(dsc);
  const SGRec* gr = reinterpret_cast<const SGRec*>(dsc + sizeof(SHdr));
  const STRec* tr = reinterpret_cast<const STRec*>(dsc + sizeof(SHdr) + h.ng * sizeof(SGRec));
  const SORec* orr =
      reinterpret_cast<const SORec*>(dsc + sizeof(SHdr) + h.ng * sizeof(SGRec) + h.nt * sizeof(STRec));
  const char* P = resolve(h.p, b);
  char* out = const_cast<char*>(resolve(h.out, b));
  const uint32_t r1 = h.p_rank - 1u, pk = h.p_k;
  const uint64_t n_all = 1ull << h.R;
  const uint64_t o0 = tpi == 256 ? (uint64_t)blockIdx.y * kSmallChunk : 0;
  if (o0 >= n_all) return;
  const uint64_t n_out = tpi == 256 ? min(n_all, o0 + kSmallChunk) : n_all;
  for (uint64_t o = o0 + lane; o < n_out; o += tpi) {
    const uint64_t op = o & ((1ull << r1) - 1);
    const uint64_t p0 = (op & ((1ull << pk) - 1)) | ((op >> pk) << (pk + 1));
    double2 a0 = ldg_c(P, p0, h.p_c64), a1 = ldg_c(P, p0 | (1ull << pk), h.p_c64);
    for (uint32_t q = 0; q < h.nt; ++q) {
      const uint64_t bits = gather(o, tr[q].runs, tr[q].n_runs);
      for (uint32_t k = 0; k < tr[q].n_ops; ++k) {
        const SORec& O = orr[tr[q].first_op + k];
        const char* op_p = resolve(O.ptr, b);
        const uint64_t idx = gather(bits, O.runs, O.n_runs);
        a0 = cmul(a0, ldg_c(op_p, idx, O.c64));
        a1 = cmul(a1, ldg_c(op_p, idx | (1ull << O.vshift), O.c64));
      }
    }
    for (uint32_t g = 0; g < h.ng; ++g) {
      const char* gp = resolve(gr[g].ptr, b);
      const uint64_t idx = gather(o, gr[g].runs, gr[g].n_runs);
      a0 = cmul(a0, ldg_c(gp, idx, gr[g].c64));
      a1 = cmul(a1, ldg_c(gp, idx | (1ull << gr[g].vshift), gr[g].c64));
    }
    const double2 r = make_double2(a0.x + a1.x, a0.y + a1.y);
    if (h.out_c64)
      reinterpret_cast<float2*>(out)[o] = make_float2((float)r.x, (float)r.y);
    else
      reinterpret_cast<double2*>(out)[o] = r;
  }
}

int launch_small(const StreamLaunch& L, uint32_t max_r, void* stream) {
  if (L.n_items == 0 || L.n_sets == 0) return QTN_OK;
  // many items: a warp each; few items (tails of one network): CTAs of
  // kSmallChunk elements each
  const uint32_t tpi_log2 = (uint64_t)L.n_items * L.n_sets >= 4u * 148u * 8u ? 5u : 8u;
  const uint32_t per_block = 256u >> tpi_log2;
  const uint32_t chunks =
      tpi_log2 == 8u ? (uint32_t)(((1ull << max_r) + kSmallChunk - 1) / kSmallChunk) : 1u;
  dim3 grid((L.n_items + per_block - 1) / per_block, chunks, L.n_sets);
  small_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(L, tpi_log2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("small_kernel launch: ") + cudaGetErrorString(e));
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
