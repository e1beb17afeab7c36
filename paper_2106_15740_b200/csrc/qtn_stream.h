// Streaming bucket executor: descriptors, work lists, launch entry points.
// Shared by the host encoder (qtn_plan.cpp) and the kernel (qtn_stream.cu).
#pragma once

#include <cstdint>
#include <vector>

namespace qtn {

// Tagged pointer: bits 62-63 select the base, the rest is a byte offset.
//   0: absolute address   1: network input block   2: network workspace
constexpr uint64_t kSelShift = 62;
constexpr uint64_t kOffMask = (1ull << kSelShift) - 1;
inline uint64_t tag_abs(const void* p) { return (uint64_t)(uintptr_t)p; }
inline uint64_t tag_in(uint64_t byte_off) { return (1ull << kSelShift) | byte_off; }
inline uint64_t tag_ws(uint64_t byte_off) { return (2ull << kSelShift) | byte_off; }
// 3: shared memory of a tiny-subtree CTA (intermediates that never leave the SM)
inline uint64_t tag_sm(uint64_t byte_off) { return (3ull << kSelShift) | byte_off; }

// pipeline geometry (overridable at build time for A/B experiments)
#ifndef QTN_STREAM_STAGES
#define QTN_STREAM_STAGES 2
#endif
#ifndef QTN_TILE_BITS_C64
#define QTN_TILE_BITS_C64 12
#endif
constexpr int kStreamStages = QTN_STREAM_STAGES;
constexpr int kTileBitsC64 = QTN_TILE_BITS_C64;      // tile = 2^11 complex64 outputs
constexpr int kTileBitsC128 = QTN_TILE_BITS_C64 - 1;
constexpr int kStreamChunk = 16 << kTileBitsC64;     // primary slice bytes per stage

constexpr int kSMaxG = 3;        // gathered operands besides the primary
constexpr int kSMaxT = 4;        // lookup tables
constexpr int kSMaxTOps = 16;    // small operands folded into tables
constexpr int kSGRuns = 33;
constexpr int kSTRuns = 8;

// Descriptor of one bucket (16-byte aligned, variable length:
// header, ng GRec, nt TRec, ntop ORec).
struct SHdr {
  uint64_t out;          // tagged
  uint64_t p;            // tagged primary operand
  uint8_t R;             // output rank
  uint8_t out_c64;
  uint8_t p_c64;
  uint8_t p_k;           // bit of v inside the primary
  uint8_t p_rank;
  uint8_t ng, nt, ntop;
  uint8_t tb;            // tile bits = ta + tn
  uint8_t ta;            // tile-local bits taken from the primary's low bits
  uint8_t tn;            // tile-local bits taken from the new (high) bits
  uint8_t pad0;
  uint16_t table_entries;
  uint16_t desc_bytes;
  uint64_t n_tiles;
  uint8_t pad1[24];
};
// Tile-local element e (tb bits) maps to output bits: e[0,ta) -> o[0,ta),
// e[ta,tb) -> o[rP-1, rP-1+tn) (rP = primary rank).  Every gather is split
// into a per-tile part over o (`runs`, applied to the tile base) and a
// tile-local part over e (`erun`).
constexpr int kStageMaxK = 7;    // stage a gathered operand's tile slice if it
                                 // depends on <= 7 tile-local bits
constexpr int kERuns = 12;
struct SGRec {
  uint64_t ptr;          // tagged
  uint8_t vshift, c64, n_runs;
  uint8_t stage_k;       // 0xff: not staged; else #tile-local bits the operand depends on
  uint32_t runs[kSGRuns];  // output bits -> operand bits (src | dst<<8 | len<<16)
  uint8_t n_srun, n_grun, n_erun, pad2;
  uint32_t srun[kStageMaxK];  // tile-local e bits -> slice index bits
  uint32_t grun[kStageMaxK];  // slice index bits -> operand bits
  uint32_t erun[kERuns];      // tile-local e bits -> operand bits
  uint32_t pad3[5];
};
struct STRec {
  uint8_t nbits, n_runs, first_op, n_ops;
  uint16_t smem_off;
  uint8_t n_erun, pad;
  uint32_t runs[kSTRuns];  // output bits -> table index bits
  uint32_t erun[kSTRuns];  // tile-local e bits -> table index bits
  uint32_t pad2[2];
};
struct SORec {
  uint64_t ptr;          // tagged
  uint8_t vshift, c64, n_runs, pad;
  uint32_t runs[kSTRuns];  // table index bits -> operand bits
};
static_assert(sizeof(SHdr) == 64, "SHdr");
static_assert(sizeof(SGRec) % 16 == 0, "SGRec");
static_assert(sizeof(STRec) % 16 == 0, "STRec");
static_assert(sizeof(SORec) == 48, "SORec");
constexpr int kSDescMax = sizeof(SHdr) + kSMaxG * sizeof(SGRec) + kSMaxT * sizeof(STRec) +
                          kSMaxTOps * sizeof(SORec);

// A bucket in "operand form" before encoding.
struct BucketSpec {
  std::vector<std::vector<int32_t>> opvars;  // operand variable lists (MSB first)
  std::vector<uint8_t> opc64;
  std::vector<uint64_t> optag;               // tagged pointers
  int32_t primary;                           // index of the aligned primary operand
  int32_t v;
  std::vector<int32_t> out_vars;
  bool out_c64;
  uint64_t out_tag;
};

// Host encoder: appends the descriptor bytes; returns QTN_OK or QTN_EINVAL
// (bucket not expressible: too many wide operands).
int encode_stream_desc(const BucketSpec& b, std::vector<uint8_t>& blob);

// Work list of one launch: items = (descriptor, network), tiles flattened.
struct StreamLaunch {
  const uint8_t* descs;         // device blob
  const uint64_t* item_desc;    // device: descriptor byte offset per item
  const uint32_t* item_net;     // device: network index per item
  const uint64_t* tile_prefix;  // device: n_items + 1
  uint32_t n_items;
  uint32_t n_sets;
  uint64_t total_tiles;         // tiles of one set
  const char* in_base;          // inputs
  int64_t in_set_stride;        // bytes
  const int64_t* net_in_off;    // device, bytes
  char* ws_base;
  int64_t ws_set_stride;        // bytes
  const int64_t* net_ws_off;    // device, bytes
};

// wide: the 512-consumer build of the kernel (levels of many small items)
int launch_stream(const StreamLaunch& L, void* stream, bool wide = false);
namespace s256 {
int launch_list(const StreamLaunch& L, void* stream);
int launch_one(const std::vector<uint8_t>& desc, void* stream);
}  // namespace s256
namespace s512 {
int launch_list(const StreamLaunch& L, void* stream);
int launch_one(const std::vector<uint8_t>& desc, void* stream);
}  // namespace s512

// Small buckets (output rank <= kSmallR, or every bucket of a tiny level):
// a warp or a CTA per (item, chunk, set), threads over output elements, every operand gathered through L1/L2 from the same
// descriptors — no tile pipeline, no shared-memory tables.  Uses L.descs,
// L.item_desc, L.item_net, L.n_items, L.n_sets and the base/offset fields.
constexpr int kSmallR = 9;

// Fused single-operand chains: out[o] = sum over k eliminated source bits.
struct RedDev {
  uint64_t src, out;            // tagged pointers
  uint32_t net;                 // network index (bases)
  uint8_t src_c64, out_c64, R, k;
  uint8_t pos[8];               // eliminated bit positions, ascending
};
static_assert(sizeof(RedDev) == 32, "RedDev");
// outputs per CTA: 512 (256 threads x 2 adjacent outputs) x max(1, 8 / 2^k)
// steps, so a CTA reads ~4096 x 2 source entries whatever k is
#ifdef __CUDACC__
#define QTN_HD __host__ __device__
#else
#define QTN_HD
#endif
QTN_HD inline uint32_t red_chunk(uint32_t k) { return 512u * (k >= 3 ? 1u : (8u >> k)); }
// items: device array; prefix: device, n_items + 1 CTA prefix (chunks of red_chunk(k))
int launch_reduce(const StreamLaunch& L, const RedDev* items, const uint32_t* prefix,
                  uint32_t n_items, uint32_t total_chunks, void* stream);
// pdl: programmatic dependent launch (the kernel stages its descriptors
// before waiting on the previous launch; used between tiny levels)
int launch_small(const StreamLaunch& L, uint32_t max_r, void* stream, bool pdl = false);
// A run of consecutive tiny levels in one launch (a CTA cluster per set,
// cluster barriers between levels).  L.item_desc/item_net: the small-item
// lists; level_item0_dev[0..n_levels]: item range of each level (absolute
// indices into those lists).
int launch_chain(const StreamLaunch& L, const uint32_t* level_item0_dev, uint32_t n_levels,
                 void* stream);
// ---- expanding buckets (output wider than its primary operand): the
// outer-product form.  Output bits split into tile-local A bits (9: 256
// threads x 2 adjacent outputs, bits 0-5 always among them so a warp writes
// 512 contiguous bytes), tile-local B bits (h, among the bits no A-side
// operand depends on) and per-tile base bits.  A-side operands (the primary
// and every operand whose variables are the primary's) give, per thread,
// A_v(e) for its 2 outputs; B-side operands (all others) are multiplied once
// per tile into a shared-memory stage Bst[x_b][x_c][v] over the B bits and
// the c tile-local A bits they depend on; then
//   out[base | e | x_b] = A_0(e) Bst[x_b][c(e)][0] + A_1(e) Bst[x_b][c(e)][1]
// is two 16-byte shared loads, ~10 FMAs and one 16-byte store per 2 outputs.
constexpr int kXMaxOps = 6;      // per side
constexpr int kXRuns = 24;
constexpr int kXABits = 9;       // tile-local A bits (256 threads x 2)
constexpr int kXStageMax = 4096; // staged B entries (x_b, x_c, v)
struct XOp {
  uint64_t ptr;                  // tagged
  uint8_t vshift, c64, n_runs, pad;
  uint32_t runs[kXRuns];         // output bits -> operand bits
  uint32_t pad2;
};
struct XDesc {
  uint64_t out;                  // tagged
  uint64_t n_tiles;
  uint8_t R, out_c64, h, c, nA, nB, n_trun, n_arun, n_brun, n_crun, n_acrun, pad[5];
  uint32_t trun[kXRuns];         // tile index bits -> output bits
  uint32_t arun[kXRuns];         // tile-local A element bits -> output bits
  uint32_t brun[kXRuns];         // x_b bits -> output bits
  uint32_t crun[kXRuns];         // x_c bits -> output bits
  uint32_t acrun[kXRuns];        // tile-local A element bits -> x_c bits
  XOp ops[2 * kXMaxOps];         // A-side ops [0, nA), B-side [nA, nA + nB)
};
static_assert(sizeof(XOp) % 16 == 0, "XOp");
static_assert(sizeof(XDesc) % 16 == 0, "XDesc");
// Host encoder: fills d and returns true when the bucket takes the
// expanding-bucket kernel (output rank >= 14, >= 2 B bits, operand limits).
bool encode_expand_desc(const BucketSpec& b, XDesc& d);
struct XLaunch {
  const XDesc* descs;            // device
  const uint32_t* item_desc;     // device: descriptor index per item
  const uint32_t* item_net;      // device: network index per item
  const uint64_t* tile_prefix;   // device: n_items + 1
  uint32_t n_items;
  uint32_t n_sets;
  uint64_t total_tiles;          // tiles of one set
  uint32_t stage_bytes;          // dynamic shared memory (max over items)
  const char* in_base;
  int64_t in_set_stride;
  const int64_t* net_in_off;
  char* ws_base;
  int64_t ws_set_stride;
  const int64_t* net_ws_off;
};
int launch_expand(const XLaunch& L, void* stream);

// ---- expanding bucket + its consumers as one pass (qtn_xt.cu).  The
// union-size result O1 of an expanding bucket (eliminating v1) is read by
// exactly one bucket, which eliminates v2 of it, often a (weighted) partial
// trace, and that result by further partial traces (s_1 .. s_K):
// contraction.py:90-96 K + 2 times in a row.  When the consumers add no
// variables,
//   F[o] = sum_{s_1..s_K} sum_{v2} W_{v2}(o,s) * sum_{v1} A_{v1,v2}(o,s) * B_{v1,v2}(o,s)
// is evaluated per element of the last result F, and O1 (the largest tensor
// of the network) and the chain's intermediates are never written or read
// back.  Index space: F's bits [0, R), then the trailing summed variables
// s_j as extended bits R + j; v2 and v1 are strides of their own.
//   A-type operands: every operand that depends on no loop bit (the
//     expanding bucket's A side, the consumers' operands on A-side
//     variables): loaded per thread for its 2 adjacent outputs x 2^g groups
//     x 4 (v2, v1) values;
//   B group: the expanding bucket's B side, staged per tile as
//     Bst[v2][x_b][x_c][v1] (x_c: thread-owned bits it depends on);
//   W group: the consumers' operands that depend on loop bits, staged as
//     Wst[x_b][x_w][v2].
// Tile = 9 tile-local A bits of F (256 threads x 2 adjacent outputs) x 2^g
// groups (the trailing summed variables the A side depends on: a thread sums
// over them in registers) x h loop bits (hs of them trailing summed
// variables, innermost; the other h - hs are F bits no A-side operand depends
// on).  complex64 intermediates only (float math).
constexpr int kYMaxA = 6;        // A-type operands
constexpr int kYMaxG = 2;        // operands per staged group
constexpr int kYOps = kYMaxA + 2 * kYMaxG;
constexpr int kYMaxH = 6;        // loop bits per tile
constexpr int kYMaxGB = 2;       // group bits (2^g summed positions per thread)
constexpr int kYMaxK = 3;        // trailing traces
constexpr int kYStageB = 8192;   // staged B entries (v2, x_b, x_c, v1)
constexpr int kYStageW = 4096;   // staged W entries (x_b, x_w, v2)
struct YOp {
  uint64_t ptr;                  // tagged
  uint8_t vs1, vs2, c64, n_runs; // bit of v1 / v2 in the operand index (0xff: none)
  uint32_t runs[kXRuns];         // extended bits (F bits, then s_j at R + j) -> operand bits
  uint32_t pad;
};
struct YDesc {
  uint64_t out;                  // tagged
  uint64_t n_tiles;
  uint8_t R, h, c, cw, nA, nB, nW, n_trun, n_arun, n_brun, n_crun, n_wrun, n_acrun, n_awrun, g, hs;
  uint32_t trun[kXRuns];         // tile index bits -> F bits
  uint32_t arun[kXRuns];         // element bits (9 tile-local A bits, then g group bits) -> extended bits
  uint32_t brun[kXRuns];         // x_b bits (hs summed, then h - hs kept) -> extended bits
  uint32_t crun[kXRuns];         // x_c bits -> extended bits
  uint32_t wrun[kXRuns];         // x_w bits -> extended bits
  uint32_t acrun[kXRuns];        // element bits -> x_c bits
  uint32_t awrun[kXRuns];        // element bits -> x_w bits
  YOp ops[kYOps];                // A-type [0, nA), B group [nA, nA+nB), W group after
};
static_assert(sizeof(YOp) % 16 == 0, "YOp");
static_assert(sizeof(YDesc) % 16 == 0, "YDesc");
struct YPairSpec {
  std::vector<std::vector<int32_t>> opvars;  // the expanding bucket's operands, then the consumers' others
  std::vector<uint8_t> opc64;
  std::vector<uint64_t> optag;
  int32_t n1;                                // operands of the expanding bucket
  int32_t primary;                           // its primary
  int32_t v1, v2;
  std::vector<int32_t> trailing;             // s_1 .. s_K, in elimination order
  std::vector<int32_t> out_vars;             // F's layout, MSB first
  uint64_t out_tag;
};
// Host encoder: true when the chain takes xt_kernel.
bool encode_xt_desc(const YPairSpec& s, YDesc& d);
inline uint32_t xt_stage_bytes(const YDesc& d) {
  return 8u * ((4u << (d.h + d.c)) + (d.nW ? (2u << (d.h + d.cw)) : 0u));
}
struct YLaunch {
  const YDesc* descs;            // device
  const uint32_t* item_desc;     // device: descriptor index per item
  const uint32_t* item_net;      // device: network index per item
  const uint64_t* tile_prefix;   // device: n_items + 1
  uint32_t n_items;
  uint32_t n_sets;
  uint64_t total_tiles;          // tiles of one set
  uint32_t stage_bytes;          // dynamic shared memory (max over items)
  uint32_t g;                    // group bits of every item of this launch
  uint32_t pad;
  const char* in_base;
  int64_t in_set_stride;
  const int64_t* net_in_off;
  char* ws_base;
  int64_t ws_set_stride;
  const int64_t* net_ws_off;
};
int launch_xt(const YLaunch& L, void* stream);

// ---- single-operand buckets (partial traces, contraction.py:94-96 on a
// bucket of one tensor): out[o] = P[o with 0 at bit pk] + P[o with 1 at pk],
// the output layout being the primary's minus v.  A pure stream of 3 entries
// per output, run by trace_kernel: 4096 outputs per CTA, 16-byte loads and
// stores, many items per launch (prefix over 4096-output chunks).
// Operands of the bucket that hold only v (rank-1 diagonal factors) are
// folded in as per-v weights: out[o] = w_0 P[o|0] + w_1 P[o|1].
// Complex64 buckets may also carry up to kR1MaxS "staged" operands: any
// operand depending on <= 7 of the output's 12 low bits (the 4096 outputs of
// a CTA touch 2^(kl+1) of its entries): they are gathered into shared memory
// per CTA and read from there per output (config 4's [2,16,26]->25).
constexpr int kR1MaxW = 3;
constexpr int kR1MaxS = 2;
constexpr int kR1StageBits = 7;
struct R1Stage {
  uint64_t ptr;                  // tagged
  uint8_t vshift, c64, kl, n_hrun, n_lrun, n_erun, pad[2];
  uint32_t hrun[24];             // output bits >= 12 -> operand bits (per-CTA base)
  uint32_t lrun[kR1StageBits];   // compact local index bits -> operand bits
  uint32_t erun[kR1StageBits];   // output bits < 12 -> compact local index bits
  uint32_t pad2[2];
};
static_assert(sizeof(R1Stage) % 8 == 0, "R1Stage");
struct R1Dev {
  uint64_t src, out;             // tagged pointers
  uint64_t w[kR1MaxW];           // tagged pointers of rank-1 (v-only) operands
  uint32_t net;                  // network index (bases)
  uint8_t R, pk, src_c64, out_c64;
  uint8_t nw, w_c64[kR1MaxW];
  uint8_t ns;
  uint8_t pr;                    // the primary's non-v bits = the output's low bits (new bits above)
  uint8_t pad[2];
  R1Stage st[kR1MaxS];
};
constexpr uint32_t kTraceChunk = 4096;
// chunk_item (optional): the item of each chunk (no search over the prefix)
int launch_trace(const StreamLaunch& L, const R1Dev* items, const uint64_t* prefix,
                 uint32_t n_items, uint64_t total_chunks, void* stream,
                 const uint32_t* chunk_item = nullptr);

// ---- fused product chains: a bucket of >= 2 operands whose result is then
// reduced by k single-operand buckets (partial traces) is one contraction
//   out[o] = sum_{s in 2^K} prod_t T_t[idx_t(o, s)]      K = k + 1 summed vars
// (contraction.py:42-54 products + k+1 times :94-96 `.sum`), i.e. a batched
// GEMM  out[b,m,n] = sum_k A[b,m,k] B[b,n,k]  with the small operands folded
// in.  The union-size product and the chain's intermediates are never
// written.  Index space U = R output bits [0, R) + K summed bits [R, R+K);
// every operand index is a bit gather of U.  U is cut into
//   q  tile bits (nq <= 16): q = e | s << nto, e = nto output bits (ascending
//      output position), s = the tile's summed bits; the 256 threads take q's
//      low min(8, nq) bits, each thread loops over the rest;
//   l  loop bits: summed bits outside the tile, iterated by the CTA;
//   g  grid bits: output bits outside the tile, one work unit each.
// Per (unit, l): every operand's entries touched by the tile are staged in
// shared memory (compact index over the tile bits it depends on), converted
// to the math type (float for complex64 outputs, double for complex128).
constexpr int kFMaxOps = 8;
constexpr int kFGRuns = 24;
constexpr int kFQRuns = 16;
constexpr int kFMaxQ = 16;            // tile bits
constexpr int kFThreadBits = 8;       // 256 threads
constexpr int kFMaxAcc = 2;           // <= 4 output accumulators per thread
constexpr uint32_t kFBufBytes = 24576;  // one stage buffer (two per CTA: double buffered; measured best of 16-48 KiB)
constexpr int kFLTabBits = 8;         // loop-offset tables up to 2^8 loop values
// Operands are staged raw (their storage type, cp.async, no register round
// trip) into a stage buffer over their compact index (the tile bits they
// depend on).  Operands are grouped into "sides": the compute loop multiplies
// one entry per side.  A side of one operand stored in the math type reads
// the operand's raw region directly; any other side (gate tensors folded into
// a reused wide operand, or a complex128 operand under float math) gets a
// region of its own, filled from the raw regions by a shared-memory pass.
struct FOp {
  uint64_t ptr;                       // tagged
  uint8_t c64, side, nst, n_grun, n_lrun, n_srun, n_ocrun, pairs;
  uint32_t raw_off;                   // byte offset of the raw region in a stage buffer
  uint32_t pad[3];
  uint32_t srun[kFQRuns];             // op compact index bits -> operand bits
  uint32_t ocrun[kFQRuns];            // side compact index bits -> op compact bits
  uint32_t grun[kFGRuns];             // grid index bits -> operand bits
  uint32_t lrun[kFGRuns];             // loop index bits -> operand bits
};
// side kinds: raw region of its single operand (cp.async) / one small
// operand converted to the math type through a register (<= 256 entries) /
// product of several operands (or a large conversion) formed by a shared
// memory pass from their raw regions
// kFSideStream: a raw single-operand side that depends on every tile bit
// (each entry feeds exactly one term): not staged, its terms read it from
// global memory (coalesced), so the stage holds only reused operands
constexpr uint8_t kFSideRaw = 0, kFSideConv = 1, kFSideProd = 2, kFSideStream = 3;
struct FSide {
  uint8_t nst, n_qrun, kind, first_op, n_ops, tconst, aind, pad;  // tconst: no in-thread bits;
                                                                  // aind: independent of the slot bits
  uint32_t st_off;                    // byte offset of the side's region in a stage buffer
  uint32_t qrun[kFQRuns];             // tile index (q) bits -> side compact bits
  uint32_t pad2;
};
struct FDesc {
  uint64_t out;                       // tagged
  uint64_t n_units;                   // 2^ng work units
  uint8_t R, K, out_c64, n_ops, nq, nto, ng, nl;
  uint8_t n_ogrun, n_oqrun, upc_log2, sk, n_sides, has_finish, math_f32, n_var;
  // upc: units per CTA; sk: split-K bits; math_f32: products in float (the
  // chain's head product is a complex64 intermediate), sums in double;
  // n_var: sides [0, n_var) depend on in-thread bits, the rest are per-thread
  // constants of a stage
  uint32_t buf_bytes;                 // bytes of one stage buffer
  uint32_t tab_words;                 // host-built tables (fused_build_tables), 32-bit words
  uint64_t part;                      // tagged: partial sums [unit][2^sk][2^nto] (complex128), sk > 0
  uint64_t tab_off;                   // byte offset of the tables in the batch's table blob
  uint64_t pad3;
  uint32_t ogrun[kFGRuns];            // grid index bits -> output bits
  uint32_t oqrun[kFQRuns];            // tile output bits (q's low nto) -> output bits
  FSide sides[kFMaxOps];
  FOp ops[kFMaxOps];                  // grouped by side, sides in order
};
static_assert(sizeof(FSide) % 16 == 0, "FSide");
static_assert(sizeof(FOp) % 16 == 0, "FOp");
static_assert(sizeof(FDesc) % 16 == 0, "FDesc");
// Host encoder for a fused chain: opvars (MSB-first variable lists), summed
// variables, output variables (MSB first).  Returns false when the chain is
// not expressible (operand count, runs, ranks).
struct FChainSpec {
  std::vector<std::vector<int32_t>> opvars;
  std::vector<uint8_t> opc64;
  std::vector<uint64_t> optag;
  std::vector<int32_t> summed;
  std::vector<int32_t> out_vars;
  bool out_c64;
  bool math_f32;                      // products in float (head product stored complex64)
  uint64_t out_tag;
};
bool encode_fused_desc(const FChainSpec& s, FDesc& d);
// Per-CTA record of a fused launch (built with the batch): where the CTA's
// descriptor + tables sit in the blob, its network and its index within the
// item — one load instead of a search over the item prefix.
struct FCta {
  uint64_t blob;                      // byte offset of [descriptor | tables] in FLaunch::blob
  uint32_t desc16, tab16;             // 16-byte words of the descriptor part / table part
  uint32_t net;                       // network index (bases)
  uint32_t c;                         // CTA index within its item
  uint32_t pad[2];
};
static_assert(sizeof(FCta) == 32, "FCta");
struct FLaunch {
  const FDesc* descs;                 // device
  const uint32_t* tabs;               // device: table blob (FDesc::tab_off)
  const FCta* ctas;                   // device: per-CTA records (fused_kernel)
  const uint8_t* blob;                // device: per descriptor [header, sides, used ops | tables]
  const uint32_t* item_desc;          // device: descriptor index per item
  const uint32_t* item_net;           // device: network index per item
  const uint64_t* cta_prefix;         // device: n_items + 1 (CTAs of one set)
  uint32_t n_items;
  uint32_t n_sets;
  uint64_t total_ctas;                // CTAs of one set
  uint32_t smem_bytes;                // dynamic shared memory (max over items)
  uint32_t f64;                       // items compute in double (complex128 math); one type per launch
  const char* in_base;
  int64_t in_set_stride;
  const int64_t* net_in_off;
  char* ws_base;
  int64_t ws_set_stride;
  const int64_t* net_ws_off;
};
// dynamic shared memory of one descriptor: stage buffers + tables
uint32_t fused_smem_bytes(const FDesc& d);
// the descriptor's lookup tables (pure function of d): appended to `blob`;
// d.tab_words is set, d.tab_off is left to the caller
void fused_build_tables(FDesc& d, std::vector<uint32_t>& blob);
// bytes of the partial-sum block of a split descriptor (0 when sk == 0)
inline uint64_t fused_part_bytes(const FDesc& d) {  // partial sums are complex128
  return d.sk ? (d.n_units << (d.sk + d.nto)) * 16ull : 0ull;
}
int launch_fused(const FLaunch& L, void* stream);
// split items: one CTA per (item, unit) sums the 2^sk partials in order;
// cta_prefix = the units of split items (0 for the others)
int launch_fused_combine(const FLaunch& L, void* stream);

// ---- warp-granular fused chains (qtn_fusedw.cu): the same contraction
//   out[o] = sum_{s in 2^K} prod_t T_t[idx_t(o, s)]
// for chains of 2-4 operands, output rank >= 5 and K <= kWMaxK, one warp per
// 32 * NI outputs: lanes = output bits 0..4, NI in-lane slots over 3 more
// output bits (NI = 8 when R >= 8, else 1), the rest a chunk index per warp.
// No staging and no per-CTA tables: a warp reads its chain's blob (header,
// op records, host-built lane / slot / summed-offset tables) and loads the
// operand entries straight from L1/L2 (chain operands are small and were
// just produced).  Index maps are OR-linear: idx_t = chunk_t + lane_t[l] +
// slot_t[i] + hs_t[s].  The fused_kernel's per-CTA setup (descriptor and
// tables copied to shared memory, cp.async stages) dominated these small
// chains (config 3 default: ~60 % of its stall samples in code run once per
// warp).
constexpr int kWMaxOps = 4;
constexpr int kWMaxK = 10;
constexpr int kWRuns = 12;
struct WHdr {
  uint64_t out;                 // tagged
  uint8_t R, K, n_ops, out_c64;
  uint8_t math_f32, ni_log2, match, n_ocrun;  // match: every operand stored in the math type
  uint32_t ocrun[kWRuns];       // chunk index bits -> output bits
  uint32_t slot_out[8];         // output offset of in-lane slot i
  uint32_t pad[4];
};
struct WOpRec {
  uint64_t ptr;                 // tagged
  uint8_t c64, inv, n_crun, pad;  // inv: independent of the slot bits (one load per s)
  uint32_t crun[kWRuns];        // chunk index bits -> operand bits
  uint32_t lane_off, slot_off, hs_off;  // word offsets of its tables (from the blob start)
  uint32_t pad2[2];
};
static_assert(sizeof(WHdr) % 16 == 0, "WHdr");
static_assert(sizeof(WOpRec) % 16 == 0, "WOpRec");
// host encoder: appends the chain's blob (16-byte aligned) to `blob` and
// returns its number of warps (chunks), or 0 when the chain does not fit
uint32_t encode_warp_chain(const FChainSpec& s, std::vector<uint8_t>& blob);
struct WRec {
  uint32_t blob16;              // chain blob offset, 16-byte units
  uint32_t chunk;               // chunk index within the chain
  uint32_t net;                 // network index (bases)
  uint32_t pad;
};
struct WLaunch {
  const uint8_t* blob;          // device: chain blobs
  const WRec* recs;             // device: one per warp
  uint32_t n_warps;
  uint32_t n_sets;
  uint32_t f64;                 // complex128 math (one type per launch)
  uint32_t pad;
  const char* in_base;
  int64_t in_set_stride;
  const int64_t* net_in_off;
  char* ws_base;
  int64_t ws_set_stride;
  const int64_t* net_ws_off;
};
int launch_fusedw(const WLaunch& L, void* stream);

// ---- tiny subtrees: a connected set of small buckets (output rank <= 9)
// of one elimination tree, evaluated by ONE CTA in elimination order with
// its internal intermediates in shared memory (operand tags with selector
// 3); the subtree's external operands come from the inputs / workspace, its
// root's result goes to the workspace.  One launch per level covers every
// subtree of the level (a CTA per subtree and angle set): the levels of
// tiny buckets and their launch-to-launch latency disappear.
struct SubItem {
  uint32_t net;                 // network index (bases)
  uint32_t first, count;        // member descriptors sub_desc[first .. first+count)
  uint32_t smem;                // shared-memory bytes of its intermediates
};
int launch_subtree(const StreamLaunch& L, const SubItem* items, uint32_t n_items,
                   const uint64_t* sub_desc, uint32_t smem_bytes, void* stream);

// ---- weighted full sums (qtn_wsum.cu): the tail of an elimination order is
// a linear chain of buckets that each eliminate one more variable of the
// previous result T with rank-1/2 gates as the only other operands, down to
// the scalar (contraction.py:90-96 repeated R times).  The chain is one sum
//   Z = sum_x T[x] * prod_k g_k(x[vars_k])
// over T's 2^R entries: T is read once, no intermediate of the chain exists.
// Tile = the low kWsL bits of x: gates on tile bits only form a lookup table
// (built per CTA), gates on high bits a per-tile factor, gates across both
// are multiplied per element.
constexpr int kWsL = 11;          // tile bits (a warp sums one tile)
constexpr int kWsMaxGates = 64;
constexpr int kWsMaxSt = 4;       // gates across the tile boundary
constexpr int kWsMaxCtas = 296;   // CTAs (partial sums) per item
struct WsGate {
  uint64_t ptr;                   // tagged (inputs: complex128 entries)
  uint8_t rank;                   // 1 or 2
  uint8_t b0, b1;                 // T index bits of the gate's variables (entry index = x[b0] << 1 | x[b1]; rank 1: x[b0])
  uint8_t c64;
  uint32_t pad;
};
struct WsDesc {
  uint64_t src, part, out;        // tagged: T (complex64), the CTA partial sums (complex128), the scalar
  uint64_t n_tiles;               // 2^(R - kWsL)
  uint32_t n_ctas;
  uint8_t R, out_c64, n_lo, n_hi, n_st, pad[3];
  uint8_t lo_first[kWsL + 1];     // lo gates sorted by highest bit: those with highest bit b are [lo_first[b], lo_first[b+1])
  uint8_t pad2[16 - (kWsL + 1) % 16];
  WsGate g[kWsMaxGates];          // lo gates, then hi gates, then the gates across
};
static_assert(sizeof(WsGate) == 16, "WsGate");
static_assert(sizeof(WsDesc) % 16 == 0, "WsDesc");
struct WsSpec {
  std::vector<int32_t> src_vars;                  // T's layout, MSB first
  uint64_t src_tag, out_tag;
  bool out_c64;
  std::vector<std::vector<int32_t>> gate_vars;    // rank-1/2 gates, in bucket order
  std::vector<uint64_t> gate_tag;
  std::vector<uint8_t> gate_c64;
};
// Host encoder: false when the chain does not fit (gate counts).  part is set by the caller.
bool encode_wsum_desc(const WsSpec& s, WsDesc& d);
struct WsLaunch {
  const WsDesc* descs;           // device
  const uint32_t* item_desc;     // device: descriptor index per item
  const uint32_t* item_net;      // device: network index per item
  const uint32_t* cta_prefix;    // device: n_items + 1
  uint32_t n_items;
  uint32_t n_sets;
  uint32_t total_ctas;
  uint32_t pad;
  const char* in_base;
  int64_t in_set_stride;
  const int64_t* net_in_off;
  char* ws_base;
  int64_t ws_set_stride;
  const int64_t* net_ws_off;
};
// stage 1 (partial sums per CTA) and stage 2 (their sum -> the scalar) on one stream
int launch_wsum(const WsLaunch& L, void* stream);

// single descriptor with absolute pointers, descriptor passed by value
int launch_stream_single(const std::vector<uint8_t>& desc, void* stream);

}  // namespace qtn
