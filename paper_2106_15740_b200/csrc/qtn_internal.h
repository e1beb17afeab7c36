// Internal structures shared by the host plan compiler (qtn_plan.cpp) and the
// sm_100a kernels (qtn_kernels.cu).  Not part of the C ABI.
#pragma once

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/qtn_b200.h"
#include "qtn_stream.h"

#include <cuda_runtime_api.h>

namespace qtn {

// Function attributes (dynamic shared-memory opt-in) are per device: a
// one-time setup flag is a bit per device ordinal, not a process-wide bool,
// so a process that later launches on another GPU sets them there too.
inline uint64_t current_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}
inline bool needs_setup(const std::atomic<uint64_t>& seen) {
  return !(seen.load(std::memory_order_acquire) & current_device_bit());
}
inline void mark_setup(std::atomic<uint64_t>& seen) {
  seen.fetch_or(current_device_bit(), std::memory_order_release);
}

// ---------------------------------------------------------------- bit runs
// An operand's flat index is a bit-gather of the output index o:
//   idx(o, v) = sum_k ((o >> src_k) & (2^len_k - 1)) << dst_k  +  v << vshift
// Consecutive variables that sit on consecutive bits of both o and the
// operand collapse into one run, so an operand aligned with the output
// (the primary operand) costs two runs.  Packed as src | dst<<8 | len<<16.
inline uint32_t pack_run(uint32_t src, uint32_t dst, uint32_t len) {
  return src | (dst << 8) | (len << 16);
}

constexpr int kMaxRuns = 32;   // >= max rank handled (w <= 32)
constexpr int kMaxG = 8;       // streamed/gathered operands per bucket
constexpr int kMaxT = 4;       // smem lookup tables per bucket
constexpr int kMaxTOps = 24;   // small operands folded into tables
constexpr int kTBits = 8;      // non-v bits per lookup table
constexpr int kTileBits = 12;  // output elements per tile = 2^kTileBits

struct GOpArg {                // operand read from global memory
  const void* ptr;
  uint32_t vshift;             // bit of v in the operand index
  uint32_t c64;
  uint32_t n_lo, n_hi;         // runs on tile-local bits / on tile bits
  uint32_t lo[kMaxRuns];
  uint32_t hi[kMaxRuns];
};

struct TOpArg {                // small operand folded into a table
  const void* ptr;
  uint32_t vshift;
  uint32_t c64;
  uint32_t n_runs;
  uint32_t runs[kTBits];       // table-index bits -> operand index bits
};

struct TableArg {
  uint32_t nbits;              // table has 2^(nbits+1) entries (v is the LSB)
  uint32_t n_lo, n_hi;
  uint32_t lo[kTBits];         // output bits -> table index (tile-local part)
  uint32_t hi[kTBits];
  uint32_t first_op, n_ops;
  uint32_t smem_off;           // in complex128 entries
};

struct BucketArgs {
  void* out;
  uint64_t n_out;              // 2^R
  uint32_t R;
  uint32_t out_c64;
  uint32_t primary;            // op 0 is aligned with the output low bits
  uint32_t p_k;                // bit position of v in the primary operand
  uint32_t ng, nt, ntop;
  uint32_t table_entries;      // total smem table entries
  GOpArg g[kMaxG];
  TableArg t[kMaxT];
  TOpArg top[kMaxTOps];
};

// ---------------------------------------------------- SMEM executor program
// One network = one warp.  Program blob, 16-byte aligned sections:
//   SmemHeader | SmemBucket[n_buckets] | SmemOp[n_ops] | u16 scalars[n_scalars]
// All offsets are complex128-element offsets into the warp's data region
// (packed inputs first, then the intermediate arena).
struct SmemHeader {
  uint32_t n_buckets;
  uint32_t n_ops;
  uint32_t n_scalars;
  uint32_t pow2;               // number of empty buckets (factor 2 each)
  uint32_t in_elems;           // packed input elements (complex128)
  uint32_t data_elems;         // inputs + arena
  uint32_t prog_bytes;         // whole blob, multiple of 16
  uint32_t gen_off;            // byte offset of the generator section (0: none)
  uint32_t n_params;           // generator: distinct gate parameters
  uint32_t n_recs;             // generator: one record per input tensor ENTRY
  uint32_t tab_off;            // byte offset of the u16 gather tables
  uint32_t in_off;             // byte offset of the SmemIn records
  uint32_t n_init;             // leading SmemIn records materialised before bucket 0
  uint32_t n_init_gen;         // leading generator entries materialised before bucket 0
  uint32_t pad[2];
};
// Generator section (appended by qtn_batch_set_recipes): the warp builds its
// own input tensors in shared memory from the angles of its set — the
// on-device form of gate_matrix + slicing (circuit.py:186-205,
// network.py:153-165) fused into the executor.
struct SmemGenParam {          // phase e^{-i t}, t = scale*angles[angle] + offset
  double scale;
  double offset;
  int32_t angle;               // -1: constant t = offset; -2: literal value (scale + i*offset)
  int32_t pad;
};
struct SmemGenRec {            // one tensor ENTRY (entries of all inputs, flattened)
  uint16_t sm_off;             // element offset in the warp's data region
  uint8_t kind;                // QTN_GATE_*
  uint8_t full;                // index into the unsliced gate tensor
  uint8_t param;               // parameter slot
  uint8_t pad[3];
};
static_assert(sizeof(SmemGenParam) == 24, "gen param");
static_assert(sizeof(SmemGenRec) == 8, "gen rec");
struct SmemBucket {
  uint16_t out_off;
  uint8_t R;
  uint8_t n_ops;
  uint16_t first_op;
  uint16_t first_in;           // input tensors materialised just before this bucket
  uint8_t n_in;
  uint8_t pad0;
  uint16_t first_gen;          // ... as generator entries (set by qtn_batch_set_recipes)
  uint16_t n_gen;
  uint8_t pad[2];
};
// An input tensor is generated (or copied) into shared memory right before
// the bucket that consumes it (every input is consumed exactly once), so it
// occupies smem only for that bucket: the data region holds the live
// intermediates plus one bucket's inputs, not the whole network.
struct SmemIn {
  uint16_t input;              // input tensor index (generator record / packed input)
  uint16_t sm_off;             // destination element offset in the data region
  uint16_t in_off;             // element offset in the packed input (copy path)
  uint8_t rank;
  uint8_t pad;
};
static_assert(sizeof(SmemIn) == 8, "in");
// Operand of a bucket: element e of the output reads
//   D[off + tab[lo + (e & 31)] + (R > 5 ? tab[hi + (e >> 5)] : 0) (+ vstep for v=1)]
// where tab is the program's u16 gather table (the bit gather of the output
// index, precomputed at plan time; gathers are OR-linear, so the 5 low and
// the R-5 high output bits are tabulated separately).
constexpr int kSmemMaxR = 10;
struct SmemOp {
  uint16_t off;
  uint16_t vstep;
  uint16_t lo;                 // u16 index of the low-bits table (32 entries or 2^R)
  uint16_t hi;                 // u16 index of the high-bits table (2^(R-5) entries)
};
static_assert(sizeof(SmemHeader) == 64, "header");
static_assert(sizeof(SmemBucket) == 16, "bucket");
static_assert(sizeof(SmemOp) == 8, "op");

// ------------------------------------------------------------- host plan
struct TensorRec {
  std::vector<int32_t> vars;   // layout, most significant first
  bool input = false;
  int64_t in_off = 0;          // packed-input element offset (inputs)
  int64_t ws_off = -1;         // workspace byte offset (HBM intermediates)
  int64_t sm_off = -1;         // SMEM data-region element offset
  bool c64 = false;            // storage type (HBM intermediates)
  int32_t born = -1;           // bucket index that produces it (-1: input)
  int32_t last_use = -1;       // bucket index that consumes it (n: final fold)
  int rank() const { return (int)vars.size(); }
};

// A chain of single-operand buckets fused into one multi-variable sum
// (HBM executor): out[o] = sum over the k eliminated bits of src.
constexpr int kMaxRed = 12;
struct RedRec {
  int32_t level = 0;
  uint64_t src = 0, out = 0;   // tagged pointers (qtn_stream.h)
  uint8_t src_c64 = 0, out_c64 = 0, R = 0, k = 0;
  uint8_t pos[kMaxRed] = {};   // eliminated bit positions in src's index, ascending
};

struct BucketRec {
  int32_t v;
  std::vector<int32_t> ops;    // tensor ids, ascending (reference order)
  int32_t primary;             // index into ops
  int32_t out;                 // tensor id of the result
  int32_t rank;                // output rank
};

}  // namespace qtn

struct qtn_plan {
  std::vector<qtn::TensorRec> tensors;   // inputs, then intermediates
  std::vector<qtn::BucketRec> buckets;
  std::vector<int32_t> step_ranks;       // per order entry
  std::vector<int32_t> scalars;          // rank-0 tensors folded at the end
  int32_t n_inputs = 0;
  int32_t n_empty = 0;
  int32_t width = 0;
  int32_t executor = QTN_EXEC_HBM;
  int32_t dtype = QTN_DTYPE_C128;        // requested storage policy
  int64_t input_elems = 0;
  int64_t workspace_bytes = 0;
  int64_t smem_bytes = 0;
  double alg_bytes = 0.0;
  double exec_bytes = -1.0;              // < 0: equal to alg_bytes (no fusion)
  double flops_sum = 0.0;
  std::vector<uint8_t> program;          // SMEM executor blob
  // HBM executor: one streaming descriptor per bucket (tagged pointers
  // relative to the network's input block / workspace), its level in the
  // elimination tree (level-synchronous execution) and its tile count.
  std::vector<uint8_t> hbm_desc;
  std::vector<uint64_t> hbm_desc_off;
  std::vector<int32_t> hbm_level;        // -1: absorbed into a fused reduction
  std::vector<qtn::RedRec> hbm_red;      // fused single-operand chains
  std::vector<uint64_t> hbm_tiles;
  std::vector<int32_t> hbm_xidx;         // expanding-bucket descriptor per bucket, or -1
  std::vector<qtn::XDesc> hbm_xdesc;
  std::vector<qtn::YDesc> hbm_ydesc;     // expanding bucket + consumer pairs (qtn_xt.cu)
  std::vector<int32_t> hbm_ylevel;       // their levels
  std::vector<qtn::WsDesc> hbm_wsdesc;   // weighted full sums: the tail chains (qtn_wsum.cu)
  std::vector<int32_t> hbm_wslevel;      // their levels
  std::vector<int32_t> hbm_r1idx;        // single-operand (trace) record per bucket, or -1
  std::vector<qtn::R1Dev> hbm_r1;        // net = 0 here; set per batch
  struct SubRec {                        // tiny subtree (qtn_stream.h SubItem)
    int32_t level;
    uint32_t first, count, smem;         // member descriptors hbm_sub_desc[first .. +count)
  };
  std::vector<SubRec> hbm_sub;
  std::vector<uint64_t> hbm_sub_desc;    // member descriptor byte offsets (hbm_desc), in order
  std::vector<qtn::FDesc> hbm_fdesc;     // fused product chains (qtn_fused.cu)
  std::vector<int32_t> hbm_flevel;       // their levels
  std::vector<uint8_t> hbm_wblob;        // warp-granular forms of the fused chains (qtn_fusedw.cu)
  std::vector<int64_t> hbm_woff;         // per fused chain: its blob offset, or -1 (CTA kernel only)
  std::vector<uint32_t> hbm_wwarps;      // per fused chain: warps of one set (0: none)
  int32_t n_levels = 0;
  // Set-major form of an SMEM-eligible network (qtn_setmajor.cu): angle
  // sets are the fastest-varying dimension of every tensor in HBM, one
  // region per intermediate (no reuse: buckets of a level run concurrently),
  // input tensors generated on the fly.
  struct SMOpRec {
    int32_t input;                       // input tensor index, or -1
    uint32_t off;                        // data-region element offset (intermediates)
    std::vector<uint16_t> idx;           // per output element e: v=0, v=1 operand element
  };
  struct SMBucketRec {
    int32_t level;
    uint32_t out_off;
    int32_t R;
    std::vector<SMOpRec> ops;            // primary first
  };
  std::vector<SMBucketRec> sm_buckets;
  uint32_t sm_elems = 0;                 // data-region elements (intermediates)
  std::vector<uint32_t> sm_scalar_off;   // rank-0 intermediates folded at the end
  std::vector<int32_t> sm_scalar_in;     // rank-0 inputs folded at the end
  int32_t sm_levels = 0;
  qtn_batch* self_batch = nullptr;       // device copy for single-plan runs
  ~qtn_plan();
};

namespace qtn {
void set_error(const std::string& msg);
// device-side launchers (qtn_kernels.cu)
int launch_bucket(const BucketArgs& a, void* stream);
int launch_fold(const void* const* ptrs, const uint8_t* c64, int n, int pow2,
                void* result, bool accumulate, void* stream);
int device_alloc(void** p, size_t bytes);
int device_free(void* p);
int h2d(void* dst, const void* src, size_t bytes);
int device_check();
// pure host helpers (qtn_plan.cpp)
void make_runs(const std::vector<std::pair<int, int>>& src_dst, std::vector<uint32_t>& runs);
}  // namespace qtn
