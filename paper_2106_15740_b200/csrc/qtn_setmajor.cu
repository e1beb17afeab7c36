// Set-major executor (sm_100a): many small networks x many angle sets.
//
// The QAOA loop evaluates the same networks at many angle vectors.  Here the
// angle-set index is made the fastest-varying dimension of every tensor:
// element x of network n for set s lives at ws[(base_n + x) * A + s].  A
// bucket  out[e][s] = sum_v prod_t T_t[idx_t(e, v)][s]
// (contraction.py:42-54, 90-96) then reads and writes 32 consecutive sets
// per warp — fully coalesced 512-byte rows — and every (bucket, element) is
// one CTA streaming the A sets.  All buckets of one level of the elimination
// trees of every network run in one launch (level-synchronous; each
// intermediate has its own region, so concurrent buckets never alias).
// Input tensors are never stored: an operand that is a gate tensor is
// generated on the fly from its gate kind, the entry's index in the unsliced
// gate (slicing resolved at build time, network.py:153-165) and the set's
// phase e^{-i t} for the gate's angle (circuit.py:186-205), read from a
// [param][set] phase table computed once per evaluation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "qtn_setmajor.h"

namespace qtn {

struct SMOpDev {
  uint32_t tab;     // u16 table index: 2 entries per output element (v = 0, 1)
  uint32_t off;     // data-region offset (intermediates)
  uint8_t gen;      // 1: generated gate tensor
  uint8_t kind;     // QTN_GATE_* (gen)
  uint16_t param;   // phase-table row (gen)
  uint32_t pad;
};
struct SMBucketDev {
  uint32_t net;
  uint32_t out_off;
  uint32_t first_op;
  uint8_t R, n_ops;
  uint16_t pad;
};
static_assert(sizeof(SMOpDev) == 16 && sizeof(SMBucketDev) == 16, "sm layouts");

struct SMParam {
  double scale, offset;
  int32_t angle;  // -1 constant, -2 literal (scale + i offset)
  int32_t pad;
};

// Fused form: one warp evaluates one network for a tile of S = 2^sh sets,
// every intermediate in shared memory ([element][set], liveness-packed).
struct SMFNet {
  uint32_t first_bk, n_bk;
  uint32_t first_par, n_par;   // net-local phase slots
  uint32_t first_sc, n_sc;     // rank-0 intermediates (data offsets)
  uint32_t first_sg, n_sg;     // rank-0 gate inputs (kind | idx << 8 | slot << 16)
  double2 cst;
  uint32_t sh;                 // log2 sets per warp
  int32_t gidx;
  uint32_t n_elems;            // peak live data elements
  uint32_t pad;
};
struct SMFBucket {
  uint32_t out_off, first_op;
  uint16_t R, n_ops;
  uint32_t pad;
};
static_assert(sizeof(SMFNet) == 64 && sizeof(SMFBucket) == 16, "smf layouts");

struct SetMajor {
  int32_t n_nets = 0, n_total = 0, n_levels = 0;
  uint64_t total_elems = 0;
  std::vector<uint32_t> level_blocks;  // CTAs per level
  std::vector<uint32_t> level_rec;     // first CTA record of each level
  uint32_t* d_recs = nullptr;          // kRecWords per CTA (see sm_level_kernel)
  // bucket-tile form (sm_bucket_kernel)
  std::vector<uint32_t> level_bk;      // buckets per level
  std::vector<uint32_t> level_bk_first;
  uint32_t* d_brec = nullptr;          // variable-size bucket records
  uint32_t* d_brec_off = nullptr;      // word offset of each bucket's record (level-major)
  uint32_t* d_btab = nullptr;          // per (operand, element) index pair / coefficient codes
  uint64_t* d_base = nullptr;
  SMParam* d_params = nullptr;
  int32_t n_params = 0;
  double2* d_const = nullptr;          // per net: 2^n_empty * rank-0 inputs
  uint32_t* d_scal_first = nullptr;
  uint32_t* d_scal_off = nullptr;
  uint32_t* d_sgen_first = nullptr;    // per net: rank-0 gate inputs (all vars sliced)
  uint32_t* d_sgen = nullptr;          // kind | full index << 8 | param << 16
  int32_t* d_gidx = nullptr;
  // fused form
  bool fused_ok = false;
  int64_t f_smem = 0;                  // dynamic shared memory per warp-CTA
  std::vector<uint32_t> f_sh;          // per fused net (unit order)
  SMFNet* d_fnets = nullptr;
  SMFBucket* d_fbk = nullptr;
  SMOpDev* d_fops = nullptr;
  uint32_t* d_ftabs = nullptr;
  SMParam* d_fpar = nullptr;
  uint32_t* d_fsc = nullptr;
  uint32_t* d_fsg = nullptr;
  std::map<int32_t, std::pair<uint32_t*, uint32_t>> f_prefix;  // n_sets -> (unit prefix, units)
};

static bool fused_on(const SetMajor* S) {
  const char* v = getenv("QTN_SETMAJOR_FUSED");
  return S->fused_ok && v && v[0] == '1';  // opt-in: slower than the level form on config 2/3
}

namespace {

constexpr int kMaxOps = 8;  // operands per bucket in the set-major form

// Gate entry as an affine form of the phase ph = e^{-i t}:
// entry = (a + u * ph.x, w * ph.y)  (host mirror of gate_entry below).
struct GateCoef {
  double a, u, w;
};
GateCoef gate_coef(uint32_t kind, uint32_t i) {
  const double s = 0.70710678118654757;
  const uint32_t row = i >> 2, col = i & 3;
  switch (kind) {
    case QTN_GATE_INIT: return {i == 0 ? 1.0 : 0.0, 0.0, 0.0};
    case QTN_GATE_H: return {i == 3 ? -s : s, 0.0, 0.0};
    case QTN_GATE_ZPOW: return i == 0 ? GateCoef{1.0, 0.0, 0.0} : (i == 3 ? GateCoef{0.0, 1.0, 1.0} : GateCoef{0.0, 0.0, 0.0});
    case QTN_GATE_ZPOW_DIAG: return i == 0 ? GateCoef{1.0, 0.0, 0.0} : GateCoef{0.0, 1.0, 1.0};
    case QTN_GATE_XPOW: return (i == 0 || i == 3) ? GateCoef{0.5, 0.5, 0.5} : GateCoef{0.5, -0.5, -0.5};
    case QTN_GATE_CNOT: return {col == (row < 2 ? row : (row ^ 1)) ? 1.0 : 0.0, 0.0, 0.0};
    case QTN_GATE_ZZ:
      if (row != col) return {0.0, 0.0, 0.0};
      return (row == 0 || row == 3) ? GateCoef{0.0, 1.0, -1.0} : GateCoef{0.0, 1.0, 1.0};
    case QTN_GATE_ZZ_DIAG: return (i == 0 || i == 3) ? GateCoef{0.0, 1.0, -1.0} : GateCoef{0.0, 1.0, 1.0};
    case QTN_GATE_SCALAR: return {0.0, 1.0, 1.0};
  }
  return {0.0, 0.0, 0.0};
}

// the distinct affine forms gate_coef produces (kGateCoef on device)
constexpr int kNumCoef = 8;
const double kCoefHost[kNumCoef][3] = {
    {0.0, 0.0, 0.0}, {1.0, 0.0, 0.0}, {0.70710678118654757, 0.0, 0.0},
    {-0.70710678118654757, 0.0, 0.0}, {0.0, 1.0, 1.0}, {0.0, 1.0, -1.0},
    {0.5, 0.5, 0.5}, {0.5, -0.5, -0.5}};
int coef_code(const GateCoef& c) {
  for (int i = 0; i < kNumCoef; ++i)
    if (kCoefHost[i][0] == c.a && kCoefHost[i][1] == c.u && kCoefHost[i][2] == c.w) return i;
  return -1;
}

template <typename T>
int upload_vec(T** dst, const std::vector<T>& v) {
  int rc = device_alloc((void**)dst, std::max<size_t>(v.size(), 1) * sizeof(T));
  if (rc) return rc;
  if (!v.empty()) rc = h2d(*dst, v.data(), v.size() * sizeof(T));
  return rc;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// Gate entry from the phase ph = e^{-i t} (same conventions as the SMEM
// executor's generator).
__device__ __forceinline__ double2 gate_entry(uint32_t kind, uint32_t i, double2 ph) {
  const double s = 0.70710678118654757;
  switch (kind) {
    case QTN_GATE_INIT: return make_double2(i == 0 ? 1.0 : 0.0, 0.0);
    case QTN_GATE_H: return make_double2(i == 3 ? -s : s, 0.0);
    case QTN_GATE_ZPOW: return i == 0 ? make_double2(1.0, 0.0) : (i == 3 ? ph : make_double2(0.0, 0.0));
    case QTN_GATE_ZPOW_DIAG: return i == 0 ? make_double2(1.0, 0.0) : ph;
    case QTN_GATE_XPOW: {
      const bool d = (i == 0 || i == 3);
      return d ? make_double2(0.5 * (1.0 + ph.x), 0.5 * ph.y)
               : make_double2(0.5 * (1.0 - ph.x), -0.5 * ph.y);
    }
    case QTN_GATE_CNOT: {
      const uint32_t row = i >> 2, col = i & 3;
      return make_double2(col == (row < 2 ? row : (row ^ 1)) ? 1.0 : 0.0, 0.0);
    }
    case QTN_GATE_ZZ: {
      const uint32_t row = i >> 2, col = i & 3;
      if (row != col) return make_double2(0.0, 0.0);
      return (row == 0 || row == 3) ? make_double2(ph.x, -ph.y) : ph;
    }
    case QTN_GATE_ZZ_DIAG: return (i == 0 || i == 3) ? make_double2(ph.x, -ph.y) : ph;
    case QTN_GATE_SCALAR: return ph;
  }
  return make_double2(0.0, 0.0);
}

__device__ __forceinline__ double2 phase_of(const SMParam& q, const double* __restrict__ row) {
  if (q.angle == -2) return make_double2(q.scale, q.offset);
  const double t = q.angle >= 0 ? q.scale * row[q.angle] + q.offset : q.offset;
  double sn, cs;
  sincos(t, &sn, &cs);
  return make_double2(cs, -sn);
}

// Fused set-major executor: one 32-thread CTA = one (network, tile of S sets).
// Lane = (group g, set s); the G = 32/S groups split each bucket's output
// elements, the S lanes of a group read/write S consecutive sets of one
// element (S*16 contiguous bytes of shared memory).
__global__ void __launch_bounds__(32) smf_kernel(
    const SMFNet* __restrict__ nets, const uint32_t* __restrict__ prefix, int n_nets,
    const SMFBucket* __restrict__ bks, const SMOpDev* __restrict__ ops,
    const uint32_t* __restrict__ tabs, const SMParam* __restrict__ par,
    const uint32_t* __restrict__ sc, const uint32_t* __restrict__ sg,
    const double* __restrict__ angles, int n_angles, int A, int n_total,
    double2* __restrict__ results) {
  extern __shared__ double2 smf[];
  const uint32_t u = blockIdx.x;
  uint32_t lo = 0, hi = n_nets;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= u) lo = mid;
    else hi = mid;
  }
  const SMFNet& net = nets[lo];
  const uint32_t sh = net.sh, S = 1u << sh, G = 32u >> sh;
  const uint32_t lane = threadIdx.x, s = lane & (S - 1), g = lane >> sh;
  const int set = (int)((u - prefix[lo]) * S + s);
  const bool valid = set < A;
  const double* row = angles + (int64_t)(valid ? set : A - 1) * n_angles;
  double2* ph = smf;
  double2* data = smf + net.n_par * S;
  for (uint32_t p = g; p < net.n_par; p += G) ph[p * S + s] = phase_of(par[net.first_par + p], row);
  __syncwarp();
  for (uint32_t b = 0; b < net.n_bk; ++b) {
    const SMFBucket bk = bks[net.first_bk + b];
    const uint32_t ne = 1u << bk.R;
    for (uint32_t e = g; e < ne; e += G) {
      double2 a0, a1;
      for (uint32_t k = 0; k < bk.n_ops; ++k) {
        const SMOpDev o = ops[bk.first_op + k];
        const uint32_t t = __ldg(tabs + o.tab + e);
        const uint32_t i0 = t & 0xffffu, i1 = t >> 16;
        double2 x, y;
        if (o.gen) {
          const double2 pp = ph[o.param * S + s];
          x = gate_entry(o.kind, i0, pp);
          y = gate_entry(o.kind, i1, pp);
        } else {
          x = data[(o.off + i0) * S + s];
          y = data[(o.off + i1) * S + s];
        }
        if (k == 0) {
          a0 = x;
          a1 = y;
        } else {
          a0 = cmul(a0, x);
          a1 = cmul(a1, y);
        }
      }
      data[(bk.out_off + e) * S + s] = make_double2(a0.x + a1.x, a0.y + a1.y);
    }
    __syncwarp();
  }
  if (g == 0 && valid) {
    double2 r = net.cst;
    for (uint32_t k = 0; k < net.n_sc; ++k) r = cmul(r, data[sc[net.first_sc + k] * S + s]);
    for (uint32_t k = 0; k < net.n_sg; ++k) {
      const uint32_t q = sg[net.first_sg + k];
      r = cmul(r, gate_entry(q & 0xff, (q >> 8) & 0xff, ph[(q >> 16) * S + s]));
    }
    results[(int64_t)set * n_total + net.gidx] = r;
  }
}

__global__ void sm_phase_kernel(const SMParam* __restrict__ par, int n_params,
                                const double* __restrict__ angles, int n_angles, int A,
                                double2* __restrict__ ph) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (s >= A || k >= n_params) return;
  const SMParam q = par[k];
  double2 r;
  if (q.angle == -2) {
    r = make_double2(q.scale, q.offset);
  } else {
    const double t = q.angle >= 0 ? q.scale * angles[(int64_t)s * n_angles + q.angle] + q.offset
                                  : q.offset;
    double sn, cs;
    sincos(t, &sn, &cs);
    r = make_double2(cs, -sn);
  }
  ph[(int64_t)k * A + s] = r;
}

// ---- level kernel
// One CTA per (bucket, output element e) of a level; 256 threads stream the
// sets, J per thread per pass.  Everything the CTA needs is one fixed-size
// record (a single dependent load): word 0 = absolute output element, word 1 =
// operand count, then per operand two words —
//   intermediate: absolute elements of entries idx(e, v=0) and idx(e, v=1);
//   gate        : 0x80000000 | phase row, and the affine-coefficient codes of
//                 its two entries (code0 | code1 << 8, see kGateCoef).
// The operand loop stays rolled (~31-48 registers, full occupancy): the L2
// round trip of each operand is hidden by resident warps, not by unrolling.
constexpr int kRecWords = 2 + 2 * kMaxOps;

__constant__ double kGateCoef[kNumCoef][3];

struct OpSetup {
  const double2* px;  // intermediate: row of entry v=0; gate: phase row
  const double2* py;  // intermediate: row of entry v=1
  double c[6];        // gate: (a, u, w) for v = 0, 1
  int gen;
  int pad;
};

// per-iteration shared-memory reads (asm volatile: not hoisted out of the set
// loop, which would pin every operand's setup in registers)
__device__ __forceinline__ uint64_t lds_u64(const void* p) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ double lds_f64(const void* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

// grid.y > 1 (levels with few CTAs): CTA y covers sets [y*256*J, (y+1)*256*J).
struct OpRow {
  uint64_t ox, oy;  // row starts (double2 units): intermediates in ws, gates in ph
  double c[6];      // gate: (a, u, w) for v = 0, 1
  int gen;
  int pad;
};

__device__ __forceinline__ int lds_s32(const void* p) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

// Values of operand k at sets s0 + 256 j (0 beyond A).  Rows read here were
// written by earlier launches only, hence the non-coherent path (__ldg).
template <int J, bool FULL>
__device__ __forceinline__ void load_operand(const OpRow* su, int k, int s0, int A,
                                             const double2* __restrict__ ph,
                                             const double2* ws, double2 (&x)[J],
                                             double2 (&y)[J]) {
  const uint64_t ox = lds_u64(&su[k].ox);
  if (lds_s32(&su[k].gen)) {
    const double* c = su[k].c;
    const double c0 = lds_f64(c), c1 = lds_f64(c + 1), c2 = lds_f64(c + 2);
    const double c3 = lds_f64(c + 3), c4 = lds_f64(c + 4), c5 = lds_f64(c + 5);
    const double2* pp = ph + ox;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int s = s0 + 256 * j;
      const double2 p = (J == 1 || FULL || s < A) ? __ldg(pp + s) : make_double2(0.0, 0.0);
      x[j] = make_double2(fma(c1, p.x, c0), c2 * p.y);
      y[j] = make_double2(fma(c4, p.x, c3), c5 * p.y);
    }
  } else {
    const double2* px = ws + ox;
    const double2* py = ws + lds_u64(&su[k].oy);
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const int s = s0 + 256 * j;
      const bool ok = J == 1 || FULL || s < A;
      x[j] = ok ? __ldg(px + s) : make_double2(0.0, 0.0);
      y[j] = ok ? __ldg(py + s) : make_double2(0.0, 0.0);
    }
  }
}

// FULL: A is a multiple of 256 * J * gridDim.y (no per-set bounds checks)
template <int J, bool FULL>
__global__ void __launch_bounds__(256) sm_level_kernel(const uint32_t* __restrict__ recs,
                                                       const double2* __restrict__ ph,
                                                       double2* ws, int A) {
  __shared__ OpRow su[kMaxOps];
  const uint32_t* r = recs + (size_t)blockIdx.x * kRecWords;
  const uint2 hd = *reinterpret_cast<const uint2*>(r);
  const int n = (int)hd.y;
  if (threadIdx.x < n) {
    const uint2 w = reinterpret_cast<const uint2*>(r + 2)[threadIdx.x];
    OpRow& u = su[threadIdx.x];
    if (w.x & 0x80000000u) {
      u.gen = 1;
      u.ox = u.oy = (uint64_t)(w.x & 0x7fffffffu) * A;
      const uint32_t c0 = w.y & 0xff, c1 = w.y >> 8;
      for (int i = 0; i < 3; ++i) {
        u.c[i] = kGateCoef[c0][i];
        u.c[3 + i] = kGateCoef[c1][i];
      }
    } else {
      u.gen = 0;
      u.ox = (uint64_t)w.x * A;
      u.oy = (uint64_t)w.y * A;
    }
  }
  __syncthreads();
  double2* out = ws + (size_t)hd.x * A;
  const int s_step = 256 * J * gridDim.y;
#pragma unroll 1
  for (int s0 = blockIdx.y * 256 * J + threadIdx.x; s0 < A; s0 += s_step) {
    double2 a0[J], a1[J];
    load_operand<J, FULL>(su, 0, s0, A, ph, ws, a0, a1);
#pragma unroll 1
    for (int k = 1; k < n; ++k) {
      double2 x[J], y[J];
      load_operand<J, FULL>(su, k, s0, A, ph, ws, x, y);
#pragma unroll
      for (int j = 0; j < J; ++j) {
        a0[j] = cmul(a0[j], x[j]);
        a1[j] = cmul(a1[j], y[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (FULL || s0 + 256 * j < A) out[s0 + 256 * j] = make_double2(a0[j].x + a1[j].x, a0[j].y + a1[j].y);
  }
}

// Software-pipelined variant: the (set pass, operand) steps of a thread form
// one flattened sequence and the loads of step t+1 are issued before step t
// is multiplied in, so a warp pays roughly one L2/DRAM round trip per CTA
// instead of one per operand.  grid.y > 1 splits the sets over CTAs.
__global__ void __launch_bounds__(256) sm_level_pipe_kernel(const uint32_t* __restrict__ recs,
                                                            const double2* __restrict__ ph,
                                                            double2* ws, int A) {
  __shared__ OpSetup su[kMaxOps];
  const uint32_t* r = recs + (size_t)blockIdx.x * kRecWords;
  const uint2 hd = *reinterpret_cast<const uint2*>(r);
  const int n = (int)hd.y;
  if (threadIdx.x < n) {
    const uint2 w = reinterpret_cast<const uint2*>(r + 2)[threadIdx.x];
    OpSetup& u = su[threadIdx.x];
    if (w.x & 0x80000000u) {
      u.gen = 1;
      u.px = u.py = ph + (size_t)(w.x & 0x7fffffffu) * A;
      const uint32_t c0 = w.y & 0xff, c1 = w.y >> 8;
      for (int i = 0; i < 3; ++i) {
        u.c[i] = kGateCoef[c0][i];
        u.c[3 + i] = kGateCoef[c1][i];
      }
    } else {
      u.gen = 0;
      u.px = ws + (size_t)w.x * A;
      u.py = ws + (size_t)w.y * A;
    }
  }
  __syncthreads();
  double2* out = ws + (size_t)hd.x * A;
  const int s_first = blockIdx.y * 256 + threadIdx.x, s_step = 256 * gridDim.y;
  if (s_first >= A) return;
  const int passes = (A - 1 - s_first) / s_step + 1;
  const int steps = passes * n;
  // step t: set s_first + (t / n) * s_step, operand t % n
  int k = 0, s = s_first;
  double2 r0 = reinterpret_cast<const double2*>(lds_u64(&su[0].px))[s];
  double2 r1 = su[0].gen ? r0 : reinterpret_cast<const double2*>(lds_u64(&su[0].py))[s];
  double2 a0 = make_double2(1.0, 0.0), a1 = a0;
#pragma unroll 1
  for (int t = 0; t < steps; ++t) {
    // prefetch step t + 1
    int kn = k + 1, sn = s;
    if (kn == n) {
      kn = 0;
      sn += s_step;
    }
    double2 q0 = r0, q1 = r1;
    if (t + 1 < steps) {
      q0 = reinterpret_cast<const double2*>(lds_u64(&su[kn].px))[sn];
      if (!su[kn].gen) q1 = reinterpret_cast<const double2*>(lds_u64(&su[kn].py))[sn];
    }
    double2 x = r0, y = r1;
    if (su[k].gen) {
      const double* c = su[k].c;
      y = make_double2(fma(lds_f64(c + 4), r0.x, lds_f64(c + 3)), lds_f64(c + 5) * r0.y);
      x = make_double2(fma(lds_f64(c + 1), r0.x, lds_f64(c + 0)), lds_f64(c + 2) * r0.y);
    }
    if (k == 0) {
      a0 = x;
      a1 = y;
    } else {
      a0 = cmul(a0, x);
      a1 = cmul(a1, y);
    }
    if (k == n - 1) out[s] = make_double2(a0.x + a1.x, a0.y + a1.y);
    k = kn;
    s = sn;
    r0 = q0;
    r1 = q1;
  }
}

// ---- bucket-tile kernel
// One CTA per (bucket, tile of kTile = 64 sets); 256 threads = 4 element
// groups x 64 sets.  Operands whose rows are reused across the bucket's
// output elements (every intermediate of rank < R + 1, every gate's phase
// row) are staged once into shared memory for the tile; full-rank operands
// (each row read once) stream from L2/HBM.  This removes the L2 re-reads of
// the per-element form (one CTA per output element re-fetching shared rows).
// Record (u32 words, 16-byte aligned): [0] first output element (absolute),
// [1] R | n_ops << 8, [2..3] pad, then per operand a uint4:
//   x = mode << 30 | v   mode 0 stream: v = absolute base element
//                        mode 1 staged: v = first shared-memory row
//                        mode 2 gate  : v = shared-memory row of its phase
//   y = staged: absolute base element; gate: phase-table row
//   z = staged: rows
//   w = word offset of its per-element table in btab
//       (intermediates: i0 | i1 << 16; gates: code0 | code1 << 8)
constexpr int kTile = 64;
constexpr int64_t kStageBudget = 32 * 1024;

__global__ void __launch_bounds__(256) sm_bucket_kernel(const uint32_t* __restrict__ brec,
                                                        const uint32_t* __restrict__ boff,
                                                        const uint32_t* __restrict__ btab,
                                                        const double2* __restrict__ ph,
                                                        double2* ws, int A) {
  extern __shared__ double2 stg[];
  __shared__ uint4 od[kMaxOps];
  const uint32_t* r = brec + boff[blockIdx.x];
  const uint2 hd = *reinterpret_cast<const uint2*>(r);
  const uint32_t R = hd.y & 0xff;
  const int n = (int)((hd.y >> 8) & 0xff);
  if (threadIdx.x < n) od[threadIdx.x] = reinterpret_cast<const uint4*>(r + 4)[threadIdx.x];
  __syncthreads();
  const int s0 = blockIdx.y * kTile;
  for (int k = 0; k < n; ++k) {
    const uint4 o = od[k];
    const uint32_t mode = o.x >> 30, dst = o.x & 0x3fffffffu;
    if (mode == 1) {
      for (uint32_t i = threadIdx.x; i < o.z * kTile; i += 256) {
        const uint32_t row = i / kTile, c = i % kTile;
        const int s = s0 + (int)c;
        stg[(dst + row) * kTile + c] = s < A ? ws[(size_t)(o.y + row) * A + s] : make_double2(0.0, 0.0);
      }
    } else if (mode == 2) {
      if (threadIdx.x < kTile) {
        const int s = s0 + (int)threadIdx.x;
        stg[dst * kTile + threadIdx.x] = s < A ? ph[(size_t)o.y * A + s] : make_double2(0.0, 0.0);
      }
    }
  }
  __syncthreads();
  const uint32_t c = threadIdx.x % kTile, g = threadIdx.x / kTile;
  const int s = s0 + (int)c;
  const bool valid = s < A;
  const uint32_t ne = 1u << R;
#pragma unroll 1
  for (uint32_t e = g; e < ne; e += 256 / kTile) {
    double2 a0 = make_double2(1.0, 0.0), a1 = a0;
#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      const uint4 o = od[k];
      const uint32_t t = __ldg(btab + o.w + e);
      const uint32_t mode = o.x >> 30, v = o.x & 0x3fffffffu;
      double2 x, y;
      if (mode == 0) {
        x = valid ? ws[(size_t)(v + (t & 0xffffu)) * A + s] : make_double2(0.0, 0.0);
        y = valid ? ws[(size_t)(v + (t >> 16)) * A + s] : make_double2(0.0, 0.0);
      } else if (mode == 1) {
        x = stg[(v + (t & 0xffffu)) * kTile + c];
        y = stg[(v + (t >> 16)) * kTile + c];
      } else {
        const double2 p = stg[v * kTile + c];
        const uint32_t c0 = t & 0xff, c1 = (t >> 8) & 0xff;
        x = make_double2(fma(kGateCoef[c0][1], p.x, kGateCoef[c0][0]), kGateCoef[c0][2] * p.y);
        y = make_double2(fma(kGateCoef[c1][1], p.x, kGateCoef[c1][0]), kGateCoef[c1][2] * p.y);
      }
      if (k == 0) {
        a0 = x;
        a1 = y;
      } else {
        a0 = cmul(a0, x);
        a1 = cmul(a1, y);
      }
    }
    if (valid) ws[(size_t)(hd.x + e) * A + s] = make_double2(a0.x + a1.x, a0.y + a1.y);
  }
}

__global__ void sm_fold_kernel(const double2* __restrict__ cst, const uint32_t* __restrict__ first,
                               const uint32_t* __restrict__ off, const uint32_t* __restrict__ gfirst,
                               const uint32_t* __restrict__ gen, const uint64_t* __restrict__ base,
                               const int32_t* __restrict__ gidx, int n_nets, int n_total,
                               const double2* __restrict__ ph, const double2* ws, int A,
                               double2* __restrict__ results) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  if (s >= A || n >= n_nets) return;
  double2 r = cst[n];
  for (uint32_t k = first[n]; k < first[n + 1]; ++k) r = cmul(r, ws[(base[n] + off[k]) * A + s]);
  for (uint32_t k = gfirst[n]; k < gfirst[n + 1]; ++k) {
    const uint32_t g = gen[k];
    r = cmul(r, gate_entry(g & 0xff, (g >> 8) & 0xff, ph[(int64_t)(g >> 16) * A + s]));
  }
  results[(int64_t)s * n_total + gidx[n]] = r;
}

}  // namespace

int setmajor_build(SetMajor** out, const std::vector<const qtn_plan*>& plans,
                   const std::vector<int32_t>& gidx, const qtn_tensor_recipe* rec,
                   const int64_t* offsets, int32_t n_total) {
  SetMajor* S = new SetMajor();
  S->n_nets = (int32_t)plans.size();
  S->n_total = n_total;
  std::map<std::tuple<double, double, int32_t>, int32_t> pidx;
  std::vector<SMParam> params;
  auto param_of = [&](const qtn_tensor_recipe& q) -> int32_t {
    SMParam p{};
    if (q.kind == QTN_GATE_SCALAR) {
      p.scale = q.scale;
      p.offset = q.offset;
      p.angle = -2;
    } else {
      const bool has_t = q.kind == QTN_GATE_ZPOW || q.kind == QTN_GATE_XPOW || q.kind == QTN_GATE_ZZ ||
                         q.kind == QTN_GATE_ZPOW_DIAG || q.kind == QTN_GATE_ZZ_DIAG;
      p.scale = has_t ? q.scale : 0.0;
      p.offset = has_t ? q.offset : 0.0;
      p.angle = has_t ? (q.angle >= 0 ? q.angle : -1) : -1;
    }
    auto key = std::make_tuple(p.scale, p.offset, p.angle);
    auto it = pidx.find(key);
    if (it != pidx.end()) return it->second;
    const int32_t k = (int32_t)params.size();
    params.push_back(p);
    pidx.emplace(key, k);
    return k;
  };
  // full (unsliced) index of kept entry j of recipe q
  auto full_of = [](const qtn_tensor_recipe& q, uint32_t j) {
    const int kept = __builtin_popcount(q.keep_mask);
    uint32_t full = 0;
    int kb = kept - 1;
    for (int pos = 0; pos < q.full_rank; ++pos) {
      const uint32_t bit = ((q.keep_mask >> pos) & 1) ? (j >> kb--) & 1 : (q.fixed_bits >> pos) & 1;
      full = (full << 1) | bit;
    }
    return full;
  };
  int32_t max_lev = 0;
  for (auto* P : plans) max_lev = std::max(max_lev, P->sm_levels);
  S->n_levels = max_lev;
  std::vector<uint64_t> base;
  std::vector<double2> cst;
  std::vector<uint32_t> scal_first, scal_off, sgen_first, sgen;
  uint64_t elems = 0;
  for (size_t k = 0; k < plans.size(); ++k) {
    const qtn_plan* P = plans[k];
    base.push_back(elems);
    elems += P->sm_elems;
    double re = std::ldexp(1.0, P->n_empty), im = 0.0;
    sgen_first.push_back((uint32_t)sgen.size());
    for (int32_t id : P->sm_scalar_in) {
      const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + id];
      if (q.kind != QTN_GATE_SCALAR) {
        // a gate whose variables are all sliced: one angle-dependent entry
        sgen.push_back((uint32_t)q.kind | (full_of(q, 0) << 8) | ((uint32_t)param_of(q) << 16));
        continue;
      }
      const double nr = re * q.scale - im * q.offset, ni = re * q.offset + im * q.scale;
      re = nr;
      im = ni;
    }
    cst.push_back(make_double2(re, im));
    scal_first.push_back((uint32_t)scal_off.size());
    for (uint32_t o : P->sm_scalar_off) scal_off.push_back(o);
  }
  scal_first.push_back((uint32_t)scal_off.size());
  sgen_first.push_back((uint32_t)sgen.size());
  S->total_elems = elems;
  if (elems >= 0x80000000ull) {
    delete S;
    set_error("set-major executor: too many elements");
    return QTN_EINVAL;
  }
  // level-major CTA records over all networks, heaviest buckets of a level first
  std::vector<uint32_t> recs;
  uint32_t n_cta = 0;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    S->level_rec.push_back(n_cta);
    std::vector<std::tuple<uint64_t, size_t, const qtn_plan::SMBucketRec*>> lvb;
    for (size_t k = 0; k < plans.size(); ++k)
      for (const auto& rb : plans[k]->sm_buckets)
        if (rb.level == lev) lvb.emplace_back(~((uint64_t)rb.ops.size() << rb.R), k, &rb);
    std::stable_sort(lvb.begin(), lvb.end(),
                     [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
    uint32_t acc = 0;
    for (const auto& it : lvb) {
      const size_t k = std::get<1>(it);
      const auto& rb = *std::get<2>(it);
      if (rb.ops.size() > (size_t)kMaxOps) {
        delete S;
        set_error("set-major executor: bucket with more than 8 operands");
        return QTN_EINVAL;
      }
      for (uint32_t e = 0; e < (1u << rb.R); ++e) {
        const size_t r0 = recs.size();
        recs.resize(r0 + kRecWords, 0);
        recs[r0] = (uint32_t)(base[k] + rb.out_off + e);
        recs[r0 + 1] = (uint32_t)rb.ops.size();
        for (size_t t = 0; t < rb.ops.size(); ++t) {
          const auto& o = rb.ops[t];
          const uint32_t i0 = o.idx[2 * e], i1 = o.idx[2 * e + 1];
          if (o.input >= 0) {
            const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + o.input];
            const int c0 = coef_code(gate_coef(q.kind, full_of(q, i0)));
            const int c1 = coef_code(gate_coef(q.kind, full_of(q, i1)));
            if (c0 < 0 || c1 < 0) {
              delete S;
              set_error("set-major executor: unsupported gate coefficient");
              return QTN_EINVAL;
            }
            recs[r0 + 2 + 2 * t] = 0x80000000u | (uint32_t)param_of(q);
            recs[r0 + 3 + 2 * t] = (uint32_t)c0 | ((uint32_t)c1 << 8);
          } else {
            recs[r0 + 2 + 2 * t] = (uint32_t)(base[k] + o.off + i0);
            recs[r0 + 3 + 2 * t] = (uint32_t)(base[k] + o.off + i1);
          }
        }
        ++acc;
      }
    }
    S->level_blocks.push_back(acc);
    n_cta += acc;
  }

  // bucket-tile records (sm_bucket_kernel), same level-major heaviest-first order
  std::vector<uint32_t> brec, boff, btab;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    S->level_bk_first.push_back((uint32_t)boff.size());
    std::vector<std::tuple<uint64_t, size_t, const qtn_plan::SMBucketRec*>> lvb;
    for (size_t k = 0; k < plans.size(); ++k)
      for (const auto& rb : plans[k]->sm_buckets)
        if (rb.level == lev) lvb.emplace_back(~((uint64_t)rb.ops.size() << rb.R), k, &rb);
    std::stable_sort(lvb.begin(), lvb.end(),
                     [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
    for (const auto& it : lvb) {
      const size_t k = std::get<1>(it);
      const auto& rb = *std::get<2>(it);
      const uint32_t ne = 1u << rb.R;
      const size_t r0 = brec.size();
      boff.push_back((uint32_t)r0);
      brec.resize(r0 + 4 + 4 * rb.ops.size(), 0);
      brec[r0] = (uint32_t)(base[k] + rb.out_off);
      brec[r0 + 1] = rb.R | ((uint32_t)rb.ops.size() << 8);
      // staging choice: gates always (one phase row), intermediates by reuse
      std::vector<std::pair<uint32_t, size_t>> cand;  // (rows, op)
      std::vector<uint32_t> rows_of(rb.ops.size(), 0);
      for (size_t t = 0; t < rb.ops.size(); ++t) {
        const auto& o = rb.ops[t];
        uint32_t mx = 0;
        for (uint16_t v : o.idx) mx = std::max<uint32_t>(mx, v);
        rows_of[t] = mx + 1;
        if (o.input < 0 && rows_of[t] < 2 * ne) cand.emplace_back(rows_of[t], t);
      }
      std::sort(cand.begin(), cand.end());
      uint32_t nrows = 0;
      for (const auto& o : rb.ops)
        if (o.input >= 0) ++nrows;
      std::vector<int> staged(rb.ops.size(), 0);
      for (const auto& cd : cand)
        if ((int64_t)(nrows + cd.first) * kTile * 16 <= kStageBudget) {
          staged[cd.second] = 1;
          nrows += cd.first;
        }
      uint32_t row = 0;
      for (size_t t = 0; t < rb.ops.size(); ++t) {
        const auto& o = rb.ops[t];
        uint32_t* q4 = &brec[r0 + 4 + 4 * t];
        q4[3] = (uint32_t)btab.size();
        if (o.input >= 0) {
          const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + o.input];
          q4[0] = (2u << 30) | row;
          q4[1] = (uint32_t)param_of(q);
          q4[2] = 1;
          row += 1;
          for (uint32_t e = 0; e < ne; ++e) {
            const int c0 = coef_code(gate_coef(q.kind, full_of(q, o.idx[2 * e])));
            const int c1 = coef_code(gate_coef(q.kind, full_of(q, o.idx[2 * e + 1])));
            if (c0 < 0 || c1 < 0) {
              delete S;
              set_error("set-major executor: unsupported gate coefficient");
              return QTN_EINVAL;
            }
            btab.push_back((uint32_t)c0 | ((uint32_t)c1 << 8));
          }
        } else {
          if (staged[t]) {
            q4[0] = (1u << 30) | row;
            q4[1] = (uint32_t)(base[k] + o.off);
            q4[2] = rows_of[t];
            row += rows_of[t];
          } else {
            q4[0] = (uint32_t)(base[k] + o.off);
          }
          for (uint32_t e = 0; e < ne; ++e)
            btab.push_back((uint32_t)o.idx[2 * e] | ((uint32_t)o.idx[2 * e + 1] << 16));
        }
      }
    }
    S->level_bk.push_back((uint32_t)(boff.size() - S->level_bk_first.back()));
  }

  // ---- fused form: per network, liveness-packed offsets and local phase slots
  std::vector<SMFNet> fnets;
  std::vector<SMFBucket> fbk;
  std::vector<SMOpDev> fops;
  std::vector<uint32_t> ftabs, fsc, fsg;
  std::vector<SMParam> fpar;
  std::vector<uint64_t> fcost;
  const char* bv = getenv("QTN_SMF_BUDGET");
  const int64_t budget = bv ? atoll(bv) : 32768;
  const int64_t kMaxSmem = 227 * 1024;
  int64_t need_max = 0;
  bool fused_ok = true;
  for (size_t k = 0; k < plans.size() && fused_ok; ++k) {
    const qtn_plan* P = plans[k];
    SMFNet fn{};
    fn.first_bk = (uint32_t)fbk.size();
    fn.first_par = (uint32_t)fpar.size();
    std::map<int32_t, uint32_t> slot;  // global param -> local slot
    auto slot_of = [&](const qtn_tensor_recipe& q) -> uint32_t {
      const int32_t gp = param_of(q);
      auto it = slot.find(gp);
      if (it != slot.end()) return it->second;
      const uint32_t sl = (uint32_t)slot.size();
      slot.emplace(gp, sl);
      fpar.push_back(params[gp]);
      return sl;
    };
    // first-fit allocator over data elements; an output is allocated before
    // its operands are released, so a bucket never overwrites what it reads
    std::vector<uint8_t> used;
    std::vector<uint32_t> remap(P->sm_elems + 1, 0), rsize(P->sm_elems + 1, 0);
    uint32_t peak = 0;
    auto alloc = [&](uint32_t n) {
      uint32_t a = 0;
      for (;;) {
        uint32_t r = 0;
        while (r < n && a + r < used.size() && !used[a + r]) ++r;
        if (r == n || a + r >= used.size()) break;
        a += r + 1;
      }
      if (a + n > used.size()) used.resize(a + n, 0);
      for (uint32_t i = 0; i < n; ++i) used[a + i] = 1;
      peak = std::max(peak, a + n);
      return a;
    };
    uint64_t cost = 0;
    for (const auto& rb : P->sm_buckets) {
      SMFBucket d{};
      const uint32_t n = 1u << rb.R;
      d.out_off = alloc(n);
      remap[rb.out_off] = d.out_off;
      rsize[rb.out_off] = n;
      d.first_op = (uint32_t)fops.size();
      d.R = (uint16_t)rb.R;
      d.n_ops = (uint16_t)rb.ops.size();
      cost += (uint64_t)n * rb.ops.size();
      for (const auto& o : rb.ops) {
        SMOpDev od{};
        od.tab = (uint32_t)ftabs.size();
        if (o.input >= 0) {
          const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + o.input];
          od.gen = 1;
          od.kind = q.kind;
          od.param = (uint16_t)slot_of(q);
          for (size_t e = 0; e < o.idx.size(); e += 2)
            ftabs.push_back(full_of(q, o.idx[e]) | (full_of(q, o.idx[e + 1]) << 16));
        } else {
          od.off = remap[o.off];
          for (size_t e = 0; e < o.idx.size(); e += 2)
            ftabs.push_back((uint32_t)o.idx[e] | ((uint32_t)o.idx[e + 1] << 16));
        }
        fops.push_back(od);
      }
      for (const auto& o : rb.ops)
        if (o.input < 0)
          for (uint32_t i = 0; i < rsize[o.off]; ++i) used[remap[o.off] + i] = 0;
      fbk.push_back(d);
    }
    fn.n_bk = (uint32_t)(fbk.size() - fn.first_bk);
    fn.first_sc = (uint32_t)fsc.size();
    for (uint32_t o : P->sm_scalar_off) fsc.push_back(remap[o]);
    fn.n_sc = (uint32_t)(fsc.size() - fn.first_sc);
    fn.first_sg = (uint32_t)fsg.size();
    double re = std::ldexp(1.0, P->n_empty), im = 0.0;
    for (int32_t id : P->sm_scalar_in) {
      const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + id];
      if (q.kind != QTN_GATE_SCALAR) {
        fsg.push_back((uint32_t)q.kind | (full_of(q, 0) << 8) | (slot_of(q) << 16));
        continue;
      }
      const double nr = re * q.scale - im * q.offset, ni = re * q.offset + im * q.scale;
      re = nr;
      im = ni;
    }
    fn.n_sg = (uint32_t)(fsg.size() - fn.first_sg);
    fn.cst = make_double2(re, im);
    fn.n_par = (uint32_t)slot.size();
    fn.n_elems = peak;
    fn.gidx = gidx[k];
    const int64_t per_set = (int64_t)(peak + fn.n_par) * 16;
    uint32_t sh = 5;
    while (sh > 0 && per_set * (1 << sh) > budget) --sh;
    fn.sh = sh;
    need_max = std::max(need_max, per_set << sh);
    if (need_max > kMaxSmem || fn.n_par > 65535) fused_ok = false;
    fnets.push_back(fn);
    fcost.push_back(cost);
  }
  if (fused_ok && !fnets.empty()) {
    // heaviest units first (work per unit ~ cost * S / min(32, ...)): sort by
    // per-set cost, stable
    std::vector<size_t> perm(fnets.size());
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = i;
    std::stable_sort(perm.begin(), perm.end(), [&](size_t a, size_t b) {
      return (fcost[a] << fnets[a].sh) > (fcost[b] << fnets[b].sh);
    });
    std::vector<SMFNet> sorted;
    for (size_t i : perm) sorted.push_back(fnets[i]);
    fnets.swap(sorted);
    for (const auto& fn : fnets) S->f_sh.push_back(fn.sh);
    S->f_smem = need_max;
    int rc;
    if ((rc = upload_vec(&S->d_fnets, fnets)) || (rc = upload_vec(&S->d_fbk, fbk)) ||
        (rc = upload_vec(&S->d_fops, fops)) || (rc = upload_vec(&S->d_ftabs, ftabs)) ||
        (rc = upload_vec(&S->d_fpar, fpar)) || (rc = upload_vec(&S->d_fsc, fsc)) ||
        (rc = upload_vec(&S->d_fsg, fsg))) {
      setmajor_destroy(S);
      return rc;
    }
    S->fused_ok = true;
  }

  if (params.size() > 65535) {
    delete S;
    set_error("set-major executor: too many gate parameters");
    return QTN_EINVAL;
  }
  S->n_params = (int32_t)params.size();
  int rc;
  static bool coef_up = false;
  if (!coef_up) {
    if (cudaMemcpyToSymbol(kGateCoef, kCoefHost, sizeof(kCoefHost)) != cudaSuccess) {
      setmajor_destroy(S);
      set_error("set-major executor: coefficient upload failed");
      return QTN_ECUDA;
    }
    coef_up = true;
  }
  if ((rc = upload_vec(&S->d_recs, recs)) || (rc = upload_vec(&S->d_brec, brec)) ||
      (rc = upload_vec(&S->d_brec_off, boff)) || (rc = upload_vec(&S->d_btab, btab)) || (rc = upload_vec(&S->d_base, base)) || (rc = upload_vec(&S->d_params, params)) ||
      (rc = upload_vec(&S->d_const, cst)) || (rc = upload_vec(&S->d_scal_first, scal_first)) ||
      (rc = upload_vec(&S->d_scal_off, scal_off)) || (rc = upload_vec(&S->d_sgen_first, sgen_first)) ||
      (rc = upload_vec(&S->d_sgen, sgen)) ||
      (rc = upload_vec(&S->d_gidx, std::vector<int32_t>(gidx.begin(), gidx.end())))) {
    setmajor_destroy(S);
    return rc;
  }
  *out = S;
  return QTN_OK;
}

int64_t setmajor_workspace(const SetMajor* S, int32_t n_sets) {
  if (fused_on(S)) return 256;
  return (int64_t)(S->total_elems + (uint64_t)S->n_params) * n_sets * 16 + 256;
}

int setmajor_launches(const SetMajor* S, int32_t n_sets) {
  if (fused_on(S)) return 1;
  int c = 2;  // phases + fold
  for (uint32_t b : S->level_blocks) c += b ? 1 : 0;
  return c;
}

int setmajor_run(SetMajor* S, const double* angles, int32_t n_angles, int32_t n_sets,
                 void* workspace, void* results, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (fused_on(S)) {
    auto it = S->f_prefix.find(n_sets);
    if (it == S->f_prefix.end()) {
      std::vector<uint32_t> pre;
      uint32_t acc = 0;
      for (uint32_t sh : S->f_sh) {
        pre.push_back(acc);
        acc += (uint32_t)((n_sets + (1 << sh) - 1) >> sh);
      }
      uint32_t* d = nullptr;
      int rc = upload_vec(&d, pre);
      if (rc) return rc;
      it = S->f_prefix.emplace(n_sets, std::make_pair(d, acc)).first;
    }
    static int64_t attr_set = -1;
    if (attr_set < S->f_smem) {
      cudaFuncSetAttribute(smf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->f_smem);
      attr_set = S->f_smem;
    }
    smf_kernel<<<it->second.second, 32, S->f_smem, st>>>(
        S->d_fnets, it->second.first, S->n_nets, S->d_fbk, S->d_fops, S->d_ftabs, S->d_fpar,
        S->d_fsc, S->d_fsg, angles, n_angles, n_sets, S->n_total,
        reinterpret_cast<double2*>(results));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error(std::string("set-major fused executor launch: ") + cudaGetErrorString(e));
      return QTN_ECUDA;
    }
    return QTN_OK;
  }
  double2* ws = reinterpret_cast<double2*>(workspace);
  double2* ph = ws + S->total_elems * (uint64_t)n_sets;
  {
    dim3 g((n_sets + 127) / 128, std::max(S->n_params, 1));
    sm_phase_kernel<<<g, 128, 0, st>>>(S->d_params, S->n_params, angles, n_angles, n_sets, ph);
  }
  for (int32_t lev = 0; lev < S->n_levels; ++lev) {
    const uint32_t blocks = S->level_blocks[lev];
    if (!blocks) continue;
    const uint32_t* r = S->d_recs + (size_t)S->level_rec[lev] * kRecWords;
    // few CTAs (tail levels): split the sets over grid.y so the level is not
    // bound by one CTA's chain of operand round trips
    const uint32_t split = blocks < 4u * 148u ? (uint32_t)((n_sets + 255) / 256) : 1u;
    const char* bv = getenv("QTN_SM_BUCKET");
    const char* pv = getenv("QTN_SM_PIPE");
    if (bv && bv[0] == '1') {
      const uint32_t nbk = S->level_bk[lev];
      sm_bucket_kernel<<<dim3(nbk, (n_sets + kTile - 1) / kTile), 256, kStageBudget, st>>>(
          S->d_brec, S->d_brec_off + S->level_bk_first[lev], S->d_btab, ph, ws, n_sets);
    } else if (pv && pv[0] == '1')
      sm_level_pipe_kernel<<<dim3(blocks, split), 256, 0, st>>>(r, ph, ws, n_sets);
    else if (split > 1)
      sm_level_kernel<1, false><<<dim3(blocks, split), 256, 0, st>>>(r, ph, ws, n_sets);
    else if (n_sets >= 1024 && n_sets % 512 == 0)
      sm_level_kernel<2, true><<<blocks, 256, 0, st>>>(r, ph, ws, n_sets);
    else if (n_sets >= 1024)
      sm_level_kernel<2, false><<<blocks, 256, 0, st>>>(r, ph, ws, n_sets);
    else
      sm_level_kernel<1, false><<<blocks, 256, 0, st>>>(r, ph, ws, n_sets);
  }
  {
    dim3 g((n_sets + 127) / 128, S->n_nets);
    sm_fold_kernel<<<g, 128, 0, st>>>(S->d_const, S->d_scal_first, S->d_scal_off, S->d_sgen_first,
                                      S->d_sgen, S->d_base, S->d_gidx, S->n_nets, S->n_total, ph,
                                      ws, n_sets,
                                      reinterpret_cast<double2*>(results));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("set-major executor launch: ") + cudaGetErrorString(e));
    return QTN_ECUDA;
  }
  return QTN_OK;
}

void setmajor_destroy(SetMajor* S) {
  if (!S) return;
  for (void* p : {(void*)S->d_recs, (void*)S->d_brec, (void*)S->d_brec_off, (void*)S->d_btab, (void*)S->d_base, (void*)S->d_params, (void*)S->d_const, (void*)S->d_scal_first,
                  (void*)S->d_scal_off, (void*)S->d_sgen_first, (void*)S->d_sgen, (void*)S->d_gidx,
                  (void*)S->d_fnets, (void*)S->d_fbk, (void*)S->d_fops, (void*)S->d_ftabs,
                  (void*)S->d_fpar, (void*)S->d_fsc, (void*)S->d_fsg})
    device_free(p);
  for (auto& kv : S->f_prefix) device_free(kv.second.first);
  delete S;
}

}  // namespace qtn
