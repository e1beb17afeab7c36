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
// intermediate has its own rows, so concurrent buckets never alias).
//
// Input tensors are never stored.  Every gate entry is an affine form of the
// phase e^{-i t} of its angle (circuit.py:186-205): entry = (a + u cos t,
// -w sin t) with (a, u, w) from a table of 8 forms.  One small kernel writes,
// per evaluation, one "gate row" [s] for every (angle parameter, form) pair
// the batch uses, appended to the workspace after the intermediates; a gate
// operand is then just two more rows, and the level kernel has a single code
// path: two row loads and a complex multiply per operand.  Slicing of gate
// variables (network.py:153-165) is resolved when the records are built.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "qtn_pdl.cuh"
#include "qtn_setmajor.h"

namespace qtn {

// angle parameter of a gate: t = scale * angles[angle] + offset; angle -1:
// constant t = offset; angle -2: literal entry (scale + i offset)
struct SMParam {
  double scale, offset;
  int32_t angle;
  int32_t pad;
};

// one gate row: form `code` of parameter `param`
struct SMGateRow {
  int32_t param;
  int32_t code;
};

struct SetMajor {
  int32_t n_nets = 0, n_total = 0, n_levels = 0;
  uint64_t total_elems = 0;            // intermediate rows
  int32_t n_gate_rows = 0;             // gate rows, after the intermediates
  bool c64 = false;                    // complex64 rows (float32 products)
  std::vector<uint32_t> level_blocks;  // CTAs per level
  std::vector<uint32_t> level_rec;     // first CTA record of each level
  uint32_t* d_recs = nullptr;          // kRecWords per CTA (see sm_level_kernel)
  SMParam* d_params = nullptr;
  SMGateRow* d_grows = nullptr;
  double2* d_const = nullptr;          // per net: 2^n_empty * literal rank-0 inputs
  uint32_t* d_scal_first = nullptr;    // per net: rank-0 rows (absolute) folded at the end
  uint32_t* d_scal = nullptr;
  int32_t* d_gidx = nullptr;
};

namespace {

constexpr int kMaxOps = 8;  // operands per bucket in the set-major form
constexpr int kRecWords = 2 + 2 * kMaxOps;

// Gate entry as an affine form of the phase ph = e^{-i t}:
// entry = (a + u * ph.x, w * ph.y).
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

// the distinct affine forms gate_coef produces
constexpr int kNumCoef = 8;
const double kCoefHost[kNumCoef][3] = {
    {0.0, 0.0, 0.0}, {1.0, 0.0, 0.0}, {0.70710678118654757, 0.0, 0.0},
    {-0.70710678118654757, 0.0, 0.0}, {0.0, 1.0, 1.0}, {0.0, 1.0, -1.0},
    {0.5, 0.5, 0.5}, {0.5, -0.5, -0.5}};
// statically initialised: __constant__ memory is per device, and a static
// initializer is loaded with the module on every device the process uses
__constant__ double kGateCoef[kNumCoef][3] = {
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

// gate rows: grow[r][s] = form code_r of the phase of param_r at set s
// (formed in float64; complex64 rows round the entry).  Sets A..stride-1 of
// a padded complex64 row are written as zero.
template <typename RowT>
__global__ void sm_gate_rows_kernel(const SMGateRow* __restrict__ rows, int n_rows,
                                    const SMParam* __restrict__ par,
                                    const double* __restrict__ angles, int n_angles, int A,
                                    int stride, RowT* __restrict__ grow) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  pdl_trigger();
  pdl_wait();
  if (s >= stride || r >= n_rows) return;
  double2 v = make_double2(0.0, 0.0);
  if (s < A) {
    const SMGateRow g = rows[r];
    const SMParam q = par[g.param];
    double2 ph;
    if (q.angle == -2) {
      ph = make_double2(q.scale, q.offset);
    } else {
      const double t = q.angle >= 0 ? q.scale * angles[(int64_t)s * n_angles + q.angle] + q.offset
                                    : q.offset;
      double sn, cs;
      sincos(t, &sn, &cs);
      ph = make_double2(cs, -sn);
    }
    v = make_double2(fma(kGateCoef[g.code][1], ph.x, kGateCoef[g.code][0]),
                     kGateCoef[g.code][2] * ph.y);
  }
  if constexpr (sizeof(RowT) == 8)
    grow[(int64_t)r * stride + s] = make_float2((float)v.x, (float)v.y);
  else
    grow[(int64_t)r * stride + s] = v;
}

// ---- level kernel
// One CTA per (bucket, output element e) of a level; 256 threads stream the
// sets, J per thread per pass.  Everything the CTA needs is one fixed-size
// record (a single dependent load): word 0 = absolute output row, word 1 =
// operand count, then per operand the absolute rows of its entries
// idx(e, v=0) and idx(e, v=1) — intermediate rows or gate rows alike.  The
// operand loop stays rolled (~40 registers, high occupancy): the L2/HBM round
// trip of each operand is hidden by resident warps.  Rows read here were
// written by earlier launches only, hence the non-coherent load path.

// per-iteration shared-memory read (asm volatile: not hoisted out of the set
// loop, which would pin every operand's row pointers in registers)
__device__ __forceinline__ uint64_t lds_u64(const void* p) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ double2 ldg_nc(uint64_t gaddr) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(gaddr));
  return v;
}

// FULL: A is a multiple of 256 * J * gridDim.y (no per-set bounds checks).
// grid.y > 1 (levels with few CTAs) splits the sets over CTAs.
template <int J, bool FULL>
__global__ void __launch_bounds__(256) sm_level_kernel(const uint32_t* __restrict__ recs,
                                                       double2* ws, int A) {
  __shared__ uint64_t rowp[kMaxOps][2];  // global byte addresses of the two rows
  const uint32_t* r = recs + (size_t)blockIdx.x * kRecWords;
  const uint2 hd = *reinterpret_cast<const uint2*>(r);
  const int n = (int)hd.y;
  if (threadIdx.x < n) {
    const uint2 w = reinterpret_cast<const uint2*>(r + 2)[threadIdx.x];
    rowp[threadIdx.x][0] = reinterpret_cast<uint64_t>(ws + (size_t)w.x * A);
    rowp[threadIdx.x][1] = reinterpret_cast<uint64_t>(ws + (size_t)w.y * A);
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();  // rows of earlier levels
  double2* out = ws + (size_t)hd.x * A;
  const int s_step = 256 * J * gridDim.y;
#pragma unroll 1
  for (int s0 = blockIdx.y * 256 * J + threadIdx.x; s0 < A; s0 += s_step) {
    const uint64_t so = (uint64_t)s0 * sizeof(double2);
    double2 a0[J], a1[J];
    {
      const uint64_t p0 = lds_u64(&rowp[0][0]) + so, p1 = lds_u64(&rowp[0][1]) + so;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool ok = J == 1 || FULL || s0 + 256 * j < A;
        a0[j] = ok ? ldg_nc(p0 + 4096 * j) : make_double2(0.0, 0.0);
        a1[j] = ok ? ldg_nc(p1 + 4096 * j) : make_double2(0.0, 0.0);
      }
    }
#pragma unroll 1
    for (int k = 1; k < n; ++k) {
      const uint64_t p0 = lds_u64(&rowp[k][0]) + so, p1 = lds_u64(&rowp[k][1]) + so;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool ok = J == 1 || FULL || s0 + 256 * j < A;
        const double2 x = ok ? ldg_nc(p0 + 4096 * j) : make_double2(0.0, 0.0);
        const double2 y = ok ? ldg_nc(p1 + 4096 * j) : make_double2(0.0, 0.0);
        a0[j] = cmul(a0[j], x);
        a1[j] = cmul(a1[j], y);
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (FULL || s0 + 256 * j < A)
        out[s0 + 256 * j] = make_double2(a0[j].x + a1[j].x, a0[j].y + a1[j].y);
  }
}

__device__ __forceinline__ float4 ldg_nc_f4(uint64_t gaddr) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(gaddr));
  return v;
}
// two complex64 products at once: (a.xy * b.xy, a.zw * b.zw)
__device__ __forceinline__ float4 cmul2(float4 a, float4 b) {
  return make_float4(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x),
                     fmaf(a.z, b.z, -a.w * b.w), fmaf(a.z, b.w, a.w * b.z));
}

// Complex64 rows (the configs' complex64 storage; products in float32): the
// same records, each thread streams J float4 = 2 consecutive sets per pass,
// half the bytes of the complex128 form.  Rows are padded to an even
// stride; a pass covers 512*J sets.  FULL: stride is a multiple of
// 512 * J * gridDim.y.
template <int J, bool FULL>
__global__ void __launch_bounds__(256) sm_level_kernel_c64(const uint32_t* __restrict__ recs,
                                                           float2* ws, int stride) {
  __shared__ uint64_t rowp[kMaxOps][2];
  const uint32_t* r = recs + (size_t)blockIdx.x * kRecWords;
  const uint2 hd = *reinterpret_cast<const uint2*>(r);
  const int n = (int)hd.y;
  if (threadIdx.x < n) {
    const uint2 w = reinterpret_cast<const uint2*>(r + 2)[threadIdx.x];
    rowp[threadIdx.x][0] = reinterpret_cast<uint64_t>(ws + (size_t)w.x * stride);
    rowp[threadIdx.x][1] = reinterpret_cast<uint64_t>(ws + (size_t)w.y * stride);
  }
  pdl_trigger();
  __syncthreads();
  pdl_wait();  // rows of earlier levels
  float4* out = reinterpret_cast<float4*>(ws + (size_t)hd.x * stride);
  const int s_step = 512 * J * gridDim.y;
#pragma unroll 1
  for (int s0 = blockIdx.y * 512 * J + 2 * threadIdx.x; s0 < stride; s0 += s_step) {
    const uint64_t so = (uint64_t)s0 * sizeof(float2);
    float4 a0[J], a1[J];
    {
      const uint64_t p0 = lds_u64(&rowp[0][0]) + so, p1 = lds_u64(&rowp[0][1]) + so;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool ok = J == 1 || FULL || s0 + 512 * j < stride;
        a0[j] = ok ? ldg_nc_f4(p0 + 4096 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
        a1[j] = ok ? ldg_nc_f4(p1 + 4096 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll 1
    for (int k = 1; k < n; ++k) {
      const uint64_t p0 = lds_u64(&rowp[k][0]) + so, p1 = lds_u64(&rowp[k][1]) + so;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool ok = J == 1 || FULL || s0 + 512 * j < stride;
        const float4 x = ok ? ldg_nc_f4(p0 + 4096 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 y = ok ? ldg_nc_f4(p1 + 4096 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
        a0[j] = cmul2(a0[j], x);
        a1[j] = cmul2(a1[j], y);
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (FULL || s0 + 512 * j < stride)
        out[(s0 >> 1) + 256 * j] = make_float4(a0[j].x + a1[j].x, a0[j].y + a1[j].y,
                                               a0[j].z + a1[j].z, a0[j].w + a1[j].w);
  }
}

// per (network, set): 2^n_empty * literals * product of its rank-0 rows
// (float64 products)
template <typename RowT>
__global__ void sm_fold_kernel(const double2* __restrict__ cst, const uint32_t* __restrict__ first,
                               const uint32_t* __restrict__ rows, const int32_t* __restrict__ gidx,
                               int n_nets, int n_total, const RowT* ws, int A, int stride,
                               double2* __restrict__ results) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  pdl_trigger();
  pdl_wait();
  if (s >= A || n >= n_nets) return;
  double2 r = cst[n];
  for (uint32_t k = first[n]; k < first[n + 1]; ++k) {
    const RowT x = ws[(size_t)rows[k] * stride + s];
    r = cmul(r, make_double2((double)x.x, (double)x.y));
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
  // complex64 rows when every network asked for complex64 storage
  // (QTN_SETMAJOR_C64=0 keeps complex128 rows for A/B measurements)
  {
    bool c64 = !plans.empty();
    for (auto* P : plans) c64 = c64 && P->dtype == QTN_DTYPE_C64;
    const char* ev = getenv("QTN_SETMAJOR_C64");
    if (ev && ev[0] == '0') c64 = false;
    S->c64 = c64;
  }
  auto fail = [&](const char* msg) {
    delete S;
    set_error(std::string("set-major executor: ") + msg);
    return QTN_EINVAL;
  };
  // angle parameters, deduplicated over the batch
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
  // gate rows (param, form); their row numbers follow the intermediates
  std::map<std::pair<int32_t, int32_t>, int32_t> grow_idx;
  std::vector<SMGateRow> grows;
  auto grow_of = [&](const qtn_tensor_recipe& q, uint32_t full) -> int32_t {
    const int code = coef_code(gate_coef(q.kind, full));
    if (code < 0) return -1;
    const auto key = std::make_pair(param_of(q), (int32_t)code);
    auto it = grow_idx.find(key);
    if (it != grow_idx.end()) return it->second;
    const int32_t k = (int32_t)grows.size();
    grows.push_back(SMGateRow{key.first, key.second});
    grow_idx.emplace(key, k);
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
  // Level of each bucket (QTN_SM_ALIGN): 0 = as soon as possible (ASAP, the
  // plan's own levels), 1 / 2 = whole shallower networks centred / moved to
  // the end, 3 (default) = every bucket as late as its consumer allows
  // (ALAP).  ASAP piles every gate-only bucket into level 0 and leaves the
  // tail levels to the deepest networks (latency-bound launches); ALAP
  // evens the level widths: config 2 682 M -> 722 M contractions/s,
  // config 3 99.7 M -> 102.7 M (measured; 2: 701 M).
  std::vector<int32_t> shift(plans.size(), 0);
  std::vector<std::vector<int32_t>> alap;
  const char* align_v = getenv("QTN_SM_ALIGN");
  const int align = align_v ? atoi(align_v) : 3;
  {
    for (size_t k = 0; k < plans.size(); ++k) {
      const int32_t slack = max_lev - plans[k]->sm_levels;
      shift[k] = align == 2 ? slack : (align == 1 ? slack / 2 : 0);
    }
    // 3: every bucket as late as its consumer allows (per-bucket ALAP)
    if (align >= 3) {
      alap.resize(plans.size());
      for (size_t k = 0; k < plans.size(); ++k) {
        const qtn_plan* P = plans[k];
        const int nb = (int)P->sm_buckets.size();
        alap[k].assign(nb, max_lev - 1);
        if (nb != (int)P->buckets.size()) continue;  // (not expected) keep ASAP + shift
        for (int bi = nb - 1; bi >= 0; --bi) {
          const int32_t c = P->tensors[P->buckets[bi].out].last_use;
          if (c >= 0 && c < nb) alap[k][bi] = alap[k][c] - 1;
        }
      }
    }
  }
  // 4: list scheduling towards even level widths: level by level, every
  // ready bucket whose ALAP deadline is this level, then ready buckets by
  // increasing deadline until the level holds total / levels CTAs
  if (align == 4 && !alap.empty()) {
    std::vector<std::vector<int32_t>> lev(plans.size());
    std::vector<std::vector<int32_t>> npend(plans.size());  // unscheduled producers
    double total = 0.0;
    for (size_t k = 0; k < plans.size(); ++k) {
      const qtn_plan* P = plans[k];
      const int nb = (int)P->sm_buckets.size();
      lev[k].assign(nb, -1);
      npend[k].assign(nb, 0);
      for (int bi = 0; bi < nb; ++bi) {
        total += std::ldexp(1.0, P->sm_buckets[bi].R);
        const int32_t c = P->tensors[P->buckets[bi].out].last_use;
        if (c >= 0 && c < nb) ++npend[k][c];
      }
    }
    const double target = total / std::max(1, max_lev);
    std::vector<std::tuple<int32_t, size_t, int32_t>> ready;  // (deadline, net, bucket)
    for (size_t k = 0; k < plans.size(); ++k)
      for (int bi = 0; bi < (int)lev[k].size(); ++bi)
        if (npend[k][bi] == 0) ready.emplace_back(alap[k][bi], k, bi);
    for (int32_t l = 0; l < max_lev; ++l) {
      std::sort(ready.begin(), ready.end());
      double width = 0.0;
      std::vector<std::tuple<int32_t, size_t, int32_t>> later, placed;
      for (const auto& it : ready) {
        const size_t k = std::get<1>(it);
        const int32_t bi = std::get<2>(it);
        const double w = std::ldexp(1.0, plans[k]->sm_buckets[bi].R);
        if (std::get<0>(it) <= l || width + w <= target) {
          lev[k][bi] = l;
          width += w;
          placed.push_back(it);
        } else {
          later.push_back(it);
        }
      }
      ready.swap(later);
      for (const auto& it : placed) {  // consumers become ready for level l + 1
        const size_t k = std::get<1>(it);
        const int32_t bi = std::get<2>(it);
        const int32_t c = plans[k]->tensors[plans[k]->buckets[bi].out].last_use;
        if (c >= 0 && c < (int32_t)lev[k].size() && --npend[k][c] == 0)
          ready.emplace_back(alap[k][c], k, c);
      }
    }
    alap.swap(lev);
  }
  auto level_of = [&](size_t k, ptrdiff_t bi) -> int32_t {
    if (!alap.empty() && alap[k].size() == plans[k]->sm_buckets.size()) return alap[k][bi];
    return plans[k]->sm_buckets[bi].level + shift[k];
  };
  std::vector<uint64_t> base;
  uint64_t elems = 0;
  for (auto* P : plans) {
    base.push_back(elems);
    elems += P->sm_elems;
  }
  S->total_elems = elems;
  // gate rows are tagged with the high bit until every row is numbered
  constexpr uint32_t kGateTag = 0x80000000u;
  // per network: constant factor and rank-0 rows
  std::vector<double2> cst;
  std::vector<uint32_t> scal_first, scal;
  for (size_t k = 0; k < plans.size(); ++k) {
    const qtn_plan* P = plans[k];
    double re = std::ldexp(1.0, P->n_empty), im = 0.0;
    scal_first.push_back((uint32_t)scal.size());
    for (int32_t id : P->sm_scalar_in) {
      const qtn_tensor_recipe& q = rec[offsets[gidx[k]] + id];
      if (q.kind != QTN_GATE_SCALAR) {
        // a gate whose variables are all sliced: one angle-dependent entry
        const int32_t g = grow_of(q, full_of(q, 0));
        if (g < 0) return fail("unsupported gate coefficient");
        scal.push_back(kGateTag | (uint32_t)g);
        continue;
      }
      const double nr = re * q.scale - im * q.offset, ni = re * q.offset + im * q.scale;
      re = nr;
      im = ni;
    }
    cst.push_back(make_double2(re, im));
    for (uint32_t o : P->sm_scalar_off) scal.push_back((uint32_t)(base[k] + o));
  }
  scal_first.push_back((uint32_t)scal.size());
  // level-major CTA records over all networks, heaviest buckets of a level first
  std::vector<uint32_t> recs;
  uint32_t n_cta = 0;
  for (int32_t lev = 0; lev < max_lev; ++lev) {
    S->level_rec.push_back(n_cta);
    std::vector<std::tuple<uint64_t, size_t, const qtn_plan::SMBucketRec*>> lvb;
    for (size_t k = 0; k < plans.size(); ++k)
      for (const auto& rb : plans[k]->sm_buckets)
        if (level_of(k, &rb - plans[k]->sm_buckets.data()) == lev)
          lvb.emplace_back(~((uint64_t)rb.ops.size() << rb.R), k, &rb);
    std::stable_sort(lvb.begin(), lvb.end(),
                     [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
    uint32_t acc = 0;
    for (const auto& it : lvb) {
      const size_t k = std::get<1>(it);
      const auto& rb = *std::get<2>(it);
      if (rb.ops.size() > (size_t)kMaxOps) return fail("bucket with more than 8 operands");
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
            const int32_t g0 = grow_of(q, full_of(q, i0)), g1 = grow_of(q, full_of(q, i1));
            if (g0 < 0 || g1 < 0) return fail("unsupported gate coefficient");
            recs[r0 + 2 + 2 * t] = kGateTag | (uint32_t)g0;
            recs[r0 + 3 + 2 * t] = kGateTag | (uint32_t)g1;
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
  if (getenv("QTN_DEBUG_ROUTE")) {
    fprintf(stderr, "set-major levels (CTAs):");
    for (uint32_t b : S->level_blocks) fprintf(stderr, " %u", b);
    fprintf(stderr, "\n");
  }
  if (elems + grows.size() >= kGateTag) return fail("too many rows");
  // gate row g lives at row total_elems + g
  auto resolve = [&](uint32_t& w) {
    if (w & kGateTag) w = (uint32_t)(elems + (w & ~kGateTag));
  };
  for (size_t r0 = 0; r0 < recs.size(); r0 += kRecWords)
    for (uint32_t t = 0; t < recs[r0 + 1]; ++t) {
      resolve(recs[r0 + 2 + 2 * t]);
      resolve(recs[r0 + 3 + 2 * t]);
    }
  for (uint32_t& w : scal) resolve(w);
  S->n_gate_rows = (int32_t)grows.size();
  int rc;
  if ((rc = upload_vec(&S->d_recs, recs)) || (rc = upload_vec(&S->d_params, params)) ||
      (rc = upload_vec(&S->d_grows, grows)) || (rc = upload_vec(&S->d_const, cst)) ||
      (rc = upload_vec(&S->d_scal_first, scal_first)) || (rc = upload_vec(&S->d_scal, scal)) ||
      (rc = upload_vec(&S->d_gidx, std::vector<int32_t>(gidx.begin(), gidx.end())))) {
    setmajor_destroy(S);
    return rc;
  }
  *out = S;
  return QTN_OK;
}

// row stride in sets: complex64 rows are padded to an even length (float4 pairs)
static int32_t row_stride(const SetMajor* S, int32_t n_sets) {
  return S->c64 ? (n_sets + 1) & ~1 : n_sets;
}

int64_t setmajor_workspace(const SetMajor* S, int32_t n_sets) {
  return (int64_t)(S->total_elems + (uint64_t)S->n_gate_rows) * row_stride(S, n_sets) *
             (S->c64 ? 8 : 16) +
         256;
}

int setmajor_elem_bytes(const SetMajor* S) { return S->c64 ? 8 : 16; }

int setmajor_launches(const SetMajor* S, int32_t n_sets) {
  (void)n_sets;
  int c = 2;  // gate rows + fold
  for (uint32_t b : S->level_blocks) c += b ? 1 : 0;
  return c;
}

int setmajor_run(SetMajor* S, const double* angles, int32_t n_angles, int32_t n_sets,
                 void* workspace, void* results, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int stride = row_stride(S, n_sets);
  const uint64_t grow_off = S->total_elems * (uint64_t)stride;
  const dim3 gg((stride + 127) / 128, std::max(S->n_gate_rows, 1));
  const dim3 gf((n_sets + 127) / 128, S->n_nets);
  double2* res = reinterpret_cast<double2*>(results);
  if (S->c64) {
    float2* ws = reinterpret_cast<float2*>(workspace);
    launch_pdl(sm_gate_rows_kernel<float2>, gg, dim3(128), 0, st, (const SMGateRow*)S->d_grows,
               S->n_gate_rows, (const SMParam*)S->d_params, angles, (int)n_angles, (int)n_sets,
               stride, ws + grow_off);
    for (int32_t lev = 0; lev < S->n_levels; ++lev) {
      const uint32_t blocks = S->level_blocks[lev];
      if (!blocks) continue;
      const uint32_t* r = S->d_recs + (size_t)S->level_rec[lev] * kRecWords;
      const uint32_t split = blocks < 4u * 148u ? (uint32_t)((stride + 511) / 512) : 1u;
      if (split > 1)
        launch_pdl(sm_level_kernel_c64<1, false>, dim3(blocks, split), dim3(256), 0, st, r, ws, stride);
      else if (stride >= 1024 && stride % 1024 == 0)
        launch_pdl(sm_level_kernel_c64<2, true>, blocks, dim3(256), 0, st, r, ws, stride);
      else if (stride >= 1024)
        launch_pdl(sm_level_kernel_c64<2, false>, blocks, dim3(256), 0, st, r, ws, stride);
      else
        // fewer than 512 sets: one pass needs only stride/2 threads
        launch_pdl(sm_level_kernel_c64<1, false>, blocks,
                   dim3(std::min(256, std::max(32, ((stride / 2) + 31) / 32 * 32))), 0, st, r, ws,
                   stride);
    }
    launch_pdl(sm_fold_kernel<float2>, gf, dim3(128), 0, st, (const double2*)S->d_const,
               (const uint32_t*)S->d_scal_first, (const uint32_t*)S->d_scal,
               (const int32_t*)S->d_gidx, S->n_nets, S->n_total, (const float2*)ws, (int)n_sets,
               stride, res);
  } else {
    double2* ws = reinterpret_cast<double2*>(workspace);
    launch_pdl(sm_gate_rows_kernel<double2>, gg, dim3(128), 0, st, (const SMGateRow*)S->d_grows,
               S->n_gate_rows, (const SMParam*)S->d_params, angles, (int)n_angles, (int)n_sets,
               stride, ws + grow_off);
    for (int32_t lev = 0; lev < S->n_levels; ++lev) {
      const uint32_t blocks = S->level_blocks[lev];
      if (!blocks) continue;
      const uint32_t* r = S->d_recs + (size_t)S->level_rec[lev] * kRecWords;
      // few CTAs (tail levels): split the sets over grid.y so the level is not
      // bound by one CTA's chain of operand round trips
      const uint32_t split = blocks < 4u * 148u ? (uint32_t)((n_sets + 255) / 256) : 1u;
      if (split > 1)
        launch_pdl(sm_level_kernel<1, false>, dim3(blocks, split), dim3(256), 0, st, r, ws, (int)n_sets);
      else if (n_sets >= 1024 && n_sets % 512 == 0)
        launch_pdl(sm_level_kernel<2, true>, blocks, dim3(256), 0, st, r, ws, (int)n_sets);
      else if (n_sets >= 1024)
        launch_pdl(sm_level_kernel<2, false>, blocks, dim3(256), 0, st, r, ws, (int)n_sets);
      else
        launch_pdl(sm_level_kernel<1, false>, blocks, dim3(256), 0, st, r, ws, (int)n_sets);
    }
    launch_pdl(sm_fold_kernel<double2>, gf, dim3(128), 0, st, (const double2*)S->d_const,
               (const uint32_t*)S->d_scal_first, (const uint32_t*)S->d_scal,
               (const int32_t*)S->d_gidx, S->n_nets, S->n_total, (const double2*)ws, (int)n_sets,
               stride, res);
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
  for (void* p : {(void*)S->d_recs, (void*)S->d_params, (void*)S->d_grows, (void*)S->d_const,
                  (void*)S->d_scal_first, (void*)S->d_scal, (void*)S->d_gidx})
    device_free(p);
  delete S;
}

}  // namespace qtn
