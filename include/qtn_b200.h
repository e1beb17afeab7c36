/*
 * qtn_b200.h — C ABI of the B200 bucket-elimination backend.
 *
 * This is the drop-in boundary for the reference's contraction entry point
 *   contract(network, order, rank_cap=DEFAULT_RANK_CAP) -> complex
 *   (/root/reference/pkg/src/qtnsim/contraction.py:114-123)
 * and for the ordering passes it is fed by
 *   rgreedy_order / greedy_order / contraction_width
 *   (/root/reference/pkg/src/qtnsim/ordering.py:93-189).
 *
 * Plain C types only: no torch types cross this boundary.  Device pointers
 * are raw CUDA device addresses; `stream` is a cudaStream_t passed as void*.
 * The caller owns every buffer it passes in; a plan owns only host memory
 * (and, after qtn_batch_create, the device copy of its program).
 *
 * Return codes (every function returns int):
 *   QTN_OK        0  success
 *   QTN_EINVAL    1  invalid argument      -> Python ValueError
 *                    (contraction.py:61-62: order not a permutation)
 *   QTN_ERANKCAP  2  intermediate rank > rank_cap, detected at plan time
 *                    before any allocation -> RankCapExceeded(rank, cap)
 *                    (contraction.py:32-39, 85-87)
 *   QTN_ENOMEM    3  allocation failure
 *   QTN_ECUDA     4  CUDA runtime error
 *   QTN_ENODEV    5  no CUDA device (the backend never falls back to CPU)
 * qtn_last_error() returns a thread-local message for the last failure.
 */
#ifndef QTN_B200_H
#define QTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QTN_OK 0
#define QTN_EINVAL 1
#define QTN_ERANKCAP 2
#define QTN_ENOMEM 3
#define QTN_ECUDA 4
#define QTN_ENODEV 5

/* storage policy for intermediates (inputs are always complex128) */
#define QTN_DTYPE_C128 0  /* every intermediate complex128                    */
#define QTN_DTYPE_C64 1   /* complex64 for intermediates of rank >= mixed_rank */

/* executor chosen by the plan compiler */
#define QTN_EXEC_SMEM 0   /* whole network resident in one warp's shared memory */
#define QTN_EXEC_HBM 1    /* per-bucket kernels over a device arena             */

typedef struct qtn_plan qtn_plan;
typedef struct qtn_batch qtn_batch;

/* Structure of a network AFTER slicing of fixed variables
 * (network.py:153-165 `sliced_tensors`).  Tensor k has ranks[k] variables
 * vars[var_offsets[k] .. var_offsets[k]+ranks[k]), most significant first
 * (network.py:36-61 layout).  is_fixed[v] != 0 marks fixed variables, which
 * must not appear in any tensor.  Tensor data is supplied separately as one
 * packed complex128 buffer: tensor k at element offset qtn_plan_info.input_offset(k)
 * = sum_{j<k} 2^ranks[j]. */
typedef struct {
  int32_t n_tensors;
  const int32_t* ranks;
  const int32_t* var_offsets;
  const int32_t* vars;
  int32_t n_vars;
  const uint8_t* is_fixed;
} qtn_network_desc;

typedef struct {
  int32_t executor;          /* QTN_EXEC_SMEM or QTN_EXEC_HBM                    */
  int32_t n_buckets;         /* non-empty buckets                                */
  int32_t n_empty_buckets;   /* variables in no tensor: factor 2 each            */
  int32_t width;             /* max intermediate rank (== CostReport.width)      */
  int64_t input_elems;       /* complex128 elements of the packed input buffer   */
  int64_t workspace_bytes;   /* device arena for intermediates (HBM executor)    */
  int64_t smem_bytes;        /* shared memory for the SMEM executor              */
  int64_t program_bytes;     /* SMEM-executor program size                       */
  double alg_bytes;          /* sum over buckets of e*(operand + output entries) */
  double flops_sum;          /* sum 2^(rank+1) (ordering.py:60-61)               */
  int32_t n_levels;          /* HBM executor: levels of the elimination trees    */
  int32_t n_fused_chains;    /* HBM executor: product chains run as one kernel   */
  double exec_bytes;         /* bytes the executor's kernels move (fused chains:  */
                             /* operands + final output only)                   */
  int32_t n_pairs;           /* HBM executor: expanding bucket + consumer pairs  */
                             /* run as one kernel (their union-size result is    */
                             /* never stored)                                    */
  int32_t n_tails;           /* HBM executor: tail chains run as one weighted    */
                             /* sum over their first operand (qtn_wsum.cu)       */
} qtn_plan_info_t;

/* ---------------------------------------------------------------- ordering */

/* One elimination pass over a line graph given as hyperedges over compact
 * vertex ids 0..nv-1 (ordering.py:106-124).  draws == NULL selects the
 * deterministic min-degree rule (ordering.py:127-129); otherwise draws[0..nv)
 * are the uniform variates the reference would draw from
 * default_rng(seed + pass) and exp_table[d] = exp(-d/temp) computed by numpy
 * (ordering.py:139-151).  Writes the order and the per-step ranks. */
int qtn_order_pass(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                   const int32_t* edge_vertices, const double* draws,
                   const double* exp_table, int32_t temp_is_zero,
                   int32_t* out_order, int32_t* out_ranks);

/* rgreedy_order (ordering.py:154-189): pass 0 = min degree, passes 1..n-1 use
 * draws[(rep-1)*nv ...].  Best by (width, flops_sum, pass).  out_best = pass. */
int qtn_rgreedy(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                const int32_t* edge_vertices, int32_t n_repeats,
                const double* draws, const double* exp_table, int32_t temp_is_zero,
                int32_t* out_order, int32_t* out_ranks, int32_t* out_best);

/* contraction_width (ordering.py:93-100): step ranks along a given order. */
int qtn_order_ranks(int32_t nv, int32_t n_edges, const int32_t* edge_offsets,
                    const int32_t* edge_vertices, const int32_t* order,
                    int32_t* out_ranks);

/* ------------------------------------------------------------------ plans */

/* Compile (network, order) into a bucket program.  Pure host work: it needs
 * no GPU, and it raises QTN_EINVAL / QTN_ERANKCAP before any allocation.
 * On QTN_ERANKCAP *out_bad_rank is the first offending rank (reference
 * semantics, contraction.py:85-87).  dtype: QTN_DTYPE_*.  mixed_rank: rank
 * from which complex64 storage applies under QTN_DTYPE_C64.  smem_budget:
 * bytes one network may use for the SMEM executor (0 = never). */
int qtn_plan_create(const qtn_network_desc* net, const int32_t* order, int32_t n_order,
                    int32_t rank_cap, int32_t dtype, int32_t mixed_rank,
                    int64_t smem_budget, qtn_plan** out_plan, int32_t* out_bad_rank);
int qtn_plan_info(const qtn_plan* plan, qtn_plan_info_t* info);
/* step ranks of the non-empty + empty buckets in elimination order
 * (contraction.py:74-88 `ranks`), n = len(order) */
int qtn_plan_step_ranks(const qtn_plan* plan, int32_t* out_ranks);
int qtn_plan_input_offsets(const qtn_plan* plan, int64_t* out_offsets);
int qtn_plan_destroy(qtn_plan* plan);

/* Execute one plan.  inputs: packed complex128 sliced tensor data (device).
 * workspace: >= workspace_bytes of device memory (HBM executor; may be NULL
 * for the SMEM executor).  result: one complex128 (device). */
int qtn_plan_execute(qtn_plan* plan, const void* inputs, void* workspace,
                     void* result, void* stream);

/* ----------------------------------------------------- batched execution */

/* Upload n plans as one device program.  SMEM-executor networks run one
 * warp per (network, input set) in a single launch; HBM-executor networks
 * run level-synchronously: one streaming-kernel launch per level of the
 * elimination trees, covering every network and input set at once, then one
 * scalar-fold launch.  Network i's packed inputs start at element offset
 * qtn_batch_input_offsets()[i] inside one input set. */
int qtn_batch_create(qtn_plan* const* plans, int32_t n, qtn_batch** out_batch);
int qtn_batch_input_elems(const qtn_batch* batch, int64_t* out_elems);
int qtn_batch_input_offsets(const qtn_batch* batch, int64_t* out_offsets);
/* device workspace needed by qtn_batch_execute for n_sets input sets */
int qtn_batch_workspace_bytes(const qtn_batch* batch, int32_t n_sets, int64_t* out_bytes);
/* number of kernel launches one evaluation of n_sets input sets issues */
int qtn_batch_launches(const qtn_batch* batch, int32_t n_sets, int32_t* out_launches);
/* 1 if an evaluation of n_sets input sets runs the small networks on the
 * set-major executor (after qtn_batch_set_recipes), else 0 */
int qtn_batch_uses_setmajor(const qtn_batch* batch, int32_t n_sets, int32_t* out_flag);
/* bytes per stored set-major element for an evaluation of n_sets sets: 8
 * (complex64 rows: every plan of the batch asked for QTN_DTYPE_C64; products
 * in float32), 16 (complex128 rows, float64), 0 (set-major not used) */
int qtn_batch_setmajor_elem_bytes(const qtn_batch* batch, int32_t n_sets, int32_t* out_bytes);
/* results[s*n + i] = value of network i under input set s (complex128).
 * Input set s starts at inputs + s*set_stride elements (0: the batch's own
 * qtn_batch_input_elems). */
int qtn_batch_execute(qtn_batch* batch, const void* inputs, int64_t set_stride,
                      int32_t n_sets, void* workspace, void* results, void* stream);
int qtn_batch_destroy(qtn_batch* batch);

/* ------------------------------------------ parametric tensor generation */

/* One record per input tensor; see paper_2106_15740_b200/lightcone.py.
 * Gate entries follow circuit.py:186-205 with theta = scale*angles[angle] +
 * offset (angle < 0: theta = offset); kept/fixed bits implement
 * network.py:153-165 slicing. */
typedef struct {
  int64_t out_offset;  /* complex128 element offset inside one input set */
  double scale;
  double offset;
  int32_t angle;       /* index into the per-set angle vector, or -1     */
  uint8_t kind;        /* QTN_GATE_*                                     */
  uint8_t full_rank;   /* rank of the unsliced tensor                    */
  uint8_t keep_mask;   /* bit k set: position k (MSB first) is kept      */
  uint8_t fixed_bits;  /* bit k: value of sliced position k              */
} qtn_tensor_recipe;

#define QTN_GATE_INIT 0     /* (1, 0)                                */
#define QTN_GATE_H 1
#define QTN_GATE_ZPOW 2     /* full 2x2                              */
#define QTN_GATE_XPOW 3
#define QTN_GATE_CNOT 4     /* 4x4 -> (2,2,2,2)                      */
#define QTN_GATE_ZZ 5       /* full 4x4 -> (2,2,2,2)                 */
#define QTN_GATE_ZPOW_DIAG 6
#define QTN_GATE_ZZ_DIAG 7  /* diagonal reshaped (2,2)               */
#define QTN_GATE_SCALAR 8   /* rank 0: value = scale + i*offset      */

/* out[s*set_elems + rec.out_offset + e] for every set s and kept entry e. */
int qtn_tensorgen(const qtn_tensor_recipe* recipes_dev, int64_t n_recipes,
                  const double* angles_dev, int32_t n_angles, int32_t n_sets,
                  int64_t set_elems, void* out_dev, void* stream);

/* Attach per-network tensor recipes (host array; network i owns
 * recipes[offsets[i] .. offsets[i+1]), out_offset relative to the network's
 * packed input).  Afterwards qtn_batch_execute_angles builds every input on
 * device: SMEM-executor networks generate their tensors inside the executor
 * kernel (no input buffer at all), HBM networks through qtn_tensorgen.  With
 * many input sets (>= 64, env QTN_SETMAJOR_MIN_SETS) the small networks run
 * on the set-major streaming executor instead (angle sets as the fastest
 * tensor dimension in HBM, gate tensors generated on the fly). */
int qtn_batch_set_recipes(qtn_batch* batch, const qtn_tensor_recipe* recipes,
                          const int64_t* offsets);
/* One evaluation for n_sets angle vectors (angles_dev: n_sets x n_angles
 * float64).  inputs_scratch: >= n_sets * qtn_batch_input_elems complex128
 * (only touched when the batch has HBM networks; may be NULL otherwise). */
int qtn_batch_execute_angles(qtn_batch* batch, const double* angles_dev, int32_t n_angles,
                             int32_t n_sets, void* inputs_scratch, void* workspace,
                             void* results, void* stream);

/* energies[s] = sum_i (w_i - Re values[s*n + i]) / 2 and
 * zz_sum[s] = sum_i values[s*n+i] (complex128); deterministic order.
 * w_i = weights[i] (NULL: 1); an edge split into S slices has S networks of
 * weight 1/S whose values sum to <Z_iZ_j>. */
int qtn_energy_reduce(const void* values_dev, const double* weights_dev, int32_t n,
                      int32_t n_sets, double* energies_dev, void* zz_sum_dev, void* stream);

/* Host-to-host contraction of one set of packed inputs, the drop-in
 * `contract` call (contraction.py:114-123) on a kept batch: copy input_bytes
 * from inputs_pinned (page-locked host memory, the packed layout of
 * qtn_batch_input_offsets) to inputs_dev, run qtn_batch_execute for one set
 * on `stream`, copy the batch's n complex128 results to results_pinned and
 * wait for the stream. */
int qtn_batch_execute_host(qtn_batch* batch, const void* inputs_pinned, int64_t input_bytes,
                           void* inputs_dev, void* workspace, void* results_dev,
                           void* results_pinned, void* stream);

/* Host-to-host energy evaluation, the QAOA optimiser's call: copy n_sets
 * angle vectors from host memory (any host pointer; staged through pinned
 * memory owned by the batch) to angles_dev, run qtn_batch_execute_angles and
 * qtn_energy_reduce on `stream`, copy the energies back to energies_host and
 * wait for the stream.  Device buffers as for those two calls. */
int qtn_batch_energies_host(qtn_batch* batch, const double* angles_host, int32_t n_angles,
                            int32_t n_sets, double* angles_dev, void* inputs_scratch,
                            void* workspace, void* results, const double* weights_dev,
                            double* energies_dev, double* energies_host, void* stream);

/* --------------------------------------------------- single-bucket entry */

/* One bucket: out[o] = sum_{v in {0,1}} prod_t T_t[idx_t(o, v)] over
 * arbitrary operand variable subsets (contraction.py:90-96).  Operand t has
 * ranks[t] variables vars[var_offsets[t]...] (must include elim_var), data at
 * device pointer ptrs[t] with element type c64[t] ? complex64 : complex128.
 * out_vars lists the output layout (MSB first), out_c64 its element type. */
int qtn_bucket_contract(int32_t n_ops, const int32_t* ranks, const int32_t* var_offsets,
                        const int32_t* vars, const void* const* ptrs, const uint8_t* c64,
                        int32_t elim_var, int32_t out_rank, const int32_t* out_vars,
                        int32_t out_c64, void* out, void* stream);

/* the output layout the backend prefers for a bucket (primary operand's
 * order kept on the low bits); written to out_vars[0..out_rank) */
int qtn_bucket_layout(int32_t n_ops, const int32_t* ranks, const int32_t* var_offsets,
                      const int32_t* vars, int32_t elim_var, int32_t* out_rank,
                      int32_t* out_vars);

const char* qtn_last_error(void);
int qtn_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QTN_B200_H */
