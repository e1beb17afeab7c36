// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-stream-serialization attribute may start while its
// predecessor on the stream drains.  Kernels call pdl_trigger() once all
// their CTAs are resident (so the successor can be scheduled as SMs free
// up), run their prologue (descriptor/record loads, shared-memory setup —
// static data only), and pdl_wait() before touching memory the predecessor
// writes or reads.  Without the attribute both instructions are no-ops.
// Level-synchronous executors issue one launch per elimination level, so
// this hides the launch gap and the prologue latency of every level.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace qtn {

// Set-major level kernels: on by default (QTN_PDL=0 disables; measured
// config 2 +2.7 %).  HBM executor kernels: off by default (QTN_PDL_HBM=1
// enables; measured config 4 -2 %, config 3 default -7 % with the trigger at
// kernel start: early-resident dependents compete with the persistent tile
// kernel).
inline bool pdl_enabled(bool hbm) {
  static int on = -1, on_hbm = -1;
  if (on < 0) {
    const char* v = getenv("QTN_PDL");
    on = (v && v[0] == '0') ? 0 : 1;
    const char* h = getenv("QTN_PDL_HBM");
    on_hbm = (h && h[0] == '1') ? 1 : 0;
  }
  return hbm ? on_hbm == 1 : on == 1;
}

// force: PDL for this launch regardless of the executor default (chains of
// tiny HBM levels, whose kernels stage only static data before pdl_wait)
template <bool HBM = false, typename... KArgs, typename... Args>
cudaError_t launch_pdl_if(bool force, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (force || pdl_enabled(HBM)) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Set by the HBM executor around the launch of a level that is one kernel
// following a level that was one kernel too (same stream, no fork/join):
// such a launch takes PDL even where the executor default is off.
inline thread_local bool g_pdl_next = false;

template <bool HBM = false, typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl_enabled(HBM) || (HBM && g_pdl_next)) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace qtn
