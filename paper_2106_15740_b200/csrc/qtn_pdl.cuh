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

inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* v = getenv("QTN_PDL");
    on = (v && v[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
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
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace qtn
