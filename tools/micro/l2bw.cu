// L2 read-bandwidth probe: every SM streams 16-byte loads over a buffer that
// fits in L2 (after a warm-up pass); reports TB/s per buffer size.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const double2* __restrict__ p, size_t n, int reps, double* out) {
  double ax = 0, ay = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double2 v = __ldg(p + i);
      ax += v.x;
      ay += v.y;
    }
  if (ax == 12345.678) out[0] = ax + ay;
}

int main() {
  for (size_t mb : {8, 16, 32, 48, 64, 96, 256, 1024}) {
    const size_t n = mb * (1 << 20) / 16;
    double2* p;
    double* o;
    cudaMalloc(&p, n * 16);
    cudaMalloc(&o, 8);
    cudaMemset(p, 0, n * 16);
    const int reps = mb <= 96 ? 20 : 3;
    rd<<<148 * 8, 256>>>(p, n, 1, o);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rd<<<148 * 8, 256>>>(p, n, reps, o);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%5zu MB: %.2f TB/s\n", mb, (double)n * 16 * reps / (ms * 1e-3) / 1e12);
    cudaFree(p);
    cudaFree(o);
  }
  return 0;
}
