// Write-pattern probe: 512 MB of float4 stores, each CTA writing 32 rows of
// 4 KiB (256 threads x 16 B); rows of a CTA either adjacent or 16 MiB apart
// (the expanding-bucket output pattern: new bits on top).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void wk(float4* out, int rows, size_t row_stride, size_t cta_stride, int tiles_per_cta, int n_ctas_total) {
  for (int t = 0; t < tiles_per_cta; ++t) {
    size_t tile = (size_t)blockIdx.x * tiles_per_cta + t;
    float4* base = out + tile * cta_stride + threadIdx.x;
    for (int r = 0; r < rows; ++r) base[r * row_stride] = make_float4(1.f, 2.f, 3.f, (float)r);
  }
}
int main() {
  const size_t n = (512ull << 20) / 16;  // float4s
  float4* out;
  cudaMalloc(&out, n * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int rows = 32, tpb = 256;
  const size_t tiles = n / (rows * tpb);  // 4096
  for (int mode = 0; mode < 3; ++mode) {
    size_t row_stride, cta_stride;
    if (mode == 0) { row_stride = tpb; cta_stride = rows * tpb; }          // contiguous tiles
    else if (mode == 1) { row_stride = n / rows; cta_stride = tpb; }      // rows 16 MiB apart
    else { row_stride = n / rows; cta_stride = tpb; }
    int ctas = mode == 2 ? 4096 : 592;
    int tpc = (int)(tiles / ctas);
    for (int it = 0; it < 3; ++it) wk<<<ctas, tpb>>>(out, rows, row_stride, cta_stride, tpc, ctas);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) wk<<<ctas, tpb>>>(out, rows, row_stride, cta_stride, tpc, ctas);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d (%s, %d ctas): %.0f GB/s\n", mode, mode == 0 ? "contiguous" : "rows 16MiB apart", ctas,
           (double)n * 16 * 10 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
