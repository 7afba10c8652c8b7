// Sustained FP64 tensor (DMMA) throughput: back-to-back launches for ~4 s under the
// 1000 W power cap (the burst figure is in microbench_fp64.cu).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 2, threads = 256, iters = 100000;
  dmma_loop<<<blocks, threads>>>(out, 1000);
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    int launches = 0;
    float ms = 0;
    while (ms < 1000.0f) {
      for (int k = 0; k < 4; ++k) dmma_loop<<<blocks, threads>>>(out, iters);
      launches += 4;
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    double fl = 2.0 * 2048.0 * iters * blocks * (threads / 32.0) * launches;
    printf("sustained window %d: %.2f TFLOP/s over %.0f ms\n", rep, fl / ms / 1e9, ms);
  }
  return 0;
}
