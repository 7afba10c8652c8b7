// Do DMMA (tensor pipe) and DFMA (fp64 pipe) overlap on sm_100a?  Half the warps
// issue DMMA.8x8x4, half issue DFMA; compare against each alone.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x / 32;
  const bool do_mma = (mode == 0) || (mode == 2 && (warp & 1) == 0);
  const bool do_fma = (mode == 1) || (mode == 2 && (warp & 1) == 1);
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  double x[16];
  for (int i = 0; i < 16; ++i) x[i] = i;
  if (do_mma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  if (do_fma) {
    // same flop count per warp as the DMMA loop: 8 DMMA = 8*256 FMA per warp = 64 FMA per lane
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      int iters = 20000, blocks = 148 * 2, threads = warps * 32;
      mix<<<blocks, threads>>>(out, 100, mode);
      cudaEventRecord(e0);
      mix<<<blocks, threads>>>(out, iters, mode);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warps_busy = (mode == 2) ? warps : warps;
      double fl = 2.0 * 2048.0 * iters * blocks * warps_busy;  // each warp: 8 DMMA*256 FMA or 64 FMA*32 lanes per iter
      printf("warps/CTA=%2d mode=%s  %.2f TFLOP/s  (%.3f ms)\n", warps, mode == 0 ? "DMMA" : mode == 1 ? "DFMA" : "MIX ", fl / ms / 1e9, ms);
    }
  }
  return 0;
}
