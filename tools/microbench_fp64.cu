// FP64 peak probes for B200 (sm_100a): DFMA, DMMA (mma.sync f64), HBM streaming read.
// Used once to fix the roofline denominators in DESIGN.md; not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma16x8x8_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0, b1 = 2.0;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ p, double2* __restrict__ q, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) q[i] = __ldcs(p + i);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int bpsm = 1; bpsm <= 4; bpsm *= 2) {
    int iters = 20000, threads = 256, blocks = sms * bpsm * 2;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA blocks=%d: %.2f TFLOP/s\n", blocks, fl / ms / 1e9);
  }
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    int iters = 20000, threads = 128, blocks = sms * bpsm;
    dmma884_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma884_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA m8n8k4 blocks=%d warps/SM=%d: %.2f TFLOP/s\n", blocks, bpsm * 4, fl / ms / 1e9);
  }
  for (int bpsm = 1; bpsm <= 8; bpsm *= 2) {
    int iters = 10000, threads = 128, blocks = sms * bpsm;
    dmma16x8x8_kernel<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma16x8x8_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * 8 * 8 * 4 * (double)iters * blocks * (threads / 32);
    printf("DMMA m16n8k8 blocks=%d warps/SM=%d: %.2f TFLOP/s\n", blocks, bpsm * 4, fl / ms / 1e9);
  }
  size_t bytes = (size_t)8 << 30;
  double2 *p, *q; CK(cudaMalloc(&p, bytes)); CK(cudaMalloc(&q, bytes));
  cudaMemset(p, 0, bytes);
  size_t n = bytes / 16;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    read_kernel<<<sms * 8, 512>>>(p, n, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("HBM read: %.1f GB/s\n", bytes / ms / 1e6);
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(p, q, n);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("HBM copy (r+w): %.1f GB/s\n", 2.0 * bytes / ms / 1e6);
  }
  return 0;
}
