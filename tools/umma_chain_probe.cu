// Probe: throughput of tcgen05.mma kind::i8 (M=128, K=32) issued back to back by one
// thread, as a function of how consecutive MMAs' accumulator (TMEM) regions overlap.
//   pattern 0: every MMA accumulates into the same columns [0, N)
//   pattern 1: alternate between two disjoint regions [0, N) and [256, 256+N)
//   pattern 2: the sliced-MTTKRP level pattern: MMA s writes [s*RP, 6*RP) (N = (6-s) RP), RP=32
//   pattern 3: pattern 2 with RP = 64 (pieces of <= 256 columns)
// Operands are arbitrary shared-memory bytes (values do not matter for timing).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_chain_probe tools/umma_chain_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ uint32_t idesc(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id));
}

__global__ void probe(int pattern, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_sh)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tbase_sh;
  if (threadIdx.x == 0) {
    const uint64_t a = desc(smem_u32(sm));
    const uint64_t b = desc(smem_u32(sm + 65536));
    long long n_mma = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (pattern == 0) {
#pragma unroll
        for (int k = 0; k < 24; ++k) mma(tb, a, b, idesc(128));
        n_mma += 24;
      } else if (pattern == 1) {
#pragma unroll
        for (int k = 0; k < 24; ++k) mma(tb + (k & 1) * 256, a, b, idesc(128));
        n_mma += 24;
      } else if (pattern == 2) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
#pragma unroll
          for (int s = 0; s < 6; ++s) mma(tb + s * 32, a, b, idesc((6 - s) * 32));
        n_mma += 24;
      } else {
#pragma unroll
        for (int s = 0; s < 6; ++s)
#pragma unroll
          for (int n0 = 0; n0 < (6 - s) * 64; n0 += 256)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const int nn = (6 - s) * 64 - n0 < 256 ? (6 - s) * 64 - n0 : 256;
              mma(tb + s * 64 + n0, a, b, idesc(nn));
            }
        n_mma += 32;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar))
          : "memory");
    const long long t1 = clock64();
    out[0] = t1 - t0;
    out[1] = n_mma;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[4] = {"same D, N=128", "two disjoint D, N=128", "level pattern RP=32 (N=192..32)",
                          "level pattern RP=64 (pieces)"};
  // MACs per pattern iteration: 24 * 128 * N * 32 etc.
  const double macs[4] = {24.0 * 128 * 128 * 32, 24.0 * 128 * 128 * 32, 4.0 * 128 * 32 * 32 * 21,
                          4.0 * 128 * 32 * 64 * 21};
  for (int p = 0; p < 4; ++p) {
    const int iters = 2000;
    probe<<<148, 128, 140 * 1024>>>(p, iters, d);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-36s %8.1f cycles/MMA  %8.0f int8 MAC/cycle  (err %s)\n", names[p], double(h[0]) / h[1],
           macs[p] * iters / double(h[0]), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
