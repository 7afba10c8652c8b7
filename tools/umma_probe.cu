// Probe: tcgen05.mma kind::i8 with the operand layouts the sliced (Ozaki) partial
// MTTKRP uses, checked against a CPU integer GEMM.
//
//   mode 0 ("left"):  A MN-major, SWIZZLE_128B (TMA box {128 m, 64 k, L planes})
//   mode 1 ("right"): A K-major,  SWIZZLE_64B  (TMA box {64 k, 128 rows, L planes})
//   B always K-major SWIZZLE_64B (TMA box {64 k, RP rows, L planes})
//
// Level-concatenated MMAs: for A slice s, D[:, s*RP : L*RP] += A_s * [B_0 | ... | B_{L-1-s}].
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

constexpr int L = 6, RP = 32, BM = 128, BK = 64;
constexpr int A_PLANE = BM * BK;        // 8 KB
constexpr int B_PLANE = RP * BK;        // 2 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  d |= (uint64_t)layout << 61;
  return d;
}

__device__ __forceinline__ uint32_t idesc_i8(int M, int N, int a_mn) {
  uint32_t d = 0;
  d |= 2u << 4;             // D = s32
  d |= 1u << 7;             // A signed
  d |= 1u << 10;            // B signed
  d |= (uint32_t)a_mn << 15;
  d |= (uint32_t)(N >> 3) << 17;
  d |= (uint32_t)(M >> 4) << 24;
  return d;
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap mapA,
                                                const __grid_constant__ CUtensorMap mapB, int mode, int m0,
                                                int* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                 // L * 8 KB
  uint8_t* sB = smem + L * A_PLANE;   // L * 2 KB
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_full)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;

  if (threadIdx.x == 0) {
    const uint32_t bytes = L * A_PLANE + L * B_PLANE;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_full)), "r"(bytes)
                 : "memory");
    if (mode == 0) {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              smem_u32(sA)),
          "l"((uint64_t)&mapA), "r"(smem_u32(&bar_full)), "r"(m0), "r"(0), "r"(0)
          : "memory");
    } else {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
              smem_u32(sA)),
          "l"((uint64_t)&mapA), "r"(smem_u32(&bar_full)), "r"(0), "r"(m0), "r"(0)
          : "memory");
    }
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(sB)),
        "l"((uint64_t)&mapB), "r"(smem_u32(&bar_full)), "r"(0), "r"(0), "r"(0)
        : "memory");
    // wait for the data
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar_full))
          : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int s = 0; s < L; ++s) {
      const int N = (L - s) * RP;
      const uint32_t id = idesc_i8(BM, N, mode == 0 ? 1 : 0);
      for (int kk = 0; kk < BK / 32; ++kk) {
        uint64_t da;
        if (mode == 0)  // MN-major SW128: 8 k-rows x 128 B atoms, SBO = 1 KB between k-groups
          da = make_desc(smem_u32(sA + s * A_PLANE + kk * 32 * 128), 0, 1024, 2);
        else            // K-major SW64: 8 rows x 64 B atoms, SBO = 512 B between row groups
          da = make_desc(smem_u32(sA + s * A_PLANE + kk * 32), 0, 512, 4);
        const uint64_t db = make_desc(smem_u32(sB + kk * 32), 0, 512, 4);
        const uint32_t dt = tbase + s * RP;
        const uint32_t acc = (s > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
            "l"(da), "l"(db), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar_mma)));
  }
  __syncwarp();
  // all warps wait for the MMA
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar_mma))
          : "memory");
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c = 0; c < L * RP; c += 8) {
    uint32_t v[8];
    const uint32_t ta = tbase + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int q = 0; q < 8; ++q) out[row * L * RP + c + q] = (int)v[q];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return (EncodeFn)p;
}

static void map3(CUtensorMap* m, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                 uint32_t b2, CUtensorMapSwizzle sw) {
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0, d0 * d1};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
}

int main() {
  int bad_total = 0;
  for (int mode = 0; mode < 2; ++mode) {
    const int M = 256, K = BK, m0 = 128;
    // global A: mode 0 -> [L][K][M] (m fastest); mode 1 -> [L][M][K] (k fastest)
    std::vector<int8_t> hA((size_t)L * M * K), hB((size_t)L * RP * K);
    srand(1234 + mode);
    for (auto& v : hA) v = (int8_t)((rand() % 256) - 128);
    for (auto& v : hB) v = (int8_t)((rand() % 256) - 128);
    auto A = [&](int s, int m, int k) {
      return mode == 0 ? (int)hA[((size_t)s * K + k) * M + m] : (int)hA[((size_t)s * M + m) * K + k];
    };
    auto B = [&](int t, int r, int k) { return (int)hB[((size_t)t * RP + r) * K + k]; };
    int8_t *dA, *dB;
    int* dO;
    CK(cudaMalloc(&dA, hA.size()));
    CK(cudaMalloc(&dB, hB.size()));
    CK(cudaMalloc(&dO, BM * L * RP * 4));
    CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
    CUtensorMap mA, mB;
    if (mode == 0)
      map3(&mA, dA, M, K, L, 128, BK, L, CU_TENSOR_MAP_SWIZZLE_128B);
    else
      map3(&mA, dA, K, M, L, BK, 128, L, CU_TENSOR_MAP_SWIZZLE_64B);
    map3(&mB, dB, K, RP, L, BK, RP, L, CU_TENSOR_MAP_SWIZZLE_64B);
    const int smem = L * A_PLANE + L * B_PLANE + 1024;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    probe<<<1, 128, smem>>>(mA, mB, mode, m0, dO);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int> hO(BM * L * RP);
    CK(cudaMemcpy(hO.data(), dO, hO.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < BM; ++i)
      for (int l = 0; l < L; ++l)
        for (int r = 0; r < RP; ++r) {
          long long ref = 0;
          for (int s = 0; s <= l; ++s) {
            const int t = l - s;
            for (int k = 0; k < K; ++k) ref += (long long)A(s, m0 + i, k) * B(t, r, k);
          }
          const int got = hO[i * L * RP + l * RP + r];
          if (got != ref) {
            if (bad < 5) printf("mode %d mismatch i=%d l=%d r=%d got %d ref %lld\n", mode, i, l, r, got, ref);
            ++bad;
          }
        }
    printf("mode %d (%s): %d mismatches of %d\n", mode, mode == 0 ? "A MN-major SW128" : "A K-major SW64", bad,
           BM * L * RP);
    bad_total += bad;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
  }
  printf(bad_total ? "PROBE FAIL\n" : "PROBE OK\n");
  return bad_total ? 1 : 0;
}
