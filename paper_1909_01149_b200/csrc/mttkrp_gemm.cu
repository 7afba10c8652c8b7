// Partial MTTKRP (dimtree.py:102-127) as FP64 tensor-core GEMMs for sm_100a.
//
//   left : T_L[m, r] = sum_k X[m + M k] * KRP(H_{S+1..N})[k, r]     (X_(1:S) . KRP)
//   right: T_R[j, r] = sum_m X[m + M j] * KRP(H_{1..S})[m, r]       (X_(1:S)^T . KRP)
//
// X stays in the reference layout (flat, mode-1 fastest), so X_(1:S) is a
// column-major M x J matrix that a 2-D TMA descriptor addresses directly.
// Design:
//   * one producer warp per CTA: issues the TMA tile load of X for each pipeline
//     stage and generates that stage's Khatri-Rao rows on the fly into shared
//     memory (fragment-native layout) -- the KRP is never materialised in HBM;
//   * eight consumer warps run mma.sync m8n8k4 f64 (SASS DMMA.8x8x4, the only FP64
//     tensor path on sm_100a), accumulators in registers;
//   * mbarrier full/empty ring between producer and consumers (no CTA barriers in
//     the main loop);
//   * deterministic split-K (partials + fixed-order reduce) when the output tile
//     count cannot fill 148 SMs.
#include "common.cuh"

namespace nncp {

struct KrpSpec {
  const double* ptr[kMaxOrder];
  int64_t dim[kMaxOrder];
  int n;
};

// KRP row `k` (first listed factor fastest, tensor_ops.py:121-137), column r.
// Multiplication order ((H_a * H_b) * H_c) reproduces khatri_rao's rounding.
__device__ __forceinline__ double krp_value(const KrpSpec& s, int64_t k, int r, int R) {
  double v = 1.0;
#pragma unroll 1
  for (int f = 0; f < s.n - 1; ++f) {
    const int64_t d = s.dim[f];
    const int64_t q = k / d;
    v *= __ldg(s.ptr[f] + (k - q * d) * R + r);
    k = q;
  }
  return v * __ldg(s.ptr[s.n - 1] + k * R + r);
}


// Per-lane cursor over the U Khatri-Rao rows a producer lane fills in every stage.
// Row k is kept both linear (for the range check) and as its mixed-radix digits
// (first factor fastest), advanced by a fixed stride per stage: no 64-bit
// divisions in the steady state, so every factor load of a stage can be issued
// back to back (one L2 round trip per stage).
template <int U, int NFM>
struct KrpCursor {
  int64_t k[U];
  uint32_t dig[U][NFM];

  // factor count: compile-time when the launcher dispatched an exact NFM (1 or 2)
  __device__ __forceinline__ static int count(const KrpSpec& s) { return NFM <= 2 ? NFM : s.n; }

  template <class IdxFn>
  __device__ __forceinline__ void init(const KrpSpec& s, IdxFn idx_of, int c) {
    const int n = count(s);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      k[u] = idx_of(u, c);
      int64_t q = k[u];
#pragma unroll
      for (int f = 0; f < NFM; ++f) {
        const bool act = f < n, last = f == n - 1;
        const int64_t d = (act && !last) ? s.dim[f] : 1;
        const int64_t r = q % d;
        dig[u][f] = act ? uint32_t(last ? q : r) : 0u;
        q = (act && !last) ? q / d : q;
      }
    }
  }

  __device__ __forceinline__ void advance(const KrpSpec& s, uint32_t step) {
    const int n = count(s);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      k[u] += step;
      uint32_t carry = step;
#pragma unroll
      for (int f = 0; f < NFM; ++f) {
        const bool act = f < n, last = f == n - 1;
        uint32_t v = dig[u][f] + carry;
        carry = 0;
        if (act && !last) {
          const uint32_t d = uint32_t(s.dim[f]);
          if (v >= d) {
            carry = v / d;
            v -= carry * d;
          }
        }
        dig[u][f] = act ? v : 0u;
      }
    }
  }
};

// One pipeline stage of fragment-native Khatri-Rao values: for k4-step u < U and
// n-fragment j < NF, lane (g, c) writes KRP[row(u, c)][8j + g] (zero when the row
// is >= hi or the column >= R).  Multiplication order ((H_a * H_b) * H_c) is
// khatri_rao's (tensor_ops.py:121-137).
template <int NF, int U, int NFM>
struct KrpRaw {
  double f[U][NFM][NF];  // raw factor entries of one stage, loaded ahead of their use
};

// Issue every factor load of one stage (no use yet: the loads stay in flight while
// the producer waits for the stage's empty barrier).
template <int NF, int U, int NFM>
__device__ __forceinline__ void krp_load(const KrpSpec& krp, const KrpCursor<U, NFM>& cur, int lane, int R,
                                         int64_t hi, KrpRaw<NF, U, NFM>& raw) {
  const int g = lane >> 2;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool in = cur.k[u] < hi;
#pragma unroll
    for (int f = 0; f < NFM; ++f) {
      if (f < KrpCursor<U, NFM>::count(krp)) {
        const double* base = krp.ptr[f] + (in ? int64_t(cur.dig[u][f]) * R : 0);
#pragma unroll
        for (int j = 0; j < NF; ++j) raw.f[u][f][j] = __ldg(base + min(8 * j + g, R - 1));
      }
    }
  }
}

// Multiply the raw entries into KRP values (order (H_a * H_b) * H_c, as khatri_rao)
// and write them in the fragment-native layout: k4-step u, n-fragment j, lane (g, c)
// holds KRP[row(u, c)][8j + g]; zero outside the row range or beyond R.
template <int NF, int U, int NFM>
__device__ __forceinline__ void krp_store(const KrpSpec& krp, const KrpCursor<U, NFM>& cur,
                                          const KrpRaw<NF, U, NFM>& raw, double* __restrict__ bdst, int lane, int R,
                                          int64_t hi) {
  const int g = lane >> 2;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool in = cur.k[u] < hi;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      double v = 1.0;
#pragma unroll
      for (int f = 0; f < NFM; ++f)
        if (f < KrpCursor<U, NFM>::count(krp)) v *= raw.f[u][f][j];
      bdst[(u * NF + j) * 32 + lane] = (in && 8 * j + g < R) ? v : 0.0;
    }
  }
}

// Producer warps per CTA: each generates 1/PRODUCERS of every stage's KRP rows.
// A producer warp is bound by one L2 round trip per stage (the factor rows do
// not fit the ~7 KB of L1 left next to the pipeline), so stages are split
// across warps until the consumers, not the producers, set the pace.

// Deferred stage release.  A consumer warp frees the stage it read in the previous
// chunk only after the next chunk's full barrier fired: by then every DMMA of that
// chunk has issued (the loop back-edge and the wait keep ptxas from hoisting the
// arrive above them), so all of its ld.shared results have landed and the TMA
// refill cannot overwrite data still being read.  (An arrive placed right after
// the last k-step raced its in-flight loads: tools/debug_left.py.)  The final
// release of a CTA goes through a proxy fence instead.
__device__ __forceinline__ void release_stage(uint64_t* empty, int& pending, int lane) {
  if (pending >= 0) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[pending]);
    pending = -1;
  }
}

// ------------------------------------------------------------ left side ----
template <int RP>
struct LeftTile {
  static constexpr int BM = 256;  // tensor rows (retained leading modes) per CTA
  static constexpr int BK = 16;   // contracted columns per stage
  static constexpr int NF = RP / 8;
  // HBM-bound ranks (RP <= 24) keep one more stage in flight
  static constexpr int STAGES = (RP <= 24) ? 6 : (RP <= 32) ? 5 : 4;
  static constexpr int PRODUCERS = 4;
  static constexpr int THREADS = 256 + 32 * PRODUCERS;
  static constexpr int A_ELEMS = BM * BK;
  static constexpr int B_ELEMS = BK * RP;
  static constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * 8 + 2 * STAGES * 8;
};

// Persistent: gridDim.x <= SM count CTAs loop over work items (row tile, K split)
// in round-robin order; the producer/consumer ring runs continuously across items,
// so a short contraction (c4: K = 256) does not pay a pipeline fill per tile.  The
// epilogue stores straight from the accumulator registers (the smem ring is already
// being refilled with the next item's stages).
template <int RP, int NFM>
__global__ void __launch_bounds__(LeftTile<RP>::THREADS, 1)
    mttkrp_left_tma(const __grid_constant__ CUtensorMap xmap, const KrpSpec krp, const int64_t M,
                    const int64_t K, const int64_t k_per_split, const int64_t tiles, const int64_t items,
                    double* __restrict__ out, const int64_t split_stride, const int R) {
  using T = LeftTile<RP>;
  constexpr int BM = T::BM, BK = T::BK, NF = T::NF, ST = T::STAGES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + ST * T::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + ST * T::B_ELEMS);
  uint64_t* empty = full + ST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 32 * T::PRODUCERS + 1);  // producer lanes + the expect_tx arrival
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) prefetch_tma_desc(&xmap);
  const int pw = warp - 8;  // producer warp index (>= 0 for producers)
  __syncthreads();

  if (warp >= 8) {
    // ---------------- producers: TMA for X, on-the-fly KRP rows for B ---------
    constexpr int UP = BK / 4 / T::PRODUCERS;
    static_assert(UP * T::PRODUCERS == BK / 4, "stage steps must split evenly");
    uint32_t gch = 0;  // chunks produced by this CTA so far (ring position)
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
      const int64_t m0 = (w % tiles) * BM;
      const int64_t kb = (w / tiles) * k_per_split;
      const int64_t ke = min(K, kb + k_per_split);
      const int nchunks = int((ke - kb + BK - 1) / BK);
      KrpCursor<UP, NFM> cur;
      cur.init(krp, [&](int t, int cc) { return kb + 4 * (t + pw * UP) + cc; }, lane & 3);
      KrpRaw<NF, UP, NFM> raw;
      krp_load<NF, UP, NFM>(krp, cur, lane, R, ke, raw);
      for (int ch = 0; ch < nchunks; ++ch, ++gch) {
        const int s = int(gch % ST);
        if (gch >= uint32_t(ST)) mbar_wait(&empty[s], ((gch / ST) - 1) & 1);
        const int64_t k0 = kb + int64_t(ch) * BK;
        if (pw == 0 && lane == 0) {
          // one arrival that also arms the transaction count, ordered before the copy
          mbar_arrive_expect_tx(&full[s], uint32_t(T::A_ELEMS * 8));
          tma_load_2d(As + s * T::A_ELEMS, &xmap, &full[s], int(m0), int(k0));
        }
        krp_store<NF, UP, NFM>(krp, cur, raw, Bs + s * T::B_ELEMS + pw * UP * NF * 32, lane, R, ke);
        mbar_arrive(&full[s]);
        cur.advance(krp, BK);
        if (ch + 1 < nchunks) krp_load<NF, UP, NFM>(krp, cur, lane, R, ke, raw);  // next stage, in flight
      }
    }
    // producer tail: stay resident until the consumers released every stage
    for (uint32_t q = gch > uint32_t(ST) ? gch - ST : 0; q < gch; ++q) mbar_wait(&empty[q % ST], (q / ST) & 1);
    return;
  }

  // ---------------- consumers: DMMA over the staged tiles ---------------------
  uint32_t gch = 0;
  int pending = -1;  // stage read in the previous chunk, released once the next one is ready
  for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
    const int64_t m0 = (w % tiles) * BM;
    const int64_t kb = (w / tiles) * k_per_split;
    const int64_t ke = min(K, kb + k_per_split);
    const int nchunks = int((ke - kb + BK - 1) / BK);
    double acc[4][NF][2];
#pragma unroll
    for (int f = 0; f < 4; ++f)
#pragma unroll
      for (int j = 0; j < NF; ++j) acc[f][j][0] = acc[f][j][1] = 0.0;

    for (int ch = 0; ch < nchunks; ++ch, ++gch) {
      const int s = int(gch % ST);
      mbar_wait(&full[s], (gch / ST) & 1);
      release_stage(empty, pending, lane);
      const double* as = As + s * T::A_ELEMS + warp * 32 + 2 * g;
      const double* bs = Bs + s * T::B_ELEMS + lane;
#pragma unroll
      for (int t = 0; t < BK / 4; ++t) {
        double a[4], b[NF];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          // fragment rows: frag 2p row g <-> m = 16p + 2g, frag 2p+1 row g <-> m = 16p + 2g + 1
          const double2 v = *reinterpret_cast<const double2*>(as + (4 * t + c) * BM + 16 * p);
          a[2 * p] = v.x;
          a[2 * p + 1] = v.y;
        }
#pragma unroll
        for (int j = 0; j < NF; ++j) b[j] = bs[(t * NF + j) * 32];
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
          for (int j = 0; j < NF; ++j) dmma884(acc[f][j][0], acc[f][j][1], a[f], b[j]);
      }
      pending = s;
    }

    // ---------------- epilogue: accumulator registers -> HBM ------------------
    // lanes of a store cover 8 rows (stride 2) x 4 columns; the (f, f^1) pair fills
    // each 32-byte sector, merged in L2 before write-back.
    double* o = out + (w / tiles) * split_stride;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int64_t m = m0 + warp * 32 + (f >> 1) * 16 + 2 * g + (f & 1);
      if (m < M) {
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          const int r = 8 * j + 2 * c;
          if (r < R) o[m + M * r] = acc[f][j][0];
          if (r + 1 < R) o[m + M * (r + 1)] = acc[f][j][1];
        }
      }
    }
  }
  fence_proxy_async();
  release_stage(empty, pending, lane);
}

// ------------------------------------------------------------ right side ---
template <int RP>
struct RightTile {
  static constexpr int BJ = 256;   // retained trailing-mode columns per CTA
  static constexpr int BMC = 24;   // contracted rows per stage (pitch 192 B: conflict-free)
  static constexpr int KSTEPS = BMC / 4;
  static constexpr int NF = RP / 8;
  static constexpr int STAGES = (RP <= 32) ? 4 : 3;
  static constexpr int PRODUCERS = (RP <= 32) ? 6 : 3;
  static constexpr int THREADS = 256 + 32 * PRODUCERS;
  static constexpr int A_ELEMS = BJ * BMC;
  static constexpr int B_ELEMS = KSTEPS * NF * 32;
  static constexpr size_t SMEM = size_t(STAGES) * (A_ELEMS + B_ELEMS) * 8 + 2 * STAGES * 8;
  static_assert(size_t(RP) * BJ * 8 <= size_t(STAGES) * A_ELEMS * 8, "epilogue tile must fit");
};

template <int RP, int NFM>
__global__ void __launch_bounds__(RightTile<RP>::THREADS, 1)
    mttkrp_right_tma(const __grid_constant__ CUtensorMap xmap, const KrpSpec krp, const int64_t M,
                     const int64_t J, const int64_t m_per_split, double* __restrict__ out,
                     const int64_t split_stride, const int R) {
  using T = RightTile<RP>;
  constexpr int BJ = T::BJ, BMC = T::BMC, NF = T::NF, ST = T::STAGES;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + ST * T::A_ELEMS;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + ST * T::B_ELEMS);
  uint64_t* empty = full + ST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int64_t j0 = int64_t(blockIdx.x) * BJ;
  const int64_t mb = int64_t(blockIdx.y) * m_per_split;
  const int64_t me = min(M, mb + m_per_split);
  const int nchunks = int((me - mb + BMC - 1) / BMC);

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 32 * T::PRODUCERS + 1);  // producer lanes + the expect_tx arrival
      mbar_init(&empty[s], 8);
    }
    fence_barrier_init();
  }
  if (warp == 8 && lane == 0) prefetch_tma_desc(&xmap);
  const int pw = warp - 8;  // producer warp index (>= 0 for producers)
  __syncthreads();

  if (warp >= 8) {
    constexpr int UP = T::KSTEPS / T::PRODUCERS;
    static_assert(UP * T::PRODUCERS == T::KSTEPS, "stage steps must split evenly");
    KrpCursor<UP, NFM> cur;
    cur.init(krp, [&](int u, int cc) {
      const int uu = u + pw * UP;
      return mb + 8 * (uu >> 1) + 2 * cc + (uu & 1);
    }, lane & 3);
    KrpRaw<NF, UP, NFM> raw;
    krp_load<NF, UP, NFM>(krp, cur, lane, R, me, raw);
    for (int ch = 0; ch < nchunks; ++ch) {
      const int s = ch % ST;
      if (ch >= ST) mbar_wait(&empty[s], ((ch / ST) - 1) & 1);
      const int64_t mc = mb + int64_t(ch) * BMC;
      if (pw == 0 && lane == 0) {
        // one arrival that also arms the transaction count, ordered before the copy
        mbar_arrive_expect_tx(&full[s], uint32_t(T::A_ELEMS * 8));
        tma_load_2d(As + s * T::A_ELEMS, &xmap, &full[s], int(mc), int(j0));
      }
      // k4-step u: fragment column c <-> m = 8 (u/2) + 2c + (u&1)
      krp_store<NF, UP, NFM>(krp, cur, raw, Bs + s * T::B_ELEMS + pw * UP * NF * 32, lane, R, me);
      mbar_arrive(&full[s]);
      cur.advance(krp, BMC);
      if (ch + 1 < nchunks) krp_load<NF, UP, NFM>(krp, cur, lane, R, me, raw);  // next stage, in flight
    }
    // producer tail: stay resident until the consumers released every stage
    for (int ch = max(0, nchunks - ST); ch < nchunks; ++ch) mbar_wait(&empty[ch % ST], (ch / ST) & 1);
    return;
  }

  double acc[4][NF][2];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[f][j][0] = acc[f][j][1] = 0.0;

  int pending = -1;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int s = ch % ST;
    mbar_wait(&full[s], (ch / ST) & 1);
    release_stage(empty, pending, lane);
    const double* as = As + s * T::A_ELEMS + (warp * 32 + g) * BMC + 2 * c;
    const double* bs = Bs + s * T::B_ELEMS + lane;
#pragma unroll
    for (int k8 = 0; k8 < BMC / 8; ++k8) {
      double alo[4], ahi[4], blo[NF], bhi[NF];
#pragma unroll
      for (int f = 0; f < 4; ++f) {
        const double2 v = *reinterpret_cast<const double2*>(as + f * 8 * BMC + 8 * k8);
        alo[f] = v.x;
        ahi[f] = v.y;
      }
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        blo[j] = bs[((2 * k8) * NF + j) * 32];
        bhi[j] = bs[((2 * k8 + 1) * NF + j) * 32];
      }
      // all independent "lo" products first: back-to-back lo/hi on one accumulator
      // would serialise on the DMMA latency (the asm statements are not reordered)
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma884(acc[f][j][0], acc[f][j][1], alo[f], blo[j]);
#pragma unroll
      for (int f = 0; f < 4; ++f)
#pragma unroll
        for (int j = 0; j < NF; ++j) dmma884(acc[f][j][0], acc[f][j][1], ahi[f], bhi[j]);
    }
    pending = s;
  }
  fence_proxy_async();
  release_stage(empty, pending, lane);

  named_bar_sync(1, 256);
  double* Cs = As;
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int jl = warp * 32 + f * 8 + g;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      Cs[(8 * j + 2 * c) * BJ + jl] = acc[f][j][0];
      Cs[(8 * j + 2 * c + 1) * BJ + jl] = acc[f][j][1];
    }
  }
  named_bar_sync(1, 256);
  double* o = out + int64_t(blockIdx.y) * split_stride;
  const int jl = threadIdx.x;
  if (j0 + jl < J) {
    for (int r = 0; r < R; ++r) o[j0 + jl + J * r] = Cs[r * BJ + jl];
  }
}

// ------------------------------------------------- generic (any shape) -----
// Plain SIMT kernels for shapes the TMA path does not take (odd leading extent,
// tiny tensors).  Same algebra, fixed summation order.
__global__ void mttkrp_left_simt(const double* __restrict__ x, const KrpSpec krp, int64_t M, int64_t K,
                                 double* __restrict__ out, int R) {
  const int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (m >= M) return;
  double s = 0.0;
  for (int64_t k = 0; k < K; ++k) s = fma(x[m + M * k], krp_value(krp, k, r, R), s);
  out[m + M * r] = s;
}

__global__ void mttkrp_right_simt(const double* __restrict__ x, const KrpSpec krp, int64_t M, int64_t J,
                                  double* __restrict__ out, int R) {
  const int64_t j = blockIdx.x;
  const int r = blockIdx.y;
  double s = 0.0;
  for (int64_t m = threadIdx.x; m < M; m += 32) s = fma(x[m + M * j], krp_value(krp, m, r, R), s);
  s = warp_sum(s);
  if (threadIdx.x == 0) out[j + J * r] = s;
}

__global__ void splitk_reduce(const double* __restrict__ part, int splits, int64_t stride, int64_t n,
                              double* __restrict__ out) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    double s = part[e];
    for (int k = 1; k < splits; ++k) s += part[int64_t(k) * stride + e];
    out[e] = s;
  }
}

// ------------------------------------------------------------- host side ---
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

namespace {

int make_map_2d(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                uint32_t box_outer) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * sizeof(double)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return NNCP_OK;
}

}  // namespace

// Split-K chooser: the smallest split count whose CTA waves (1 resident CTA per
// SM) come within 1% of the best achievable SM fill, keeping >= 8 pipeline
// chunks per split.
int choose_splits(int64_t tiles, int64_t chunks) {
  const int64_t sms = num_sms();
  const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(chunks / 8, 4 * sms));
  double best_eff = 0.0;
  for (int64_t s = 1; s <= max_s; ++s) {
    const int64_t ctas = tiles * s;
    const int64_t waves = (ctas + sms - 1) / sms;
    best_eff = std::max(best_eff, double(ctas) / double(waves * sms));
  }
  for (int64_t s = 1; s <= max_s; ++s) {
    const int64_t ctas = tiles * s;
    const int64_t waves = (ctas + sms - 1) / sms;
    if (double(ctas) / double(waves * sms) >= best_eff - 0.01) return int(s);
  }
  return 1;
}

struct PartialPlan {
  bool tma;
  int64_t M, J;  // X_(1:S) is M x J (column-major)
  int rp;
  int64_t tiles, chunks, per_split;
  int splits;
  size_t ws_bytes;
};

PartialPlan plan_partial(int order, const int64_t* dims, int split, int side, int rank, const void* x) {
  PartialPlan p{};
  p.M = 1;
  p.J = 1;
  for (int n = 0; n < split; ++n) p.M *= dims[n];
  for (int n = split; n < order; ++n) p.J *= dims[n];
  p.rp = pad8(rank);
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16) == 0;
  p.tma = aligned && (p.M % 2 == 0) && p.M >= 64 && p.M < (int64_t(1) << 31) && p.J < (int64_t(1) << 31);
  p.splits = 1;
  p.ws_bytes = 0;
  if (!p.tma) return p;
  if (side == NNCP_SIDE_LEFT) {
    p.tiles = (p.M + 255) / 256;
    p.chunks = (p.J + 15) / 16;
    p.splits = choose_splits(p.tiles, p.chunks);
    p.per_split = ((p.chunks + p.splits - 1) / p.splits) * 16;
    p.splits = int((p.J + p.per_split - 1) / p.per_split);
    if (p.splits > 1) p.ws_bytes = size_t(p.splits) * p.M * rank * sizeof(double);
  } else {
    p.tiles = (p.J + 255) / 256;
    p.chunks = (p.M + 23) / 24;
    p.splits = choose_splits(p.tiles, p.chunks);
    p.per_split = ((p.chunks + p.splits - 1) / p.splits) * 24;
    p.splits = int((p.M + p.per_split - 1) / p.per_split);
    if (p.splits > 1) p.ws_bytes = size_t(p.splits) * p.J * rank * sizeof(double);
  }
  return p;
}

template <int RP, int NFM>
int launch_left_nf(const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst, int64_t stride,
                   int R, cudaStream_t st) {
  using T = LeftTile<RP>;
  if (int rc = set_max_smem_once<mttkrp_left_tma<RP, NFM>>(int(T::SMEM))) return rc;
  const int64_t items = p.tiles * p.splits;
  const unsigned ctas = unsigned(std::min<int64_t>(items, num_sms()));
  mttkrp_left_tma<RP, NFM><<<ctas, T::THREADS, T::SMEM, st>>>(map, krp, p.M, p.J, p.per_split, p.tiles, items, dst,
                                                              stride, R);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

template <int RP, int NFM>
int launch_right_nf(const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst, int64_t stride,
                    int R, cudaStream_t st) {
  using T = RightTile<RP>;
  if (int rc = set_max_smem_once<mttkrp_right_tma<RP, NFM>>(int(T::SMEM))) return rc;
  dim3 grid(unsigned(p.tiles), unsigned(p.splits));
  mttkrp_right_tma<RP, NFM><<<grid, T::THREADS, T::SMEM, st>>>(map, krp, p.M, p.J, p.per_split, dst, stride, R);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

template <int RP>
int launch_left(const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst, int64_t stride, int R,
                cudaStream_t st) {
  if (krp.n == 1) return launch_left_nf<RP, 1>(map, krp, p, dst, stride, R, st);
  if (krp.n == 2) return launch_left_nf<RP, 2>(map, krp, p, dst, stride, R, st);
  if (krp.n <= 4) return launch_left_nf<RP, 4>(map, krp, p, dst, stride, R, st);
  return launch_left_nf<RP, kMaxOrder>(map, krp, p, dst, stride, R, st);
}

template <int RP>
int launch_right(const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst, int64_t stride,
                 int R, cudaStream_t st) {
  if (krp.n == 1) return launch_right_nf<RP, 1>(map, krp, p, dst, stride, R, st);
  if (krp.n == 2) return launch_right_nf<RP, 2>(map, krp, p, dst, stride, R, st);
  if (krp.n <= 4) return launch_right_nf<RP, 4>(map, krp, p, dst, stride, R, st);
  return launch_right_nf<RP, kMaxOrder>(map, krp, p, dst, stride, R, st);
}

#define NNCP_RP_DISPATCH(RPV, FN, ...)                  \
  switch (RPV) {                                        \
    case 8: return FN<8>(__VA_ARGS__);                  \
    case 16: return FN<16>(__VA_ARGS__);                \
    case 24: return FN<24>(__VA_ARGS__);                \
    case 32: return FN<32>(__VA_ARGS__);                \
    case 40: return FN<40>(__VA_ARGS__);                \
    case 48: return FN<48>(__VA_ARGS__);                \
    case 56: return FN<56>(__VA_ARGS__);                \
    case 64: return FN<64>(__VA_ARGS__);                \
    default: return fail(NNCP_ERR_UNSUPPORTED, "rank above NNCP_MAX_RANK"); \
  }

int partial_finish(const PartialPlan& p, int side, int rank, double* out, const void* ws, cudaStream_t st) {
  if (!p.tma || p.splits <= 1) return NNCP_OK;
  const int64_t outn = (side == NNCP_SIDE_LEFT ? p.M : p.J) * rank;
  const int blocks = int(std::min<int64_t>((outn + 255) / 256, int64_t(num_sms()) * 8));
  splitk_reduce<<<blocks, 256, 0, st>>>(static_cast<const double*>(ws), p.splits, outn, outn, out);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int dispatch_left(int rp, const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst,
                  int64_t stride, int R, cudaStream_t st) {
  NNCP_RP_DISPATCH(rp, launch_left, map, krp, p, dst, stride, R, st);
}

int dispatch_right(int rp, const CUtensorMap& map, const KrpSpec& krp, const PartialPlan& p, double* dst,
                   int64_t stride, int R, cudaStream_t st) {
  NNCP_RP_DISPATCH(rp, launch_right, map, krp, p, dst, stride, R, st);
}

int partial_mttkrp(const double* x, int order, const int64_t* dims, int split, int side,
                   const double* const* factors, int rank, double* out, void* ws, size_t ws_bytes,
                   cudaStream_t st) {
  PartialPlan p = plan_partial(order, dims, split, side, rank, x);
  KrpSpec krp{};
  if (side == NNCP_SIDE_LEFT) {
    krp.n = order - split;
    for (int f = 0; f < krp.n; ++f) {
      krp.ptr[f] = factors[split + f];
      krp.dim[f] = dims[split + f];
    }
  } else {
    krp.n = split;
    for (int f = 0; f < krp.n; ++f) {
      krp.ptr[f] = factors[f];
      krp.dim[f] = dims[f];
    }
  }
  for (int f = 0; f < krp.n; ++f)
    if (!krp.ptr[f]) return fail(NNCP_ERR_VALUE, "null factor pointer on the contracted side");
  if (!p.tma) {
    if (side == NNCP_SIDE_LEFT) {
      dim3 grid(unsigned((p.M + 127) / 128), unsigned(rank));
      mttkrp_left_simt<<<grid, 128, 0, st>>>(x, krp, p.M, p.J, out, rank);
    } else {
      dim3 grid(unsigned(p.J), unsigned(rank));
      mttkrp_right_simt<<<grid, 32, 0, st>>>(x, krp, p.M, p.J, out, rank);
    }
    NNCP_LAUNCH_CHECK();
    return NNCP_OK;
  }
  if (p.splits > 1 && (ws == nullptr || ws_bytes < p.ws_bytes))
    return fail(NNCP_ERR_VALUE, "workspace too small for split-K partial MTTKRP");
  CUtensorMap map;
  int rc;
  const int64_t outn = (side == NNCP_SIDE_LEFT ? p.M : p.J) * rank;
  double* dst = p.splits > 1 ? static_cast<double*>(ws) : out;
  if (side == NNCP_SIDE_LEFT) {
    rc = make_map_2d(&map, x, uint64_t(p.M), uint64_t(p.J), 256, 16);
    if (rc) return rc;
    rc = dispatch_left(p.rp, map, krp, p, dst, outn, rank, st);
  } else {
    rc = make_map_2d(&map, x, uint64_t(p.M), uint64_t(p.J), 24, 256);
    if (rc) return rc;
    rc = dispatch_right(p.rp, map, krp, p, dst, outn, rank, st);
  }
  if (rc) return rc;
  return partial_finish(p, side, rank, out, ws, st);
}

}  // namespace nncp

namespace nncp {
size_t partial_ws_bytes(int order, const int64_t* dims, int split, int side, int rank) {
  // alignment of x is unknown here; assume aligned (the TMA path is the only user)
  static const double dummy[2] = {0, 0};
  PartialPlan p = plan_partial(order, dims, split, side, rank, dummy);
  return p.ws_bytes;
}
}  // namespace nncp
