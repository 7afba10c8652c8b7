// Sliced-operand partial MTTKRP on the int8 tensor cores (tcgen05.mma kind::i8).
//
// Same contraction as mttkrp_gemm.cu (dimtree.py:102-127):
//   left : T_L[m, r] = sum_j X[m + M j] * KRP(H_{S+1..N})[j, r]
//   right: T_R[j, r] = sum_m X[m + M j] * KRP(H_{1..S})[m, r]
// computed as an exact integer GEMM over fixed-point digit slices (the Ozaki
// scheme), because FP64 has no tcgen05 kind and DMMA (37 TF/s) caps the FP64
// path below the HBM roofline at R >= 23:
//
//   * X_(1:S) is sliced ONCE per run (the tensor is constant across ALS
//     iterations): row m gets a power-of-two scale 2^ex[m] >= max_j |X[m, j]|,
//     and X[m, j] / 2^ex[m] is rounded to 8L-2 fractional bits and written as L
//     balanced base-256 digits d_s in [-128, 127] (one int8 plane per digit):
//       X[m, j] ~= 2^ex[m] * sum_s d_s[m, j] 2^(-8s-6)      |error| <= 2^(ex-8L+1)
//   * the factor side B (the Khatri-Rao rows; for the right side scaled by
//     2^ex[m]) is sliced per call with one exponent per (column r, contraction
//     chunk of <= 16384 rows);
//   * per contraction chunk the tensor cores accumulate, exactly in int32 TMEM
//     columns, the L "levels" l = s + t < L of digit products.  One MMA per X
//     digit s covers all its partners t at once: B's digit planes are
//     concatenated along N, so  D[:, s*RP .. L*RP) += A_s * [B_0 | .. | B_{L-1-s}];
//   * an epilogue warpgroup converts each chunk's levels to fp64,
//     sum_l acc_l 2^(-8l-12) * 2^(ex + eb), and accumulates in registers (fixed
//     order: bitwise deterministic run to run).
// Products and sums in the MMA are exact; the only rounding is the digit
// truncation (relative 2^(1-8L) of the row / column-chunk maxima) and the fp64
// epilogue (DESIGN.md §4.4 for the bound and the parity tolerance it meets).
//
// HBM layout of the digit planes: 128 x 128 blocks, block (mb, jb) holding
// rows m in [128 mb, +128) and columns j in [128 jb, +128) of every plane as
// L contiguous 16 KB tiles ([s][j % 128][m % 128]); blocks ordered (mb, jb).
// One tile is one A operand stage of BOTH sides -- MN-major for the left
// (m contiguous = the MMA's M), K-major for the right (m = the contraction) --
// and every TMA request is one contiguous 16 KB run of HBM.  The left streams
// its m block's 96 KB blocks back to back; the right streams 96 KB per k step.
// Bytes per partial: L per tensor element (6 at L = 6) instead of fp64's 8.
//
// Kernel anatomy (one CTA per SM, persistent over output tiles / split-K items):
//   warp 0      TMA producer: per 128-deep k block one B stage (the L*RP digit
//               rows, 128 B each) and L A stages (one digit plane tile each);
//   warp 1      TMEM allocator + single-thread MMA issuer (tcgen05.mma, commits to
//               mbarriers: stage release and accumulator-ready);
//   warps 2..5  epilogue: tcgen05.ld of the level accumulators (double-buffered in
//               TMEM when 2 L RP <= 512 columns), fp64 conversion, output stores.
#include "nnls_common.cuh"

namespace nncp {
namespace sliced {

constexpr int BM = 128;                 // UMMA M: output rows per tile
constexpr int BK = 128;                 // contraction elements (int8 bytes) per k block
constexpr int TILE = BM * BK;           // bytes of one digit-plane tile (16 KB)
constexpr int64_t KC_MAX = 16384;       // contraction chunk between int32 -> fp64 conversions
                                        // (multiple of 256; L * 2^14 * KC_MAX < 2^31 keeps int32 exact)
constexpr int THREADS = 320;          // TMA warp, MMA warp, 8 epilogue warps
constexpr int MAX_SMEM = 227 * 1024;

__host__ __device__ constexpr int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// ----------------------------------------------------------------- layout --
struct TensorLayout {
  int64_t M, J, Mp, Jp, nmb, njb;
  int L;
  size_t rmax_off, plane_off, total;
};

TensorLayout tensor_layout(int order, const int64_t* dims, int split, int L) {
  TensorLayout t{};
  t.M = 1;
  t.J = 1;
  for (int n = 0; n < split; ++n) t.M *= dims[n];
  for (int n = split; n < order; ++n) t.J *= dims[n];
  t.Mp = align_up(t.M, BM);
  t.Jp = align_up(t.J, BK);
  t.nmb = t.Mp / BM;
  t.njb = t.Jp / BK;
  t.L = L;
  // [int32 row exponents][uint64 row maxima (slicing scratch)][blocked digit planes]
  t.rmax_off = size_t(align_up(t.Mp * int64_t(sizeof(int)), 1024));
  t.plane_off = t.rmax_off + size_t(align_up(t.Mp * 8, 1024));
  t.total = t.plane_off + size_t(L) * size_t(t.Mp) * size_t(t.Jp);
  return t;
}

// ---------------------------------------------------------------- digits --
// Digits.  q = round(v 2^k) (|q| <= 2^(8L-2)) has the balanced base-256 digits
// q = sum_s d_s 256^(L-1-s), d_0 in [-65, 65], d_1.. in [-128, 127].  Adding
// C = 0x80..80 (L-1 bytes of 128) makes every lower byte of u = q + C equal to
// d_s + 128 with no carries, and u >> 8(L-1) = d_0; the int8 bit pattern of d_s
// is then (byte of u) ^ 0x80.  slice_halves returns the two 32-bit halves of u
// (for L <= 6 straight from one FP64 add: |u| < 2^51 rounds q to nearest even
// into the low mantissa bits of u + 1.5 * 2^52).
template <int L>
__device__ __forceinline__ void slice_halves(double scaled, int& lo, int& hi) {
  constexpr unsigned long long C = (1ull << (8 * (L - 1))) / 255ull * 128ull;   // 0x8080..80
  if constexpr (L <= 6) {
    const double t = scaled + (6755399441055744.0 + double(C));
    lo = __double2loint(t);
    hi = __double2hiint(t) - 0x43380000;
  } else {
    const long long u = __double2ll_rn(scaled) + (long long)C;
    lo = int(u);
    hi = int(u >> 32);
  }
}

// v * 2^k rounded into slice_halves; k outside the normal range falls back to scalbn.
template <int L>
__device__ __forceinline__ void scale_halves(double v, int k, int& lo, int& hi) {
  const double scaled = (k >= -1022 && k <= 1023) ? v * __longlong_as_double((long long)(k + 1023) << 52)
                                                  : scalbn(v, k);
  slice_halves<L>(scaled, lo, hi);
}

// Digit planes of 4 consecutive values (a 4 x 4 byte transpose per 32-bit half):
// w[s] byte i = int8 digit d_s of value i.
template <int L>
__device__ __forceinline__ void pack4(const int (&lo)[4], const int (&hi)[4], uint32_t (&w)[L]) {
  const uint32_t a = __byte_perm(lo[0], lo[1], 0x5140), b = __byte_perm(lo[0], lo[1], 0x7362);
  const uint32_t c = __byte_perm(lo[2], lo[3], 0x5140), d = __byte_perm(lo[2], lo[3], 0x7362);
  w[L - 1] = __byte_perm(a, c, 0x5410) ^ 0x80808080u;   // byte 0 of u: the last digit
  w[L - 2] = __byte_perm(a, c, 0x7632) ^ 0x80808080u;
  w[L - 3] = __byte_perm(b, d, 0x5410) ^ 0x80808080u;
  w[L - 4] = __byte_perm(b, d, 0x7632) ^ 0x80808080u;
  const uint32_t e = __byte_perm(hi[0], hi[1], 0x5140), f = __byte_perm(hi[2], hi[3], 0x5140);
  if constexpr (L == 6) {
    w[1] = __byte_perm(e, f, 0x5410) ^ 0x80808080u;
    w[0] = __byte_perm(e, f, 0x7632);                   // byte 1 of hi: d_0 (no bias)
  } else {
    static_assert(L == 7, "6 or 7 digit levels");
    w[2] = __byte_perm(e, f, 0x5410) ^ 0x80808080u;
    w[1] = __byte_perm(e, f, 0x7632) ^ 0x80808080u;
    const uint32_t g = __byte_perm(hi[0], hi[1], 0x0062), h = __byte_perm(hi[2], hi[3], 0x0062);
    w[0] = __byte_perm(g, h, 0x5410);                   // byte 2 of hi: d_0
  }
}

// frexp exponent of a nonnegative double given by its bits (0 for zero)
__device__ __forceinline__ int exp_of_bits(unsigned long long bits) {
  const int field = int((bits >> 52) & 0x7FFu);
  if (field != 0) return field - 1022;
  int e = 0;
  if (bits != 0ull) frexp(__longlong_as_double((long long)bits), &e);
  return e;
}

// v * 2^e, exact (a power-of-two multiply) unless the result leaves the normal range
__device__ __forceinline__ double times_pow2(double v, int e) {
  return (e >= -1022 && e <= 1023) ? v * __longlong_as_double((long long)(e + 1023) << 52) : scalbn(v, e);
}

// ------------------------------------------------------ tensor slicing --
__global__ void slice_rowmax_kernel(const double* __restrict__ x, int64_t M, int64_t J, int64_t jper,
                                    unsigned long long* __restrict__ rmax) {
  const int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int64_t j0 = int64_t(blockIdx.y) * jper;
  const int64_t j1 = min(J, j0 + jper);
  const double* p = x + m;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  int64_t j = j0;
  for (; j + 4 <= j1; j += 4) {
    v0 = fmax(v0, fabs(__ldg(p + (j + 0) * M)));
    v1 = fmax(v1, fabs(__ldg(p + (j + 1) * M)));
    v2 = fmax(v2, fabs(__ldg(p + (j + 2) * M)));
    v3 = fmax(v3, fabs(__ldg(p + (j + 3) * M)));
  }
  for (; j < j1; ++j) v0 = fmax(v0, fabs(__ldg(p + j * M)));
  const double v = fmax(fmax(v0, v1), fmax(v2, v3));
  atomicMax(rmax + m, (unsigned long long)__double_as_longlong(v));
}

// slice_rowmax_kernel plus the engine's init-row facts in the same read of X
// (nncp_norm_squared_min's outputs: sum x^2, min x, max |x|, min nonzero |x|), so a
// run that slices reads the 8-byte tensor once before the planes pass instead of
// twice.  Per-CTA partials [4][ctas], summed / min-maxed in CTA order by the last.
__global__ void __launch_bounds__(256) norm_rowmax_kernel(const double* __restrict__ x, int64_t M, int64_t J,
                                                          int64_t jper, unsigned long long* __restrict__ rmax,
                                                          double* __restrict__ part, double* out, double* out_min,
                                                          unsigned int* ticket) {
  __shared__ double red[8];
  __shared__ double redm[3][8];
  const int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  double s0 = 0.0, s1 = 0.0, mn = INFINITY, a0 = 0.0, a1 = 0.0, anz = INFINITY;
  bool nonfinite = false;
  if (m < M) {
    const int64_t j0 = int64_t(blockIdx.y) * jper;
    const int64_t j1 = min(J, j0 + jper);
    const double* p = x + m;
    int64_t j = j0;
    for (; j + 2 <= j1; j += 2) {
      const double u = __ldcs(p + j * M), v = __ldcs(p + (j + 1) * M);
      s0 = fma(u, u, s0);
      s1 = fma(v, v, s1);
      mn = fmin(mn, fmin(u, v));
      const double au = fabs(u), av = fabs(v);
      a0 = fmax(a0, au);
      a1 = fmax(a1, av);
      anz = fmin(anz, fmin(au > 0.0 ? au : INFINITY, av > 0.0 ? av : INFINITY));
      nonfinite |= !isfinite(u) || !isfinite(v);
    }
    if (j < j1) {
      const double u = __ldcs(p + j * M), au = fabs(u);
      s0 = fma(u, u, s0);
      mn = fmin(mn, u);
      a0 = fmax(a0, au);
      anz = fmin(anz, au > 0.0 ? au : INFINITY);
      nonfinite |= !isfinite(u);
    }
    atomicMax(rmax + m, (unsigned long long)__double_as_longlong(fmax(a0, a1)));   // NaN dropped, as before
  }
  const unsigned nb = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  const double s = block_sum(s0 + s1, red);
  if (threadIdx.x == 0) part[bid] = s;
  double amax = fmax(a0, a1);
  bool bad = nonfinite;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    anz = fmin(anz, __shfl_xor_sync(0xffffffffu, anz, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    redm[0][threadIdx.x >> 5] = mn;
    redm[1][threadIdx.x >> 5] = bad ? NAN : amax;
    redm[2][threadIdx.x >> 5] = anz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = redm[0][0], a = redm[1][0], z = redm[2][0];
    bool nan = isnan(a);
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
      mm = fmin(mm, redm[0][w]);
      nan |= isnan(redm[1][w]);
      a = fmax(a, redm[1][w]);
      z = fmin(z, redm[2][w]);
    }
    part[nb + bid] = mm;
    part[2 * nb + bid] = nan ? NAN : a;
    part[3 * nb + bid] = z;
  }
  if (last_cta_ticket(ticket)) {
    finish_partials(part, int(nb), 1, out);
    if (threadIdx.x == 0) {
      double mm = part[nb], a = part[2 * nb], z = part[3 * nb];
      bool nan = isnan(a);
      for (unsigned b = 1; b < nb; ++b) {
        mm = fmin(mm, part[nb + b]);
        nan |= isnan(part[2 * nb + b]);
        a = fmax(a, part[2 * nb + b]);
        z = fmin(z, part[3 * nb + b]);
      }
      out_min[0] = mm;
      out_min[1] = nan ? NAN : a;
      out_min[2] = z;
    }
  }
}

// Thread: PR = 8 consecutive rows m at every column j of its range (padding rows /
// columns written as zeros); 8 bytes per plane into the blocked layout.  Measured at
// 2048^3 (tools/slice_timing.py): 16 rows per thread held ~200 registers, one CTA per
// SM, 25.8 ms; 8 rows, two CTAs, 21.4 ms; 4 rows, three CTAs, 22.9 ms.
constexpr int PR = 8;
template <int L, bool VEC>
__global__ void __launch_bounds__(256, 2) slice_planes_kernel(const double* __restrict__ x, int64_t M, int64_t J,
                                                              int64_t Mp, int64_t Jp, int64_t njb, int64_t jper,
                                                              const unsigned long long* __restrict__ rmax,
                                                              int* __restrict__ rowexp, int8_t* __restrict__ planes) {
  const int64_t m0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * PR;
  if (m0 >= Mp) return;
  int ex[PR];
#pragma unroll
  for (int i = 0; i < PR; ++i) ex[i] = (m0 + i < M) ? exp_of_bits(rmax[m0 + i]) : 0;
  if (blockIdx.y == 0) {
#pragma unroll
    for (int i = 0; i < PR; ++i) rowexp[m0 + i] = ex[i];
  }
  const int64_t mb = m0 / BM;
  const int64_t j0 = int64_t(blockIdx.y) * jper;
  const int64_t j1 = min(Jp, j0 + jper);
  // column j + 1's values are loaded before column j is sliced
  auto load = [&](int64_t j, double (&v)[PR]) {
    const double* src = x + M * j + m0;
    if (j >= J) {
#pragma unroll
      for (int i = 0; i < PR; ++i) v[i] = 0.0;
    } else if (VEC && m0 + PR <= M) {
#pragma unroll
      for (int i = 0; i < PR / 2; ++i) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(src) + i);
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < PR; ++i) v[i] = (m0 + i < M) ? __ldcs(src + i) : 0.0;
    }
  };
  // the rows' scalings 2^(8L-2-ex) are fixed for the whole column range: test their
  // range once (scale_halves' per-element select kept its scalbn path in the issue
  // stream); both arms compute exactly what scale_halves does
  auto sweep = [&](auto scale) {
    double vn[PR];
    if (j0 < j1) load(j0, vn);
    for (int64_t j = j0; j < j1; ++j) {
      double v[PR];
#pragma unroll
      for (int i = 0; i < PR; ++i) v[i] = vn[i];
      if (j + 1 < j1) load(j + 1, vn);
      uint32_t w[PR / 4][L];
#pragma unroll
      for (int g4 = 0; g4 < PR / 4; ++g4) {
        int lo[4], hi[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) slice_halves<L>(scale(v[4 * g4 + i], 4 * g4 + i), lo[i], hi[i]);
        pack4<L>(lo, hi, w[g4]);
      }
      int8_t* blk = planes + ((mb * njb + j / BK) * L) * int64_t(TILE) + (j % BK) * BM + (m0 % BM);
#pragma unroll
      for (int s = 0; s < L; ++s) {
        if constexpr (PR == 8)
          *reinterpret_cast<uint2*>(blk + int64_t(s) * TILE) = make_uint2(w[0][s], w[1][s]);
        else
          *reinterpret_cast<uint32_t*>(blk + int64_t(s) * TILE) = w[0][s];
      }
    }
  };
  bool fast = true;
#pragma unroll
  for (int i = 0; i < PR; ++i) fast = fast && (8 * L - 2 - ex[i] >= -1022) && (8 * L - 2 - ex[i] <= 1023);
  if (fast) {
    sweep([&ex](double v, int i) { return v * __longlong_as_double((long long)(8 * L - 2 - ex[i] + 1023) << 52); });
  } else {
    sweep([&ex](double v, int i) { return scalbn(v, 8 * L - 2 - ex[i]); });
  }
}

// ------------------------------------------------------ factor slicing --
// B[k, r] = KRP(factors)[k, r] (first factor fastest, tensor_ops.py:121-137),
// times 2^rowexp[k] for the right side.
struct BSpec {
  const double* ptr[kMaxOrder];
  int64_t dim[kMaxOrder];
  int n;
  const int* rowexp;  // nullable
  int64_t K, Kp, Kc;  // Kp: K rounded up to whole 128-deep k blocks
  int R, RP;
  int segg;           // segment-reuse path: outer indices per block (<= SEG_G)
};

constexpr int EXP_NONE = int(0x80808080);   // memset(0x80) sentinel: column chunk has no nonzero

// B preparation works on whole 128-deep k blocks (one GEMM B stage each): block
// = 8 warps x 16 rows, lane = column (coalesced factor-row loads), H = column
// halves (R <= 32: 1, else 2).  NF = number of Khatri-Rao factors when 1..3:
// the warp's first row is decomposed into factor rows once and later rows
// advance per-factor row pointers (first factor fastest; no divisions, all 16
// rows' loads independent); NF = 0: any count, one decomposition per row.
// v[i][h] = KRP[k0 + i, lane + 32 h] (0 outside the tensor / rank);
// sc[i] = 2^rowexp[k0 + i] (1 without row exponents).
template <int NF, int H>
__device__ __forceinline__ void krp_rows16(const BSpec& s, int64_t k0, int lane, double (&v)[16][H],
                                           double (&sc)[16]) {
  const bool full = k0 + 16 <= s.K;
  if constexpr (NF > 0) {
    const double* p[NF];
    uint32_t dig[NF];
    int64_t q = k0 < s.K ? k0 : 0;
#pragma unroll
    for (int f = 0; f < NF - 1; ++f) {
      dig[f] = uint32_t(q % s.dim[f]);
      q /= s.dim[f];
    }
    dig[NF - 1] = uint32_t(q);
#pragma unroll
    for (int f = 0; f < NF; ++f) p[f] = s.ptr[f] + size_t(dig[f]) * s.R + lane;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const bool in = full || k0 + i < s.K;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const bool ok = in && lane + 32 * h < s.R;
        double prod = ok ? __ldg(p[0] + 32 * h) : 0.0;
#pragma unroll
        for (int f = 1; f < NF; ++f) prod *= ok ? __ldg(p[f] + 32 * h) : 0.0;
        v[i][h] = prod;
      }
      // advance the cursor (first factor fastest)
      ++dig[0];
      p[0] += s.R;
#pragma unroll
      for (int f = 0; f < NF - 1; ++f) {
        if (dig[f] == uint32_t(s.dim[f])) {
          dig[f] = 0;
          p[f] -= s.dim[f] * s.R;
          ++dig[f + 1];
          p[f + 1] += s.R;
        }
      }
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < 16; ++i) {
      const int64_t k = k0 + i;
      const bool in = k < s.K;
      int64_t q = in ? k : 0;
      double p[H];
#pragma unroll
      for (int h = 0; h < H; ++h) p[h] = 1.0;
#pragma unroll 1
      for (int f = 0; f < s.n; ++f) {
        int64_t idx = q;
        if (f < s.n - 1) {
          idx = q % s.dim[f];
          q /= s.dim[f];
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int r = lane + 32 * h;
          p[h] *= (in && r < s.R) ? __ldg(s.ptr[f] + idx * s.R + r) : 0.0;
        }
      }
#pragma unroll
      for (int h = 0; h < H; ++h) v[i][h] = p[h];
    }
  }
  // row scales 2^rowexp (right side); the warp's 16 rows start 16-aligned
  if (s.rowexp != nullptr && full) {
    const int4* re = reinterpret_cast<const int4*>(s.rowexp + k0);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const int4 e4 = __ldg(re + q4);
      sc[4 * q4 + 0] = __longlong_as_double((long long)(e4.x + 1023) << 52);
      sc[4 * q4 + 1] = __longlong_as_double((long long)(e4.y + 1023) << 52);
      sc[4 * q4 + 2] = __longlong_as_double((long long)(e4.z + 1023) << 52);
      sc[4 * q4 + 3] = __longlong_as_double((long long)(e4.w + 1023) << 52);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int e = (s.rowexp != nullptr && k0 + i < s.K) ? __ldg(s.rowexp + k0 + i) : 0;
      sc[i] = __longlong_as_double((long long)(e + 1023) << 52);
    }
  }
}

// bexp[chunk][r] = frexp exponent of the chunk's max |B[k, r]| (B = KRP times
// 2^rowexp[k]); one atomic per k block and column.
template <int NF, int H>
__global__ void __launch_bounds__(256) bslice_exp_kernel(BSpec s, int* __restrict__ bexp) {
  __shared__ double red[8][kMaxRank];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t kb0 = int64_t(blockIdx.x) * BK;
  double v[16][H], sc[16];
  krp_rows16<NF, H>(s, kb0 + warp * 16, lane, v, sc);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double mx = 0.0;
    if (h < H) {
#pragma unroll
      for (int i = 0; i < 16; ++i) mx = fmax(mx, fabs(v[i][h < H ? h : 0] * sc[i]));
    }
    red[warp][lane + 32 * h] = mx;
  }
  __syncthreads();
  if (threadIdx.x < s.R) {
    double m = red[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmax(m, red[w][threadIdx.x]);
    if (m > 0.0) atomicMax(bexp + (kb0 / s.Kc) * s.RP + threadIdx.x, exp_of_bits(__double_as_longlong(m)));
  }
}

// Digits of one k block into shared memory (rows (t, r) of 128 digits, word
// pitch 33 so the 32 lanes' stores hit distinct banks), then one contiguous
// coalesced store of the block in the stage layout [t][r][k % 128].
template <int L, int NF, int H>
__global__ void __launch_bounds__(256) bslice_digits_kernel(BSpec s, const int* __restrict__ bexp,
                                                            int8_t* __restrict__ bs) {
  extern __shared__ __align__(16) uint32_t tile[];   // L * RP rows x 33 words
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t kb0 = int64_t(blockIdx.x) * BK;
  const int64_t chunk = kb0 / s.Kc;
  double v[16][H], sc[16];
  krp_rows16<NF, H>(s, kb0 + warp * 16, lane, v, sc);
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const int r = lane + 32 * h;
    if (r >= s.RP) continue;
    const int e = r < s.R ? bexp[chunk * s.RP + r] : EXP_NONE;
    const int k = 8 * L - 2 - (e == EXP_NONE ? 0 : e);   // digits of (v 2^rowexp) / 2^e
    auto digits = [&](auto scale) {   // range of 2^k tested once per column (see bseg_digits_kernel)
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        int lo[4], hi[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) slice_halves<L>(scale(v[4 * g + i][h] * sc[4 * g + i]), lo[i], hi[i]);
        uint32_t w[L];
        pack4<L>(lo, hi, w);
#pragma unroll
        for (int t = 0; t < L; ++t) tile[(t * s.RP + r) * 33 + warp * 4 + g] = w[t];
      }
    };
    if (k >= -1022 && k <= 1023) {
      const double p2 = __longlong_as_double((long long)(k + 1023) << 52);
      digits([p2](double x) { return x * p2; });
    } else {
      digits([k](double x) { return scalbn(x, k); });
    }
  }
  __syncthreads();
  const int nwords = L * s.RP * (BK / 4);
  uint32_t* dst = reinterpret_cast<uint32_t*>(bs + (kb0 / BK) * int64_t(L) * s.RP * BK);
  for (int q = threadIdx.x; q < nwords; q += blockDim.x) dst[q] = tile[(q >> 5) * 33 + (q & 31)];
}

// Segment-reuse B preparation for NF >= 2 Khatri-Rao factors whose first
// (fastest) factor has a multiple of 128 rows: k block kb = seg + nseg * o covers
// rows 128 seg .. 128 seg + 127 of factor 0 at the o-th combination of the other
// factors, so a block keeps its 128 factor-0 rows in registers (warp = 16 rows,
// lane = column) and sweeps G outer indices o, multiplying by one row of the
// other factors each: every factor row is read once per block instead of once
// per KRP row.  Each lane's 16 consecutive rows give 16 consecutive bytes of
// each digit plane (one 16-byte store per plane, no transpose).
constexpr int SEG_G = 16;   // outer indices per block (at most; fewer when that leaves SMs idle)

template <int NF, int H>
struct SegCursor {
  const double* p[NF];      // p[0] fixed: factor-0 rows of the segment; p[1..] advance with o
  uint32_t dig[NF];
  __device__ __forceinline__ void init(const BSpec& s, int64_t o0, int lane) {
    int64_t q = o0;
#pragma unroll
    for (int f = 1; f < NF - 1; ++f) {
      dig[f] = uint32_t(q % s.dim[f]);
      q /= s.dim[f];
    }
    dig[NF - 1] = uint32_t(q);
#pragma unroll
    for (int f = 1; f < NF; ++f) p[f] = s.ptr[f] + size_t(dig[f]) * s.R + lane;
  }
  __device__ __forceinline__ void advance(const BSpec& s) {
    ++dig[1];
    p[1] += s.R;
#pragma unroll
    for (int f = 1; f < NF - 1; ++f) {
      if (dig[f] == uint32_t(s.dim[f])) {
        dig[f] = 0;
        p[f] -= s.dim[f] * s.R;
        ++dig[f + 1];
        p[f + 1] += s.R;
      }
    }
  }
};

// Per outer index o: the 16 row exponents of the warp's rows (4 x int4) and the
// product g of the other factors' entries, loaded one o ahead (prefetch).
template <int NF, int H>
struct SegLoads {
  int4 re[4];
  double g[H];
  __device__ __forceinline__ void load(const BSpec& s, const SegCursor<NF, H>& cur, int64_t k0, int lane,
                                       bool valid) {
    if (s.rowexp != nullptr && valid) {
      const int4* p = reinterpret_cast<const int4*>(s.rowexp + k0);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) re[q4] = __ldg(p + q4);
    } else {
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) re[q4] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
      double gg = 1.0;
#pragma unroll
      for (int f = 1; f < NF; ++f) gg *= (valid && lane + 32 * h < s.R) ? __ldg(cur.p[f] + 32 * h) : 0.0;
      g[h] = gg;
    }
  }
  __device__ __forceinline__ int rexp(int i) const {
    const int4 v = re[i >> 2];
    return (i & 3) == 0 ? v.x : (i & 3) == 1 ? v.y : (i & 3) == 2 ? v.z : v.w;
  }
};

template <int NF, int H>
__global__ void __launch_bounds__(256) bseg_exp_kernel(BSpec s, int* __restrict__ bexp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nseg = s.dim[0] / BK, outer = s.K / s.dim[0];
  const int64_t seg = blockIdx.x, o0 = int64_t(blockIdx.y) * s.segg;
  const int64_t i0 = seg * BK + warp * 16;        // first factor-0 row of the warp
  double h0[16][H];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int h = 0; h < H; ++h)
      h0[i][h] = lane + 32 * h < s.R ? __ldg(s.ptr[0] + (i0 + i) * s.R + lane + 32 * h) : 0.0;
  SegCursor<NF, H> cur;
  cur.init(s, o0, lane);
  double mx[H];
#pragma unroll
  for (int h = 0; h < H; ++h) mx[h] = 0.0;
  int64_t chunk = -1;
  const int64_t oend = min(outer, o0 + s.segg);
  SegLoads<NF, H> nxt;
  nxt.load(s, cur, i0 + s.dim[0] * o0, lane, o0 < oend);
  for (int64_t o = o0; o < oend; ++o) {
    const SegLoads<NF, H> now = nxt;
    cur.advance(s);
    nxt.load(s, cur, i0 + s.dim[0] * (o + 1), lane, o + 1 < oend);
    const int64_t c = (seg + nseg * o) * BK / s.Kc;
    if (c != chunk) {
      if (chunk >= 0) {
#pragma unroll
        for (int h = 0; h < H; ++h)
          if (lane + 32 * h < s.R && mx[h] > 0.0)
            atomicMax(bexp + chunk * s.RP + lane + 32 * h, exp_of_bits(__double_as_longlong(mx[h])));
      }
#pragma unroll
      for (int h = 0; h < H; ++h) mx[h] = 0.0;
      chunk = c;
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double sc = __longlong_as_double((long long)(now.rexp(i) + 1023) << 52);
        mx[h] = fmax(mx[h], fabs(h0[i][h] * now.g[h] * sc));
      }
    }
  }
  if (chunk >= 0) {
#pragma unroll
    for (int h = 0; h < H; ++h)
      if (lane + 32 * h < s.R && mx[h] > 0.0)
        atomicMax(bexp + chunk * s.RP + lane + 32 * h, exp_of_bits(__double_as_longlong(mx[h])));
  }
}

// Digits: each warp packs its 16 rows of every (digit, column) row into 16 bytes,
// staged in shared memory (row pitch 144 B: the 8 lanes of a 16-byte store phase
// hit distinct banks) so the k block leaves as one contiguous run of full lines.
constexpr int SEG_PITCH = 144;

template <int L, int NF, int H>
__global__ void __launch_bounds__(256) bseg_digits_kernel(BSpec s, const int* __restrict__ bexp,
                                                          int8_t* __restrict__ bs) {
  extern __shared__ __align__(16) uint8_t stage[];   // L * RP rows x SEG_PITCH bytes
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nseg = s.dim[0] / BK, outer = s.K / s.dim[0];
  const int64_t seg = blockIdx.x, o0 = int64_t(blockIdx.y) * s.segg;
  const int64_t i0 = seg * BK + warp * 16;
  const int nrow = L * s.RP;
  double h0[16][H];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int h = 0; h < H; ++h)
      h0[i][h] = lane + 32 * h < s.R ? __ldg(s.ptr[0] + (i0 + i) * s.R + lane + 32 * h) : 0.0;
  SegCursor<NF, H> cur;
  cur.init(s, o0, lane);
  const int64_t oend = min(outer, o0 + s.segg);
  SegLoads<NF, H> nxt;
  nxt.load(s, cur, i0 + s.dim[0] * o0, lane, o0 < oend);
  for (int64_t o = o0; o < oend; ++o) {
    const SegLoads<NF, H> now = nxt;
    cur.advance(s);
    nxt.load(s, cur, i0 + s.dim[0] * (o + 1), lane, o + 1 < oend);
    const int64_t kb = seg + nseg * o;
    const int64_t c = kb * BK / s.Kc;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int r = lane + 32 * h;
      if (r >= s.RP) continue;
      const int e = r < s.R ? __ldg(bexp + c * s.RP + r) : EXP_NONE;
      const int kx = 8 * L - 2 - (e == EXP_NONE ? 0 : e);
      uint32_t w[4][L];
      // the column's scaling 2^kx is uniform over the 16 rows: test its range once
      // and branch (scale_halves' per-element select kept the scalbn path in the
      // issue stream, predicated off); the arithmetic is scale_halves' in both arms
      auto digits = [&](auto scale) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          int lo[4], hi[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const double sc = __longlong_as_double((long long)(now.rexp(4 * q4 + i) + 1023) << 52);
            slice_halves<L>(scale(h0[4 * q4 + i][h] * now.g[h] * sc), lo[i], hi[i]);
          }
          pack4<L>(lo, hi, w[q4]);
        }
      };
      if (kx >= -1022 && kx <= 1023) {
        const double p2 = __longlong_as_double((long long)(kx + 1023) << 52);
        digits([p2](double v) { return v * p2; });
      } else {
        digits([kx](double v) { return scalbn(v, kx); });
      }
#pragma unroll
      for (int t = 0; t < L; ++t)
        *reinterpret_cast<uint4*>(stage + (t * s.RP + r) * SEG_PITCH + warp * 16) =
            make_uint4(w[0][t], w[1][t], w[2][t], w[3][t]);
    }
    __syncthreads();
    uint4* dst = reinterpret_cast<uint4*>(bs + kb * int64_t(L) * s.RP * BK);
    for (int q = threadIdx.x; q < nrow * 8; q += blockDim.x)
      dst[q] = *reinterpret_cast<const uint4*>(stage + (q >> 3) * SEG_PITCH + (q & 7) * 16);
    __syncthreads();
  }
}

template <int L, int NF, int H>
int launch_bslice(const BSpec& b, int* bexp, int8_t* bs, unsigned kblocks, cudaStream_t st) {
  if (int rc = set_max_smem_once<bslice_digits_kernel<L, NF, H>>(int(L * kMaxRank * 33 * 4))) return rc;
  bslice_exp_kernel<NF, H><<<kblocks, 256, 0, st>>>(b, bexp);
  NNCP_LAUNCH_CHECK();
  bslice_digits_kernel<L, NF, H><<<kblocks, 256, size_t(L) * b.RP * 33 * 4, st>>>(b, bexp, bs);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

template <int L, int NF, int H>
int launch_bseg(const BSpec& b0, int* bexp, int8_t* bs, cudaStream_t st) {
  BSpec b = b0;
  const int64_t outer = b.K / b.dim[0], nseg = b.dim[0] / BK;
  // exponent pass: >= ~4 blocks per SM (512^3: 4 segments x 512 outer indices -> 3 per
  // block, 684 blocks); digit pass: ~8 blocks per SM but at least 3 outer indices per
  // block (measured, tools/ncu launch lists: 1024^3 66 -> 60 us, 512^3 unchanged)
  const int64_t work = nseg * outer, sms = num_sms();
  b.segg = int(std::max<int64_t>(1, std::min<int64_t>(SEG_G, work / (4 * sms))));
  const dim3 grid{unsigned(nseg), unsigned((outer + b.segg - 1) / b.segg), 1u};
  bseg_exp_kernel<NF, H><<<grid, 256, 0, st>>>(b, bexp);
  NNCP_LAUNCH_CHECK();
  b.segg = int(std::max<int64_t>(std::min<int64_t>(3, outer), std::min<int64_t>(SEG_G, work / (8 * sms))));
  const dim3 grid_d{unsigned(nseg), unsigned((outer + b.segg - 1) / b.segg), 1u};
  if (int rc = set_max_smem_once<bseg_digits_kernel<L, NF, H>>(int(L * kMaxRank * SEG_PITCH))) return rc;
  bseg_digits_kernel<L, NF, H><<<grid_d, 256, size_t(L) * b.RP * SEG_PITCH, st>>>(b, bexp, bs);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

template <int L, int NF>
int launch_bslice_h(const BSpec& b, int* bexp, int8_t* bs, unsigned kblocks, cudaStream_t st) {
  // segment reuse when factor 0 tiles into whole k blocks (then K = dim[0] * outer is too)
  if (NF >= 2 && b.dim[0] % BK == 0 && b.K / b.dim[0] < 65535 * SEG_G) {
    constexpr int NS = NF >= 2 ? NF : 2;
    return b.RP <= 32 ? launch_bseg<L, NS, 1>(b, bexp, bs, st) : launch_bseg<L, NS, 2>(b, bexp, bs, st);
  }
  return b.RP <= 32 ? launch_bslice<L, NF, 1>(b, bexp, bs, kblocks, st)
                    : launch_bslice<L, NF, 2>(b, bexp, bs, kblocks, st);
}

template <int L>
int dispatch_bslice(const BSpec& b, int* bexp, int8_t* bs, unsigned kblocks, cudaStream_t st) {
  switch (b.n) {
    case 1: return launch_bslice_h<L, 1>(b, bexp, bs, kblocks, st);
    case 2: return launch_bslice_h<L, 2>(b, bexp, bs, kblocks, st);
    case 3: return launch_bslice_h<L, 3>(b, bexp, bs, kblocks, st);
    default: return launch_bslice_h<L, 0>(b, bexp, bs, kblocks, st);
  }
}

// out1[i1 + I1 r] = sum over the CTAs whose contiguous item range touched i1's block
// of their partials, in CTA order (deterministic).  Items are ib * O + o.
__global__ void ttv_partials_reduce_kernel(const double* __restrict__ tpart, int64_t items, int ctas, int64_t nout,
                                           int64_t slots, int64_t I1, int R, int RP, double* __restrict__ out1) {
  const int64_t n = I1 * R;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i1 = e % I1, r = e / I1;
    const int64_t ib = i1 / 128, row = i1 % 128;
    // CTAs c with [c items / ctas, (c+1) items / ctas) overlapping [ib O, (ib+1) O)
    int64_t c_lo = (ib * nout * ctas) / items;
    while (c_lo > 0 && (c_lo * items) / ctas > ib * nout) --c_lo;
    while (c_lo < ctas - 1 && ((c_lo + 1) * items) / ctas <= ib * nout) ++c_lo;
    // contributing CTAs: c_lo .. while the CTA's first item is inside block ib (monotone
    // in c); four partials loaded ahead of the in-order additions (same sum order)
    const int64_t end_item = (ib + 1) * nout;
    double s = 0.0;
    for (int64_t c = c_lo; c < ctas; c += 4) {
      double v[4];
      bool ok[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t cc = c + q;
        const int64_t b = cc * items / ctas, en = (cc + 1) * items / ctas;
        ok[q] = cc < ctas && b < end_item && en > b;
        v[q] = ok[q] ? tpart[((cc * slots + (ib - b / nout)) * 128 + row) * RP + r] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (ok[q]) s += v[q];
      if (c + 4 >= ctas || (c + 4) * items / ctas >= end_item) break;
    }
    out1[e] = s;
  }
}

__global__ void group_reduce_kernel(const double* __restrict__ part, int groups, int64_t stride, int64_t n,
                                    double* __restrict__ out) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    double s = part[e];
    for (int g = 1; g < groups; ++g) s += part[int64_t(g) * stride + e];
    out[e] = s;
  }
}

// ------------------------------------------------------------- UMMA PTX --
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFFu);
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;                 // descriptor version (sm_100)
  d |= uint64_t(layout) << 61;            // 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
  return d;
}

__device__ __forceinline__ uint32_t idesc_s8(int N, bool a_mn_major) {
  return (2u << 4)                          // D: s32
         | (1u << 7) | (1u << 10)           // A, B: signed 8-bit
         | (uint32_t(a_mn_major) << 15)     // A major (B is K-major)
         | (uint32_t(N >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_s8(uint32_t dtmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// L2 cache policies for the TMA streams: the right side's digit planes are read
// once per partial (evict first), the factor digits are shared by the row tiles
// (evict last); measured on the B200 (the right side's DRAM reads drop to the
// algorithmic bytes, 7.8 -> 7.5 ms at 2048^3 R = 32).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// --------------------------------------------------------------- GEMM ---
// Build with -DNNCP_SLICED_STATS for per-CTA barrier wait cycles (tools only):
// [0] producer on B empty, [1] producer on A empty, [2] MMA on TMEM empty,
// [3] MMA on B full, [4] MMA on A full, [5] epilogue on TMEM full, [6] kernel cycles.
#ifdef NNCP_SLICED_STATS
__device__ unsigned long long g_sliced_stats[1024 * 8];
#define SLICED_WAIT(slot, bar, par)                                              \
  do {                                                                           \
    const long long _t0 = clock64();                                             \
    mbar_wait(bar, par);                                                         \
    atomicAdd(&g_sliced_stats[blockIdx.x * 8 + (slot)], (unsigned long long)(clock64() - _t0)); \
  } while (0)
#else
#define SLICED_WAIT(slot, bar, par) mbar_wait(bar, par)
#endif
template <int RP, int L, int SIDE>
struct GemmCfg {
  static constexpr int A_STAGE = TILE;                  // one digit-plane tile
  static constexpr int B_STAGE = L * RP * BK;           // all B digit rows of one k block
  static constexpr int NB = 2;
  // left side: the 128 x R fp64 output tile leaves through shared memory by a TMA
  // bulk store (generic-proxy global stores of the 1 GB T_L slowed the TMA read
  // stream by ~10%, measured)
  static constexpr bool TMA_OUT = SIDE == NNCP_SIDE_LEFT && RP <= 32;   // fits beside >= 9 A stages
  static constexpr int OUT_STAGE = TMA_OUT ? BM * RP * 8 : 0;
  static constexpr int NA_FIT = (MAX_SMEM - 1024 - NB * B_STAGE - OUT_STAGE) / A_STAGE;
  static constexpr int NA = NA_FIT > 12 ? 12 : NA_FIT;
  static constexpr int ACC = L * RP;                    // TMEM columns of one accumulator set
  static constexpr int NBUF = (2 * ACC <= 512) ? 2 : 1;
  static constexpr int NEED = NBUF * ACC;
  static constexpr int TCOLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static constexpr size_t SMEM = size_t(NB) * B_STAGE + size_t(NA) * A_STAGE + OUT_STAGE + 1024;
  static_assert(NA >= L, "one k block of digit tiles must fit in shared memory");
  static_assert(ACC <= 512, "accumulator does not fit in TMEM");
  static_assert(B_STAGE % 1024 == 0, "stages must keep 1 KB alignment");
};

struct GemmArgs {
  int64_t rows;        // output rows: M (left) or J (right)
  int64_t nkb;         // 128-deep k blocks of the (padded) contraction
  int64_t kbc;         // k blocks per chunk
  int64_t nchunks;
  int64_t row_tiles;
  int64_t items;       // row_tiles * groups
  int groups;
  const int* rowexp;   // left: per output row exponent; right: nullptr (folded into B)
  const int* bexp;     // [nchunks][RP] frexp exponents of the column-chunk maxima of |B|
  double* out;         // [group][r][row]
  int tma_out;         // left side: the output tensor map is valid (else direct stores)
  int64_t group_stride;
  int R;
  // fused trailing multi-TTV (left side, split S = 2, dims[0] % 128 == 0, RP <= 32):
  // the epilogue also accumulates out1[i1, r] = sum_o T_L[i1 + I1 o, r] H_1[o, r]
  // (dimtree.py:159-165); tiles visited i1-block-major in contiguous per-CTA ranges,
  // per-CTA partials [cta][slot][128][RP] reduced in CTA order afterwards
  int fuse;
  int64_t nib, nout;   // i1 blocks (I1 / 128) and outer indices (M / I1)
  const double* cf[1];  // the trailing factor H_1 (split S = 2)
  double* tpart;
  int64_t slots;       // partial slots per CTA
};

// Items of one CTA: round-robin over CTAs, or (fused TTV) one contiguous range.
__device__ __forceinline__ void item_range(const GemmArgs& a, int64_t& b, int64_t& e, int64_t& step) {
  if (a.fuse) {
    b = int64_t(blockIdx.x) * a.items / gridDim.x;
    e = int64_t(blockIdx.x + 1) * a.items / gridDim.x;
    step = 1;
  } else {
    b = blockIdx.x;
    e = a.items;
    step = gridDim.x;
  }
}

// item -> (row tile, split-K group)
__device__ __forceinline__ void item_tile(const GemmArgs& a, int64_t it, int64_t& tile, int64_t& g) {
  if (a.fuse) {
    tile = it / a.nout + a.nib * (it % a.nout);   // item = ib * O + o  ->  m block = ib + nib * o
    g = 0;
  } else {
    tile = it % a.row_tiles;
    g = it / a.row_tiles;
  }
}

template <int SIDE, int RP, int L>
__global__ void __launch_bounds__(THREADS, 1) sliced_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                const __grid_constant__ CUtensorMap mapB,
                                                                const __grid_constant__ CUtensorMap mapO,
                                                                GemmArgs a) {
  using C = GemmCfg<RP, L, SIDE>;
  constexpr bool LEFT = SIDE == NNCP_SIDE_LEFT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_b = smem;
  uint8_t* smem_a = smem + C::NB * C::B_STAGE;
  double* smem_o = reinterpret_cast<double*>(smem_a + size_t(C::NA) * C::A_STAGE);   // [R][128] (left only)
  __shared__ __align__(8) uint64_t afull[C::NA], aempty[C::NA], bfull[C::NB], bempty[C::NB];
  __shared__ __align__(8) uint64_t tfull[C::NBUF], tempty[C::NBUF];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NA; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < C::NBUF; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tma_desc(&mapA);
    prefetch_tma_desc(&mapB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "n"(C::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;
#ifdef NNCP_SLICED_STATS
  const long long t_start = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ TMA producer ----
      const uint64_t pol_a = l2_policy_evict_first(), pol_b = l2_policy_evict_last();
      int as = 0, bsx = 0;
      uint32_t aph = 0, bph = 0;
      int64_t it_b, it_e, it_s;
      item_range(a, it_b, it_e, it_s);
      for (int64_t it = it_b; it < it_e; it += it_s) {
        int64_t tile, g;
        item_tile(a, it, tile, g);
        const int64_t c0 = g * a.nchunks / a.groups, c1 = (g + 1) * a.nchunks / a.groups;
        for (int64_t kb = c0 * a.kbc, kend = min(a.nkb, c1 * a.kbc); kb < kend; ++kb) {
          SLICED_WAIT(0, &bempty[bsx], bph ^ 1u);
          mbar_arrive_expect_tx(&bfull[bsx], C::B_STAGE);
          tma_load_4d(smem_b + size_t(bsx) * C::B_STAGE, &mapB, &bfull[bsx], 0, 0, 0, int(kb), pol_b);
          if (++bsx == C::NB) {
            bsx = 0;
            bph ^= 1u;
          }
          const int mb = int(LEFT ? tile : kb), jb = int(LEFT ? kb : tile);
#pragma unroll 1
          for (int s = 0; s < L; ++s) {
            SLICED_WAIT(1, &aempty[as], aph ^ 1u);
            mbar_arrive_expect_tx(&afull[as], C::A_STAGE);
            if (LEFT)   // (measured: an evict-first hint slows the left side's stream)
              tma_load_5d(smem_a + size_t(as) * C::A_STAGE, &mapA, &afull[as], 0, 0, s, jb, mb);
            else
              tma_load_5d(smem_a + size_t(as) * C::A_STAGE, &mapA, &afull[as], 0, 0, s, jb, mb, pol_a);
            if (++as == C::NA) {
              as = 0;
              aph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer ------
      int as = 0, bsx = 0, abuf = 0;
      uint32_t aph = 0, bph = 0, tph = 0;
      int64_t it_b, it_e, it_s;
      item_range(a, it_b, it_e, it_s);
      for (int64_t it = it_b; it < it_e; it += it_s) {
        int64_t tile, g;
        item_tile(a, it, tile, g);
        const int64_t c0 = g * a.nchunks / a.groups, c1 = (g + 1) * a.nchunks / a.groups;
        for (int64_t c = c0; c < c1; ++c) {
          SLICED_WAIT(2, &tempty[abuf], tph ^ 1u);
          tc_fence_after();
          const uint32_t dcol = tbase + uint32_t(abuf * C::ACC);
          bool first = true;
          for (int64_t kb = c * a.kbc, kend = min(a.nkb, (c + 1) * a.kbc); kb < kend; ++kb) {
            SLICED_WAIT(3, &bfull[bsx], bph);
            tc_fence_after();
            // descriptors of this k block's B stage; every MMA below adds compile-time offsets
            const uint64_t db0 = smem_desc(smem_u32(smem_b + size_t(bsx) * C::B_STAGE), 1024, 2);
#pragma unroll
            for (int s = 0; s < L; ++s) {
              SLICED_WAIT(4, &afull[as], aph);
              tc_fence_after();
              const uint64_t da0 = smem_desc(smem_u32(smem_a + size_t(as) * C::A_STAGE), 1024, 2);
#pragma unroll
              for (int kk = 0; kk < BK / 32; ++kk) {
                // left: MN-major SW128 (32 k rows of 128 B per MMA); right: K-major SW128 (32 B per MMA)
                const uint64_t da = da0 + uint64_t(LEFT ? (kk * 32 * 128) >> 4 : (kk * 32) >> 4);
#pragma unroll
                for (int n0 = 0; n0 < (L - s) * RP; n0 += 256) {
                  const int nn = (L - s) * RP - n0 < 256 ? (L - s) * RP - n0 : 256;
                  const uint64_t db = db0 + uint64_t((kk * 32 + (n0 / 8) * 1024) >> 4);
                  umma_s8(dcol + uint32_t(s * RP + n0), da, db, idesc_s8(nn, LEFT),
                          (first && s == 0 && kk == 0) ? 0u : 1u);
                }
              }
              umma_commit(&aempty[as]);
              if (++as == C::NA) {
                as = 0;
                aph ^= 1u;
              }
            }
            first = false;
            umma_commit(&bempty[bsx]);
            if (++bsx == C::NB) {
              bsx = 0;
              bph ^= 1u;
            }
          }
          umma_commit(&tfull[abuf]);
          if (++abuf == C::NBUF) {
            abuf = 0;
            tph ^= 1u;
          }
        }
      }
    }
  } else {
    // -------------------------------------------------- epilogue --------
    // warp w: TMEM lane quadrant w % 4 (rows), column half (w - 2) / 4
    constexpr int RH = RP / 2;
    const int quad = warp & 3, half = (warp - 2) >> 2;
    int abuf = 0;
    uint32_t tph = 0;
    int64_t it_b, it_e, it_s;
    item_range(a, it_b, it_e, it_s);
    // fused trailing TTV state: partial sums of this CTA's current i1 block (RP <= 32:
    // the extra RH registers would spill the RP = 64 epilogue)
    constexpr bool FUSE_OK = LEFT && RP <= 32;
    double fz[RH];
#pragma unroll
    for (int r = 0; r < RH; ++r) fz[r] = 0.0;
    int64_t cur_ib = -1;
    const int64_t ib0 = a.fuse ? it_b / a.nout : 0;
    auto flush_ttv = [&](int64_t ib) {
      double* dst = a.tpart + ((int64_t(blockIdx.x) * a.slots + (ib - ib0)) * BM + quad * 32 + lane) * RP + half * RH;
#pragma unroll
      for (int r = 0; r < RH; ++r) dst[r] = fz[r];
    };
    for (int64_t it = it_b; it < it_e; it += it_s) {
      int64_t tile, g;
      item_tile(a, it, tile, g);
      const int64_t c0 = g * a.nchunks / a.groups, c1 = (g + 1) * a.nchunks / a.groups;
      const int64_t row = tile * BM + quad * 32 + lane;
      const bool valid = row < a.rows;
      const int ex = (a.rowexp != nullptr && valid) ? a.rowexp[row] : 0;
      double acc[RH];
#pragma unroll
      for (int r = 0; r < RH; ++r) acc[r] = 0.0;
      for (int64_t c = c0; c < c1; ++c) {
        SLICED_WAIT(5, &tfull[abuf], tph);
        tc_fence_after();
        const uint32_t taddr = tbase + uint32_t(abuf * C::ACC + half * RH) + (uint32_t(quad * 32) << 16);
        int eb[RH];   // column-chunk exponents, with the 2^-12 of the two digit scales and the row scale
#pragma unroll
        for (int r = 0; r < RH; ++r) {
          const int e = __ldg(a.bexp + c * RP + half * RH + r);
          eb[r] = (e == EXP_NONE ? 0 : e) - 12 + ex;   // an all-zero column chunk accumulated zeros
        }
#pragma unroll
        for (int rg = 0; rg < RH / 8; ++rg) {
          uint32_t v[L][8];
#pragma unroll
          for (int l = 0; l < L; ++l) tmem_ld8(taddr + uint32_t(l * RP + rg * 8), v[l]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            // sum_l acc_l 2^(-8l): levels combined three at a time in exact int64
            // (|acc_l| < 2^31, so each group < 2^48 converts exactly), then one fp64
            // rounding per pair of groups -- two conversions instead of six
            const long long g1 = (long long)int(v[0][i]) * 65536ll + (long long)int(v[1][i]) * 256ll +
                                 (long long)int(v[2][i]);
            const long long g2 = (long long)int(v[3][i]) * 65536ll + (long long)int(v[4][i]) * 256ll +
                                 (long long)int(v[5][i]);
            double lowp = double(g2);
            if constexpr (L == 7) lowp = lowp + double(int(v[6][i])) * 0x1p-8;   // level 6: 2^-8 below level 5
            const double s = double(g1) + lowp * 0x1p-24;   // = 2^16 sum_l acc_l 2^(-8l)
            acc[rg * 8 + i] += times_pow2(s, eb[rg * 8 + i] - 16);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[abuf]);
        if (++abuf == C::NBUF) {
          abuf = 0;
          tph ^= 1u;
        }
      }
      if (FUSE_OK && a.fuse) {
        const int64_t ib = it / a.nout, o = it % a.nout;
        if (ib != cur_ib) {
          if (cur_ib >= 0) flush_ttv(cur_ib);
#pragma unroll
          for (int r = 0; r < RH; ++r) fz[r] = 0.0;
          cur_ib = ib;
        }
        // C[o, r] = H_1[o, r] (split S = 2: one trailing factor)
        const double* crow = a.cf[0] + o * a.R;
#pragma unroll
        for (int r = 0; r < RH; ++r) {
          const int col = half * RH + r;
          fz[r] = fma(acc[r], col < a.R ? __ldg(crow + col) : 0.0, fz[r]);
        }
      }
      if (C::TMA_OUT && a.tma_out) {
        // stage [r][row] in shared memory; one thread issues the TMA bulk store
        const bool leader = threadIdx.x == 64;   // warp 2, lane 0
        if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // previous tile read out
        named_bar_sync(1, 256);
        const int rl = quad * 32 + lane;
#pragma unroll
        for (int r = 0; r < RH; ++r)
          if (half * RH + r < a.R) smem_o[(half * RH + r) * BM + rl] = acc[r];
        fence_proxy_async();
        named_bar_sync(1, 256);
        if (leader) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&mapO)),
              "r"(int(tile * BM)), "r"(0), "r"(smem_u32(smem_o))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else if (valid) {
        double* o = a.out + g * a.group_stride + row;
#pragma unroll
        for (int r = 0; r < RH; ++r)
          if (half * RH + r < a.R) __stcs(o + int64_t(half * RH + r) * a.rows, acc[r]);   // streaming store
      }
    }
    if (FUSE_OK && a.fuse && cur_ib >= 0) flush_ttv(cur_ib);
  }
  if (C::TMA_OUT && a.tma_out && threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
#ifdef NNCP_SLICED_STATS
  if (threadIdx.x == 0) g_sliced_stats[blockIdx.x * 8 + 6] += (unsigned long long)(clock64() - t_start);
#endif
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS));
  }
}

// ------------------------------------------------------------- host side --
int encode_u8(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
              const cuuint32_t* box) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, cuuint32_t(rank), const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled (u8) failed: " + std::to_string(int(r)));
  return NNCP_OK;
}

struct CallPlan {
  TensorLayout t;
  int RP;
  int64_t K, Kp, Kc, nchunks, rows, row_tiles;
  int groups;
  size_t bexp_off, bs_off, part_off, ws_bytes;
  // fused trailing TTV (left side): eligible, CTAs, partial slots per CTA, I1, outer count
  bool fuse;
  int64_t fctas, fslots, I1, nout;
};

CallPlan plan_call(int order, const int64_t* dims, int split, int side, int rank, int L) {
  CallPlan p{};
  p.t = tensor_layout(order, dims, split, L);
  p.RP = int(align_up(rank, 16));
  const bool left = side == NNCP_SIDE_LEFT;
  p.K = left ? p.t.J : p.t.M;
  p.Kp = left ? p.t.Jp : p.t.Mp;
  p.rows = left ? p.t.M : p.t.J;
  p.row_tiles = left ? p.t.nmb : p.t.njb;
  const int64_t sms = num_sms();
  if (left && p.row_tiles >= sms) {
    p.groups = 1;
    p.Kc = std::min<int64_t>(KC_MAX, align_up(p.Kp, 256));
  } else {
    // split the contraction into groups so row_tiles x groups fills the SMs; the
    // row tiles of a group stream the same B chunks at the same time (L2 reuse)
    // Chunk length chosen so every group gets the same number of chunks (q).
    // (Either side: the left one has few row tiles under a balanced split, e.g.
    // 4096 x (2048 * 256).)
    const int64_t want = std::max<int64_t>(1, sms / p.row_tiles);
    const int64_t per_group = (p.Kp + want - 1) / want;
    const int64_t q = std::max<int64_t>(1, (per_group + KC_MAX - 1) / KC_MAX);
    p.Kc = std::min<int64_t>(KC_MAX, std::max<int64_t>(256, align_up((p.Kp + want * q - 1) / (want * q), 256)));
    const int64_t nch = (p.Kp + p.Kc - 1) / p.Kc;
    p.groups = int(std::min<int64_t>(want, nch));
  }
  p.nchunks = (p.Kp + p.Kc - 1) / p.Kc;
  p.bexp_off = 0;
  p.bs_off = size_t(align_up(p.nchunks * p.RP * 4, 1024));
  p.part_off = p.bs_off + size_t(align_up(int64_t(L) * p.RP * p.Kp, 1024));
  p.ws_bytes = p.part_off + (p.groups > 1 ? size_t(p.groups) * p.rows * rank * sizeof(double) : 0);
  // fused trailing TTV: split 2, whole 128-row blocks of the first mode, RP <= 32, and
  // long row tiles in long per-CTA ranges (measured: with 2-block tiles (c4) the extra
  // epilogue work and the scattered i1-block-major order cost what the TTV saves;
  // with ~3 tiles per CTA (c3) the temporary is too small to matter)
  p.I1 = dims[0];
  p.fuse = left && split == 2 && order >= 3 && dims[0] % BM == 0 && p.RP <= 32 && p.Kp / BK >= 8 &&
           p.row_tiles >= 16 * sms;
  if (p.fuse) {
    p.nout = p.t.M / p.I1;
    p.fctas = std::min<int64_t>(p.row_tiles, sms);
    const int64_t per = (p.row_tiles + p.fctas - 1) / p.fctas;
    p.fslots = (per + p.nout - 1) / p.nout + 1;
    p.ws_bytes = std::max(p.ws_bytes, p.part_off + size_t(p.fctas) * p.fslots * BM * p.RP * sizeof(double));
  }
  return p;
}

template <int SIDE, int RP, int L>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, const GemmArgs& ga,
                cudaStream_t st) {
  using C = GemmCfg<RP, L, SIDE>;
  if (int rc = set_max_smem_once<sliced_gemm_kernel<SIDE, RP, L>>(int(C::SMEM))) return rc;
  const unsigned ctas = unsigned(std::min<int64_t>(ga.items, num_sms()));
  sliced_gemm_kernel<SIDE, RP, L><<<ctas, THREADS, C::SMEM, st>>>(ma, mb, mo, ga);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

template <int L>
int dispatch_gemm(int side, int rp, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo,
                  const GemmArgs& ga, cudaStream_t st) {
#define NNCP_SLICED_CASE(RPV)                                                   \
  case RPV:                                                                     \
    return side == NNCP_SIDE_LEFT ? launch_gemm<NNCP_SIDE_LEFT, RPV, L>(ma, mb, mo, ga, st) \
                                  : launch_gemm<NNCP_SIDE_RIGHT, RPV, L>(ma, mb, mo, ga, st);
  switch (rp) {
    NNCP_SLICED_CASE(16)
    NNCP_SLICED_CASE(32)
    NNCP_SLICED_CASE(48)
    NNCP_SLICED_CASE(64)
    default:
      return fail(NNCP_ERR_UNSUPPORTED, "sliced MTTKRP: rank above NNCP_MAX_RANK");
  }
#undef NNCP_SLICED_CASE
}

int check_levels(int L) {
  if (L != 6 && L != 7) return fail(NNCP_ERR_UNSUPPORTED, "sliced MTTKRP supports 6 or 7 digit levels");
  return NNCP_OK;
}

}  // namespace sliced

// ---------------------------------------------------------- entry points --
size_t sliced_tensor_bytes(int order, const int64_t* dims, int split, int levels) {
  return sliced::tensor_layout(order, dims, split, levels).total;
}

bool sliced_trailing_supported(int order, const int64_t* dims, int split, int rank, int levels) {
  return sliced::plan_call(order, dims, split, NNCP_SIDE_LEFT, rank, levels).fuse;
}

size_t sliced_ws_bytes(int order, const int64_t* dims, int split, int rank, int levels) {
  const auto l = sliced::plan_call(order, dims, split, NNCP_SIDE_LEFT, rank, levels);
  const auto r = sliced::plan_call(order, dims, split, NNCP_SIDE_RIGHT, rank, levels);
  return std::max(l.ws_bytes, r.ws_bytes);
}

// mode 0: row maxima + planes (nncp_slice_tensor); 1: row maxima with the init-row
// facts (nncp_norm_rowmax); 2: planes from row maxima already in the buffer
// (nncp_slice_tensor_planes)
static int slice_tensor_impl(const double* x, int order, const int64_t* dims, int split, int levels, void* out,
                             size_t bytes, cudaStream_t st, int mode, double* norm_out, double* min_out, void* ws,
                             size_t ws_bytes) {
  using namespace sliced;
  if (int rc = check_levels(levels)) return rc;
  const TensorLayout t = tensor_layout(order, dims, split, levels);
  if (bytes < t.total) return fail(NNCP_ERR_VALUE, "sliced tensor buffer too small");
  if (reinterpret_cast<uintptr_t>(out) % 1024) return fail(NNCP_ERR_VALUE, "sliced tensor buffer must be 1 KB aligned");
  if (t.nmb >= (int64_t(1) << 31) || t.njb >= (int64_t(1) << 31))
    return fail(NNCP_ERR_UNSUPPORTED, "sliced MTTKRP: unfolding dimension too large");
  uint8_t* base = static_cast<uint8_t*>(out);
  int* rowexp = reinterpret_cast<int*>(base);
  int8_t* planes = reinterpret_cast<int8_t*>(base + t.plane_off);
  unsigned long long* rmax = reinterpret_cast<unsigned long long*>(base + t.rmax_off);
  const int64_t target = int64_t(num_sms()) * 16;
  if (mode != 2) {
    NNCP_CUDA_TRY(cudaMemsetAsync(rmax, 0, size_t(t.Mp) * 8, st));
    const int64_t mblocks = (t.M + 255) / 256;
    int64_t jsplit = std::max<int64_t>(1, std::min<int64_t>(t.J, (target + mblocks - 1) / mblocks));
    int64_t jper = (t.J + jsplit - 1) / jsplit;
    jsplit = (t.J + jper - 1) / jper;
    if (mode == 1) {
      if (!norm_out || !min_out) return fail(NNCP_ERR_VALUE, "norm outputs required");
      if (t.M * t.J < 1) return fail(NNCP_ERR_VALUE, "min of an empty tensor");
      WsLayout w = ws_layout(ws, ws_bytes);
      if (w.part_elems < size_t(mblocks * jsplit) * 4) return fail(NNCP_ERR_VALUE, "workspace too small (norm)");
      norm_rowmax_kernel<<<dim3(unsigned(mblocks), unsigned(jsplit)), 256, 0, st>>>(
          x, t.M, t.J, jper, rmax, w.part, norm_out, min_out, w.tickets + T_NORM);
      NNCP_LAUNCH_CHECK();
      return NNCP_OK;
    }
    slice_rowmax_kernel<<<dim3(unsigned(mblocks), unsigned(jsplit)), 256, 0, st>>>(x, t.M, t.J, jper, rmax);
    NNCP_LAUNCH_CHECK();
  }
  const int64_t gblocks = (t.Mp / PR + 255) / 256;
  int64_t js2 = std::max<int64_t>(1, std::min<int64_t>(t.Jp, (target + gblocks - 1) / gblocks));
  int64_t jper2 = (t.Jp + js2 - 1) / js2;
  js2 = (t.Jp + jper2 - 1) / jper2;
  const dim3 grid{unsigned(gblocks), unsigned(js2), 1u};
  const bool vec = (t.M % 2 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
#define NNCP_SLICE_LAUNCH(LV, V) \
  slice_planes_kernel<LV, V><<<grid, 256, 0, st>>>(x, t.M, t.J, t.Mp, t.Jp, t.njb, jper2, rmax, rowexp, planes)
  if (levels == 6) {
    if (vec) NNCP_SLICE_LAUNCH(6, true); else NNCP_SLICE_LAUNCH(6, false);
  } else {
    if (vec) NNCP_SLICE_LAUNCH(7, true); else NNCP_SLICE_LAUNCH(7, false);
  }
#undef NNCP_SLICE_LAUNCH
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int slice_tensor(const double* x, int order, const int64_t* dims, int split, int levels, void* out, size_t bytes,
                 cudaStream_t st) {
  return slice_tensor_impl(x, order, dims, split, levels, out, bytes, st, 0, nullptr, nullptr, nullptr, 0);
}

int norm_rowmax(const double* x, int order, const int64_t* dims, int split, int levels, void* out, size_t bytes,
                double* norm_out, double* min_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  return slice_tensor_impl(x, order, dims, split, levels, out, bytes, st, 1, norm_out, min_out, ws, ws_bytes);
}

int slice_tensor_planes(const double* x, int order, const int64_t* dims, int split, int levels, void* out,
                        size_t bytes, cudaStream_t st) {
  return slice_tensor_impl(x, order, dims, split, levels, out, bytes, st, 2, nullptr, nullptr, nullptr, 0);
}

int sliced_partial_mttkrp(const void* sliced_x, int order, const int64_t* dims, int split, int side,
                          const double* const* factors, int rank, int levels, double* out, double* out_trailing,
                          void* ws, size_t ws_bytes, cudaStream_t st, const double** parts_out, int* groups_out,
                          int64_t* gstride_out) {
  using namespace sliced;
  if (int rc = check_levels(levels)) return rc;
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "sliced MTTKRP: rank outside [1, 64]");
  const CallPlan p = plan_call(order, dims, split, side, rank, levels);
  if (ws == nullptr || ws_bytes < p.ws_bytes) return fail(NNCP_ERR_VALUE, "workspace too small for sliced MTTKRP");
  if (reinterpret_cast<uintptr_t>(ws) % 1024) return fail(NNCP_ERR_VALUE, "workspace must be 1 KB aligned");
  const bool left = side == NNCP_SIDE_LEFT;
  if (out_trailing != nullptr && !p.fuse)
    return fail(NNCP_ERR_UNSUPPORTED, "fused trailing TTV needs the left side, split 2, dims[0] % 128 == 0, rank <= 32");
  const uint8_t* base = static_cast<const uint8_t*>(sliced_x);
  const int* rowexp = reinterpret_cast<const int*>(base);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int* bexp = reinterpret_cast<int*>(w + p.bexp_off);
  int8_t* bs = reinterpret_cast<int8_t*>(w + p.bs_off);

  BSpec b{};
  if (left) {
    b.n = order - split;
    for (int f = 0; f < b.n; ++f) {
      b.ptr[f] = factors[split + f];
      b.dim[f] = dims[split + f];
    }
    b.rowexp = nullptr;
  } else {
    b.n = split;
    for (int f = 0; f < b.n; ++f) {
      b.ptr[f] = factors[f];
      b.dim[f] = dims[f];
    }
    b.rowexp = rowexp;
  }
  for (int f = 0; f < b.n; ++f)
    if (!b.ptr[f]) return fail(NNCP_ERR_VALUE, "null factor pointer on the contracted side");
  b.K = p.K;
  b.Kp = p.Kp;
  b.Kc = p.Kc;
  b.R = rank;
  b.RP = p.RP;
  NNCP_CUDA_TRY(cudaMemsetAsync(bexp, 0x80, size_t(p.nchunks) * p.RP * 4, st));   // EXP_NONE
  const unsigned kblocks = unsigned(p.Kp / BK);
  if (int rc = levels == 6 ? dispatch_bslice<6>(b, bexp, bs, kblocks, st) : dispatch_bslice<7>(b, bexp, bs, kblocks, st))
    return rc;

  // A: blocked digit planes as a 5-D tensor {m % 128, j % 128, plane, jb, mb}
  CUtensorMap ma, mb;
  {
    const cuuint64_t d[5] = {BM, BK, cuuint64_t(levels), cuuint64_t(p.t.njb), cuuint64_t(p.t.nmb)};
    const cuuint64_t s[4] = {BM, TILE, cuuint64_t(levels) * TILE, cuuint64_t(p.t.njb) * levels * TILE};
    const cuuint32_t box[5] = {BM, BK, 1, 1, 1};
    if (int rc = encode_u8(&ma, base + p.t.plane_off, 5, d, s, box)) return rc;
  }
  // B: blocked digit rows as a 4-D tensor {k % 128, r, digit, kb}
  {
    const cuuint64_t d[4] = {BK, cuuint64_t(p.RP), cuuint64_t(levels), cuuint64_t(p.Kp / BK)};
    const cuuint64_t s[3] = {BK, cuuint64_t(p.RP) * BK, cuuint64_t(levels) * p.RP * BK};
    const cuuint32_t box[4] = {BK, cuuint32_t(p.RP), cuuint32_t(levels), 1};
    if (int rc = encode_u8(&mb, bs, 4, d, s, box)) return rc;
  }

  GemmArgs ga{};
  int ga_tma_out = 0;
  ga.rows = p.rows;
  ga.nkb = p.Kp / BK;
  ga.kbc = p.Kc / BK;
  ga.nchunks = p.nchunks;
  ga.row_tiles = p.row_tiles;
  ga.groups = p.groups;
  ga.items = p.row_tiles * p.groups;
  ga.rowexp = left ? rowexp : nullptr;
  ga.bexp = bexp;
  ga.out = p.groups > 1 ? reinterpret_cast<double*>(w + p.part_off) : out;
  ga.group_stride = p.rows * rank;
  ga.R = rank;
  // output map (left side: fp64 (M, R) column-major, one 128 x R box per tile; the
  // right side stores directly and ignores it)
  CUtensorMap mo;
  {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t d[2] = {cuuint64_t(p.rows), cuuint64_t(rank)};
    const cuuint64_t st2[1] = {cuuint64_t(p.rows) * sizeof(double)};
    const cuuint32_t box[2] = {BM, cuuint32_t(rank)};
    const cuuint32_t es[2] = {1, 1};
    // TMA needs 16-byte aligned rows: odd M (or an unaligned output) takes direct stores
    const bool ok = left && p.groups == 1 && (p.rows * sizeof(double)) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(out) % 16 == 0;
    if (ok) {
      CUresult r = fn(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, out, d, st2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(NNCP_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string(int(r)));
    } else {
      memset(&mo, 0, sizeof(mo));
    }
    ga_tma_out = ok ? 1 : 0;
  }
  ga.tma_out = ga_tma_out;
  if (out_trailing != nullptr) {
    if (!factors[1]) return fail(NNCP_ERR_VALUE, "null factor pointer for the trailing TTV");
    ga.fuse = 1;
    ga.nib = p.I1 / BM;
    ga.nout = p.nout;
    ga.cf[0] = factors[1];
    ga.tpart = reinterpret_cast<double*>(w + p.part_off);
    ga.slots = p.fslots;
  }
  int rc = levels == 6 ? dispatch_gemm<6>(side, p.RP, ma, mb, mo, ga, st)
                       : dispatch_gemm<7>(side, p.RP, ma, mb, mo, ga, st);
  if (rc) return rc;
  if (parts_out != nullptr) {
    // deferred: the consumer (nncp_update_grouped) sums the group partials itself
    *parts_out = ga.out;
    *groups_out = p.groups;
    *gstride_out = p.groups > 1 ? ga.group_stride : 0;
  } else if (p.groups > 1) {
    const int64_t n = p.rows * rank;
    const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
    group_reduce_kernel<<<blocks, 256, 0, st>>>(ga.out, p.groups, n, n, out);
    NNCP_LAUNCH_CHECK();
  }
  if (out_trailing != nullptr) {
    const int64_t n = p.I1 * rank;
    const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
    ttv_partials_reduce_kernel<<<blocks, 256, 0, st>>>(ga.tpart, ga.items, int(p.fctas), p.nout, p.fslots, p.I1,
                                                       rank, p.RP, out_trailing);
    NNCP_LAUNCH_CHECK();
  }
  return NNCP_OK;
}

}  // namespace nncp

#ifdef NNCP_SLICED_STATS
extern "C" int nncp_sliced_stats(unsigned long long* host, int n, int reset) {
  if (n > 1024 * 8) n = 1024 * 8;
  if (cudaMemcpyFromSymbol(host, nncp::sliced::g_sliced_stats, sizeof(unsigned long long) * n) != cudaSuccess) return 3;
  if (reset) {
    static unsigned long long zeros[1024 * 8];
    if (cudaMemcpyToSymbol(nncp::sliced::g_sliced_stats, zeros, sizeof(zeros)) != cudaSuccess) return 3;
  }
  return 0;
}
#endif
