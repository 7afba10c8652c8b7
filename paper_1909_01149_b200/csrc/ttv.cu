// Multi-TTV children of the dimension tree (dimtree.py:135-175) as streaming
// kernels.  A temporary is column-major (L * J, R) with the leading retained
// mode fastest (dimtree.py:68-99), so block r is the L x J matrix T_r.
//   trailing: out[l, r] = sum_j T_r[l, j] * KRP(coeff)[j, r]   (dimtree.py:159-165)
//   leading : out[j, r] = sum_l T_r[l, j] * H[l, r]             (dimtree.py:166-172)
// Both are HBM-bound (one read of T, R flops per element); loads are coalesced
// along the contiguous leading mode and reductions are fixed-order (warp shuffle
// trees / ordered shared-memory sums), so results are run-to-run deterministic.
#include "common.cuh"

namespace nncp {

struct CoeffSpec {
  const double* ptr[kMaxOrder];
  int64_t dim[kMaxOrder];
  int n;
};

__device__ __forceinline__ double coeff_value(const CoeffSpec& s, int64_t j, int r, int R) {
  double v = 1.0;
  for (int f = 0; f < s.n - 1; ++f) {
    const int64_t d = s.dim[f];
    const int64_t q = j / d;
    v *= __ldg(s.ptr[f] + (j - q * d) * R + r);
    j = q;
  }
  return v * __ldg(s.ptr[s.n - 1] + j * R + r);
}

// One CTA per (32 leading rows, rank r); 8 warps split the trailing index j.
__global__ void __launch_bounds__(256) ttv_trailing_kernel(const double* __restrict__ t, int64_t L, int64_t J,
                                                           const CoeffSpec cs, int R, double* __restrict__ out) {
  __shared__ double part[8][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.y;
  const int64_t l = int64_t(blockIdx.x) * 32 + lane;
  const double* tr = t + L * J * r;
  double s0 = 0.0, s1 = 0.0;
  int64_t j = warp;
  if (l < L) {
    for (; j + 8 < J; j += 16) {
      const double c0 = coeff_value(cs, j, r, R);
      const double c1 = coeff_value(cs, j + 8, r, R);
      s0 = fma(__ldcs(tr + l + L * j), c0, s0);
      s1 = fma(__ldcs(tr + l + L * (j + 8)), c1, s1);
    }
    if (j < J) s0 = fma(__ldcs(tr + l + L * j), coeff_value(cs, j, r, R), s0);
  }
  part[warp][lane] = s0 + s1;
  __syncthreads();
  if (warp == 0 && l < L) {
    double s = part[0][lane];
#pragma unroll
    for (int w = 1; w < 8; ++w) s += part[w][lane];
    out[l + L * r] = s;
  }
}

// One warp per (j, r): lanes stream the contiguous leading mode, shuffle reduce.
__global__ void __launch_bounds__(256) ttv_leading_kernel(const double* __restrict__ t, int64_t L, int64_t J,
                                                          const double* __restrict__ h, int R,
                                                          double* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = int64_t(blockIdx.x) * 8 + warp;
  const int r = blockIdx.y;
  if (j >= J) return;
  const double* col = t + L * J * r + L * j;
  double s0 = 0.0, s1 = 0.0;
  int64_t l = lane;
  for (; l + 32 < L; l += 64) {
    s0 = fma(__ldcs(col + l), __ldg(h + l * R + r), s0);
    s1 = fma(__ldcs(col + l + 32), __ldg(h + (l + 32) * R + r), s1);
  }
  if (l < L) s0 = fma(__ldcs(col + l), __ldg(h + l * R + r), s0);
  const double s = warp_sum(s0 + s1);
  if (lane == 0) out[j + J * r] = s;
}

__global__ void temp_to_rows_kernel(const double* __restrict__ t, int64_t rows, int R, double* __restrict__ out) {
  const int64_t n = rows * R;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e / R;
    const int r = int(e - i * R);
    out[e] = t[i + rows * r];
  }
}

int multi_ttv(const double* temp, int nret, const int64_t* ret_dims, int rank, int side, const double* const* coeff,
              const int64_t* coeff_rows, int ncoeff, double* out, cudaStream_t st) {
  if (nret < 2) return fail(NNCP_ERR_VALUE, "multi_ttv needs at least two retained modes");
  const int64_t L = ret_dims[0];
  int64_t J = 1;
  for (int n = 1; n < nret; ++n) J *= ret_dims[n];
  if (side == NNCP_TTV_TRAILING) {
    if (ncoeff < 1 || ncoeff > kMaxOrder) return fail(NNCP_ERR_VALUE, "bad coefficient count");
    CoeffSpec cs{};
    cs.n = ncoeff;
    int64_t prod = 1;
    for (int f = 0; f < ncoeff; ++f) {
      cs.ptr[f] = coeff[f];
      cs.dim[f] = coeff_rows[f];
      prod *= coeff_rows[f];
    }
    if (prod != J) return fail(NNCP_ERR_VALUE, "coeff rows do not match the trailing dimension");
    dim3 grid(unsigned((L + 31) / 32), unsigned(rank));
    ttv_trailing_kernel<<<grid, 256, 0, st>>>(temp, L, J, cs, rank, out);
  } else if (side == NNCP_TTV_LEADING) {
    if (ncoeff != 1 || coeff_rows[0] != L) return fail(NNCP_ERR_VALUE, "coeff rows do not match the leading dimension");
    dim3 grid(unsigned((J + 7) / 8), unsigned(rank));
    ttv_leading_kernel<<<grid, 256, 0, st>>>(temp, L, J, coeff[0], rank, out);
  } else {
    return fail(NNCP_ERR_VALUE, "side must be trailing or leading");
  }
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int temp_to_rows(const double* temp, int64_t rows, int rank, double* out, cudaStream_t st) {
  const int64_t n = rows * rank;
  if (n == 0) return NNCP_OK;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 4096));
  temp_to_rows_kernel<<<blocks, 256, 0, st>>>(temp, rows, rank, out);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

}  // namespace nncp
