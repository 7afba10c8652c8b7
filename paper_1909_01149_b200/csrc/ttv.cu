// Multi-TTV children of the dimension tree (dimtree.py:135-175) as streaming
// kernels.  A temporary is column-major (L * J, R) with the leading retained
// mode fastest (dimtree.py:68-99), so block r is the L x J matrix T_r.
//   trailing: out[l, r] = sum_j T_r[l, j] * KRP(coeff)[j, r]   (dimtree.py:159-165)
//   leading : out[j, r] = sum_l T_r[l, j] * H[l, r]             (dimtree.py:166-172)
// Both are HBM-bound (one read of T, one FMA per element).  The coefficient
// column of a CTA's rank r is gathered once into shared memory (the factor rows
// are R doubles apart, so reading them per element would cost 4x the sectors of
// T itself), T is streamed with 16-byte loads along the contiguous leading mode,
// and every reduction is fixed-order: run-to-run bitwise deterministic.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace nncp {

struct CoeffSpec {
  const double* ptr[kMaxOrder];
  int64_t dim[kMaxOrder];
  int n;
};

__device__ __forceinline__ double coeff_value(const CoeffSpec& s, int64_t j, int r, int R) {
  double v = 1.0;
#pragma unroll
  for (int f = 0; f < kMaxOrder; ++f) {
    if (f < s.n) {
      int64_t row = j;
      if (f != s.n - 1) {
        const int64_t q = j / s.dim[f];
        row = j - q * s.dim[f];
        j = q;
      }
      v *= __ldg(s.ptr[f] + row * R + r);
    }
  }
  return v;
}

constexpr int kTtvChunk = 4096;  // coefficient entries staged per pass (32 KB)

// trailing: CTA = (tile of 128 leading rows, rank r, part z of the trailing range).
// Lane pairs of rows are read as double2 (when the leading extent is even); the 8
// warps split the CTA's trailing indices, 4 loads in flight per lane; partial sums
// combined in warp order.  When the leading extent is short (few row tiles) the
// trailing range is split over the gridDim.z CTAs of a thread-block cluster, whose
// partials CTA 0 of the cluster adds in cluster-rank order through distributed
// shared memory: more loads in flight without a workspace, still fixed-order.
__global__ void __launch_bounds__(256) ttv_trailing_kernel(const double* __restrict__ t, int64_t L, int64_t J,
                                                           const CoeffSpec cs, int R, double* __restrict__ out,
                                                           bool vec) {
  __shared__ double coef[kTtvChunk];
  __shared__ double2 part[8][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.y;
  const int64_t l0 = int64_t(blockIdx.x) * 128 + 2 * lane;  // this lane: rows l0, l0+1 (+64, +65)
  const double* tr = t + L * J * r;
  const int nz = int(gridDim.z), z = int(blockIdx.z);
  const int64_t jper = (J + nz - 1) / nz, ja = min(J, jper * z), jb = min(J, ja + jper);
  double2 acc0 = make_double2(0.0, 0.0), acc1 = make_double2(0.0, 0.0);
  for (int64_t jc = ja; jc < jb; jc += kTtvChunk) {
    const int nj = int(jb - jc < kTtvChunk ? jb - jc : int64_t(kTtvChunk));
    __syncthreads();
    for (int q = threadIdx.x; q < nj; q += blockDim.x) coef[q] = coeff_value(cs, jc + q, r, R);
    __syncthreads();
    // U trailing indices per iteration: all 2U loads are issued before the FMAs,
    // which run in the same (ascending jj) order as a one-at-a-time loop
    constexpr int U = 4;
    int jj = warp;
    for (; jj + 8 * (U - 1) < nj; jj += 8 * U) {
      double2 v[U][2];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double* col = tr + L * (jc + jj + 8 * u);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t l = l0 + 64 * h;
          if (vec && l + 1 < L) {
            v[u][h] = __ldcs(reinterpret_cast<const double2*>(col + l));
          } else {
            v[u][h].x = (l < L) ? __ldcs(col + l) : 0.0;
            v[u][h].y = (l + 1 < L) ? __ldcs(col + l + 1) : 0.0;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double c = coef[jj + 8 * u];
        acc0.x = fma(v[u][0].x, c, acc0.x);
        acc0.y = fma(v[u][0].y, c, acc0.y);
        acc1.x = fma(v[u][1].x, c, acc1.x);
        acc1.y = fma(v[u][1].y, c, acc1.y);
      }
    }
    for (; jj < nj; jj += 8) {
      const double c = coef[jj];
      const double* col = tr + L * (jc + jj);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t l = l0 + 64 * h;
        double2 v;
        if (vec && l + 1 < L) {
          v = __ldcs(reinterpret_cast<const double2*>(col + l));
        } else {
          v.x = (l < L) ? __ldcs(col + l) : 0.0;
          v.y = (l + 1 < L) ? __ldcs(col + l + 1) : 0.0;
        }
        double2& a = h ? acc1 : acc0;
        a.x = fma(v.x, c, a.x);
        a.y = fma(v.y, c, a.y);
      }
    }
  }
  __syncthreads();
  part[warp][lane] = acc0;
  part[warp][lane + 32] = acc1;
  __syncthreads();
  if (threadIdx.x < 64) {
    double2 s = part[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
      s.x += part[w][threadIdx.x].x;
      s.y += part[w][threadIdx.x].y;
    }
    part[0][threadIdx.x] = s;
  }
  if (nz > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();                                   // every CTA's part[0] is complete
    if (z == 0 && threadIdx.x < 64) {
      double2 s = part[0][threadIdx.x];
      for (int q = 1; q < nz; ++q) {
        const double2 o = cl.map_shared_rank(&part[0][0], q)[threadIdx.x];
        s.x += o.x;
        s.y += o.y;
      }
      part[0][threadIdx.x] = s;
    }
    cl.sync();                                   // the others' shared memory stays alive until read
    if (z != 0) return;
  }
  if (threadIdx.x < 64) {
    const double2 s = part[0][threadIdx.x];
    const int64_t l = int64_t(blockIdx.x) * 128 + 2 * (threadIdx.x & 31) + 64 * (threadIdx.x >> 5);
    if (l < L) out[l + L * r] = s.x;
    if (l + 1 < L) out[l + 1 + L * r] = s.y;
  }
}

// leading: CTA = (rank r, 8 Q consecutive trailing indices j); H[:, r] staged in
// shared memory per pass of kTtvChunk leading rows; each warp owns Q j columns
// (Q < 8 when 8 per warp would leave the grid short of ~4 CTAs per SM: the columns
// of a warp are walked one after another, so fewer per warp is a shorter chain).
template <int Q>
__global__ void __launch_bounds__(256) ttv_leading_kernel(const double* __restrict__ t, int64_t L, int64_t J,
                                                          const double* __restrict__ h, int R,
                                                          double* __restrict__ out, bool vec) {
  __shared__ double hc[kTtvChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.y;
  const int64_t j0 = int64_t(blockIdx.x) * (8 * Q) + warp * Q;
  const double* tr = t + L * J * r;
  double acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  for (int64_t lc = 0; lc < L; lc += kTtvChunk) {
    const int nl = int(L - lc < kTtvChunk ? L - lc : int64_t(kTtvChunk));
    __syncthreads();
    for (int q = threadIdx.x; q < nl; q += blockDim.x) hc[q] = __ldg(h + (lc + q) * R + r);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int64_t j = j0 + q;
      if (j >= J) break;
      const double* col = tr + L * j + lc;
      double s = 0.0;
      if (vec) {
        int l = 2 * lane;
        // 4 loads in flight, FMAs in the same order as the one-at-a-time loop
        for (; l + 192 < nl; l += 256) {
          double2 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(col + l + 64 * u));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            s = fma(v[u].x, hc[l + 64 * u], s);
            s = fma(v[u].y, hc[l + 64 * u + 1], s);
          }
        }
        for (; l < nl; l += 64) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(col + l));
          s = fma(v.x, hc[l], s);
          s = fma(v.y, hc[l + 1], s);
        }
      } else {
        for (int l = lane; l < nl; l += 32) s = fma(__ldcs(col + l), hc[l], s);
      }
      acc[q] += s;
    }
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double s = warp_sum(acc[q]);
    const int64_t j = j0 + q;
    if (lane == 0 && j < J) out[j + J * r] = s;
  }
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
  // 16-byte loads need an even leading extent and an aligned base
  const bool vec = (reinterpret_cast<uintptr_t>(temp) % 16) == 0 && (L % 2) == 0;
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
    // split the trailing range over a cluster of up to 8 CTAs while the grid is short
    // of ~4 CTAs per SM and every part keeps >= 64 trailing indices (8 per warp)
    const int64_t tiles = (L + 127) / 128 * rank, target = 4 * int64_t(num_sms());
    int nz = 1;
    while (nz < 8 && tiles * nz < target && J / (2 * nz) >= 64) nz *= 2;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(unsigned((L + 127) / 128), unsigned(rank), unsigned(nz));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = unsigned(nz);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, ttv_trailing_kernel, temp, L, J, cs, rank, out, vec) != cudaSuccess)
      return fail(NNCP_ERR_CUDA, "ttv_trailing_kernel launch failed");
  } else if (side == NNCP_TTV_LEADING) {
    if (ncoeff != 1 || coeff_rows[0] != L) return fail(NNCP_ERR_VALUE, "coeff rows do not match the leading dimension");
    const int64_t target = 4 * int64_t(num_sms());
    int q = 8;
    while (q > 1 && (J + 8 * q - 1) / (8 * q) * rank < target) q /= 2;
    const dim3 grid(unsigned((J + 8 * q - 1) / (8 * q)), unsigned(rank));
    switch (q) {
      case 8: ttv_leading_kernel<8><<<grid, 256, 0, st>>>(temp, L, J, coeff[0], rank, out, vec); break;
      case 4: ttv_leading_kernel<4><<<grid, 256, 0, st>>>(temp, L, J, coeff[0], rank, out, vec); break;
      case 2: ttv_leading_kernel<2><<<grid, 256, 0, st>>>(temp, L, J, coeff[0], rank, out, vec); break;
      default: ttv_leading_kernel<1><<<grid, 256, 0, st>>>(temp, L, J, coeff[0], rank, out, vec); break;
    }
  } else {
    return fail(NNCP_ERR_VALUE, "side must be trailing or leading");
  }
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

// khatri_rao (tensor_ops.py:121-137) materialised: out[j, r] = prod_f H_f(j_f, r),
// row-major, the first factor's index fastest.  Not on the hot path (the partial
// MTTKRPs generate these rows on the fly); the public khatri_rao() of the mirror.
__global__ void __launch_bounds__(256) khatri_rao_kernel(const CoeffSpec cs, int64_t rows, int R,
                                                         double* __restrict__ out) {
  const int64_t n = rows * R;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / R;
    out[e] = coeff_value(cs, j, int(e - j * R), R);
  }
}

int khatri_rao(const double* const* factors, const int64_t* rows, int count, int rank, double* out, cudaStream_t st) {
  if (count < 1 || count > kMaxOrder) return fail(NNCP_ERR_VALUE, "khatri_rao needs 1..8 factors");
  CoeffSpec cs{};
  cs.n = count;
  int64_t prod = 1;
  for (int f = 0; f < count; ++f) {
    if (rows[f] < 0) return fail(NNCP_ERR_VALUE, "negative factor rows");
    cs.ptr[f] = factors[f];
    cs.dim[f] = rows[f];
    prod *= rows[f];
  }
  const int64_t n = prod * rank;
  if (n == 0) return NNCP_OK;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
  khatri_rao_kernel<<<blocks, 256, 0, st>>>(cs, prod, rank, out);
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
