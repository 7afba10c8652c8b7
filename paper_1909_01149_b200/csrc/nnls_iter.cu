// The remaining update rules of the reference (§8(f) "next"): UCP (updaters.py:77-88),
// ADMM (updaters.py:167-220) and the accelerated projected gradient "NES"
// (updaters.py:223-281) plus the elementwise pieces of Nesterov's outer
// extrapolation (driver.py:452-492).  Same row-parallel structure as nnls.cu:
// S = A^T A is rebuilt per CTA from the Grams, factored once per CTA in shared
// memory (Cholesky / Jacobi), and every row is solved by one warp.  ADMM and NES
// iterate through one launch per inner step; their stopping tests need global
// reductions (the reference's hook), so each step leaves its sums / maxima in a
// small device buffer that the host all-reduces and inspects, as the reference's
// collective-per-step does.
#include <climits>

#include "nnls_common.cuh"

namespace nncp {

// --------------------------------------------------------- small solvers --
// In-place lower Cholesky of the R x R row-major matrix A (+ shift on the diagonal),
// block-cooperative.  Returns false (uniformly) when a pivot is not positive.
static __device__ bool block_cholesky(double* A, int R, double shift) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (shift != 0.0)
    for (int i = threadIdx.x; i < R; i += blockDim.x) A[i * R + i] += shift;
  __syncthreads();
  for (int k = 0; k < R; ++k) {
    if (threadIdx.x == 0) {
      const double d = A[k * R + k];
      if (!(d > 0.0)) bad = 1;
      A[k * R + k] = sqrt(d);
    }
    __syncthreads();
    if (bad) return false;
    const double dk = A[k * R + k];
    for (int i = k + 1 + threadIdx.x; i < R; i += blockDim.x) A[i * R + k] /= dk;
    __syncthreads();
    const int n = R - k - 1;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int i = k + 1 + e / n, j = k + 1 + e % n;
      if (j <= i) A[i * R + j] = fma(-A[i * R + k], A[j * R + k], A[i * R + j]);
    }
    __syncthreads();
  }
  return true;
}

// Warp solve of L L^T x = b (L lower, row-major in smem); lane l holds entries l, l+32.
static __device__ void warp_chol_solve(const double* L, int R, double (&v)[2]) {
  const int lane = threadIdx.x & 31;
  for (int i = 0; i < R; ++i) {  // forward: z_i = (b_i - sum_{k<i} L_ik z_k) / L_ii
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int k = lane + 32 * q;
      if (k < i) p = fma(L[i * R + k], v[q], p);
    }
    p = warp_sum(p);
    if ((i & 31) == lane) {
      const int q = i >> 5;
      const double z = ((q ? v[1] : v[0]) - p) / L[i * R + i];
      if (q) v[1] = z; else v[0] = z;
    }
    __syncwarp();
  }
  for (int i = R - 1; i >= 0; --i) {  // backward: x_i = (z_i - sum_{k>i} L_ki x_k) / L_ii
    double p = 0.0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int k = lane + 32 * q;
      if (k > i && k < R) p = fma(L[k * R + i], v[q], p);
    }
    p = warp_sum(p);
    if ((i & 31) == lane) {
      const int q = i >> 5;
      const double x = ((q ? v[1] : v[0]) - p) / L[i * R + i];
      if (q) v[1] = x; else v[0] = x;
    }
    __syncwarp();
  }
}

static __device__ double trace_over_rank(const double* S, int R) {
  double t = 0.0;
  for (int i = 0; i < R; ++i) t += S[i * R + i];
  return t / R;
}

// ------------------------------------------------------------------ UCP ----
// Cyclic Jacobi eigendecomposition of the symmetric R x R matrix A (smem) by warp 0,
// eigenvectors accumulated in V (columns); A's diagonal ends as the eigenvalues.
static __device__ void warp_jacobi_eigen(double* A, double* V, int R) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < R * R; e += 32) V[e] = (e / R == e % R) ? 1.0 : 0.0;
  __syncwarp();
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int e = lane; e < R * R; e += 32) {
      if (e / R != e % R) off = fma(A[e], A[e], off);
      else dia = fma(A[e], A[e], dia);
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (!(off > 1e-32 * dia)) break;
    for (int p = 0; p < R - 1; ++p) {
      for (int q = p + 1; q < R; ++q) {
        const double apq = A[p * R + q];
        if (apq == 0.0) continue;
        const double app = A[p * R + p], aqq = A[q * R + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        __syncwarp();
        for (int k = lane; k < R; k += 32) {
          const double akp = A[p * R + k], akq = A[q * R + k];
          A[p * R + k] = cs * akp - sn * akq;
          A[q * R + k] = sn * akp + cs * akq;
        }
        __syncwarp();
        for (int k = lane; k < R; k += 32) {
          const double akp = A[k * R + p], akq = A[k * R + q];
          A[k * R + p] = cs * akp - sn * akq;
          A[k * R + q] = sn * akp + cs * akq;
          const double vkp = V[k * R + p], vkq = V[k * R + q];
          V[k * R + p] = cs * vkp - sn * vkq;
          V[k * R + q] = sn * vkp + cs * vkq;
        }
        __syncwarp();
      }
    }
  }
  __syncwarp();
}

// updaters.py:77-88: S H^T = M^T by Cholesky; singular S -> ridge 1e-12 tr(S)/R
// (status[0] bit 0 = the reference's warning); still singular -> the minimum-norm
// least-squares solution np.linalg.lstsq(S, M^T, rcond=None): S = V diag(l) V^T by
// Jacobi, h = V diag(1/l_i for |l_i| > R eps max|l|, else 0) V^T m per row.
// Dynamic shared memory: L (R x R), V (R x R), per-warp coefficients.
__global__ void __launch_bounds__(kRowWarps * 32)
    ucp_kernel(const double* __restrict__ grams, int order, int mode, int R, const double* __restrict__ mrows,
               int64_t rows, double* __restrict__ hhat, double* __restrict__ part, double* nsq, double* beta,
               int* status, unsigned int* ticket, int64_t mld, TailArgs tail) {
  extern __shared__ double dsm[];
  double* L = dsm;                       // R x R (kMaxRank^2 reserved)
  double* V = dsm + kMaxRank * kMaxRank;  // eigenvectors (lstsq fallback only)
  double* coef = V + kMaxRank * kMaxRank;  // kRowWarps x kMaxRank
  __shared__ double red[kRowWarps * 64];
  __shared__ double colbuf[kMaxRank + 1];
  __shared__ double inv_eig[kMaxRank];
  load_hadamard(L, grams, order, mode, R);
  __syncthreads();
  const double ridge = 1e-12 * trace_over_rank(L, R);
  __syncthreads();
  bool ok = block_cholesky(L, R, 0.0);
  bool lstsq = false;
  if (!ok) {
    load_hadamard(L, grams, order, mode, R);  // S again (the failed factorisation overwrote it)
    __syncthreads();
    ok = block_cholesky(L, R, ridge);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, 1);
    if (!ok) {
      lstsq = true;
      load_hadamard(L, grams, order, mode, R);
      __syncthreads();
      if (threadIdx.x < 32) warp_jacobi_eigen(L, V, R);
      __syncthreads();
      if (threadIdx.x == 0) {
        double smax = 0.0;
        for (int i = 0; i < R; ++i) smax = fmax(smax, fabs(L[i * R + i]));
        const double cut = double(R) * 2.220446049250313e-16 * smax;
        for (int i = 0; i < R; ++i) {
          const double l = L[i * R + i];
          inv_eig[i] = (fabs(l) > cut) ? 1.0 / l : 0.0;
        }
      }
      __syncthreads();
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sq[2] = {0.0, 0.0};
  double bsum = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kRowWarps + warp; i < rows; i += int64_t(gridDim.x) * kRowWarps) {
    const double* mr = mrows + i * R;
    double v[2], m[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = lane + 32 * q;
      m[q] = (r < R) ? (mld ? mrows[i + mld * r] : mr[r]) : 0.0;
      v[q] = m[q];
    }
    if (!lstsq) {
      warp_chol_solve(L, R, v);
    } else {
      double* cw = coef + warp * kMaxRank;
      for (int e = 0; e < R; ++e) {   // c_e = (V^T m)_e / l_e
        double p = 0.0;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int k = lane + 32 * q;
          if (k < R) p = fma(V[k * R + e], m[q], p);
        }
        p = warp_sum(p);
        if (lane == 0) cw[e] = p * inv_eig[e];
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 2; ++q) {   // h_k = sum_e V[k, e] c_e
        const int k = lane + 32 * q;
        double h = 0.0;
        if (k < R)
          for (int e = 0; e < R; ++e) h = fma(V[k * R + e], cw[e], h);
        v[q] = h;
      }
      __syncwarp();
    }
    double* hr = hhat + i * R;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = lane + 32 * q;
      if (r < R) {
        hr[r] = v[q];
        sq[q] = fma(v[q], v[q], sq[q]);
        bsum = fma(m[q], v[q], bsum);
      }
    }
  }
  tail.scratch = L;   // the factorisation is dead after the rows
  colsum_epilogue<2>(sq, bsum, R, red, colbuf, part, nsq, beta, ticket, &tail);
}

// ----------------------------------------------------------------- ADMM ----
// One inner step of updaters.py:196-215 for every row:
//   xhat = (S + rho I)^{-1} (m + rho (x + u));  x' = max(xhat - u, 0);  u' = u + x' - xhat
// and the five local squared norms of the stopping test (sums5).  rho <= 0 selects
// default_admm_rho (updaters.py:167-170): tr(S)/R, or 1 when that is not positive.
__global__ void __launch_bounds__(kRowWarps * 32)
    admm_step_kernel(const double* __restrict__ grams, int order, int mode, int R, double rho,
                     const double* __restrict__ mrows, const double* __restrict__ x_in, double* __restrict__ u,
                     double* __restrict__ x_out, int64_t rows, double* __restrict__ part, double* sums5,
                     int* status, unsigned int* ticket) {
  __shared__ double L[kMaxRank * kMaxRank];
  __shared__ double red[8];
  __shared__ double rho_s;
  load_hadamard(L, grams, order, mode, R);
  __syncthreads();
  if (threadIdx.x == 0) {
    double r0 = rho;
    if (!(r0 > 0.0)) {
      r0 = trace_over_rank(L, R);
      if (!(r0 > 0.0)) r0 = 1.0;
    }
    rho_s = r0;
  }
  __syncthreads();
  const double rh = rho_s;
  const bool ok = block_cholesky(L, R, rh);
  if (!ok && blockIdx.x == 0 && threadIdx.x == 0) atomicMax(status + 3, 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (ok) {
    for (int64_t i = int64_t(blockIdx.x) * kRowWarps + warp; i < rows; i += int64_t(gridDim.x) * kRowWarps) {
      double v[2], xo[2], uo[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = lane + 32 * q;
        const bool in = r < R;
        xo[q] = in ? x_in[i * R + r] : 0.0;
        uo[q] = in ? u[i * R + r] : 0.0;
        v[q] = in ? mrows[i * R + r] + rh * (xo[q] + uo[q]) : 0.0;
      }
      warp_chol_solve(L, R, v);  // v = xhat
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = lane + 32 * q;
        if (r < R) {
          const double t = v[q] - uo[q];
          const double xn = (t < 0.0) ? 0.0 : t;
          const double un = uo[q] + xn - v[q];
          x_out[i * R + r] = xn;
          u[i * R + r] = un;
          const double g = xn - v[q], s = xn - xo[q];
          acc[0] = fma(g, g, acc[0]);
          acc[1] = fma(xn, xn, acc[1]);
          acc[2] = fma(v[q], v[q], acc[2]);
          acc[3] = fma(s, s, acc[3]);
          acc[4] = fma(un, un, acc[4]);
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const double b = block_sum(acc[k], red);
    if (threadIdx.x == 0) part[size_t(blockIdx.x) * 5 + k] = b;
  }
  if (last_cta_ticket(ticket)) {
    finish_partials(part, gridDim.x, 5, sums5);
    if (threadIdx.x == 0) sums5[5] = rh;  // the rho actually used, for the host-side stopping test
  }
}

// ------------------------------------------------------------ Nesterov ----
// nesterov_hyperparams (updaters.py:223-243): cyclic Jacobi eigenvalues of S in one
// warp, then (lam, alpha, beta) from the extreme eigenvalues.
__global__ void __launch_bounds__(32)
    nes_hyper_kernel(const double* __restrict__ grams, int order, int mode, int R, double prox_floor,
                     double* __restrict__ hyper) {
  __shared__ double A[kMaxRank * kMaxRank];
  load_hadamard(A, grams, order, mode, R);
  __syncwarp();
  const int lane = threadIdx.x;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int e = lane; e < R * R; e += 32) {
      const int i = e / R, j = e % R;
      if (i != j) off = fma(A[e], A[e], off);
      else dia = fma(A[e], A[e], dia);
    }
    off = warp_sum(off);
    dia = warp_sum(dia);
    if (!(off > 1e-30 * dia)) break;
    for (int p = 0; p < R - 1; ++p) {
      for (int q = p + 1; q < R; ++q) {
        const double apq = A[p * R + q];
        if (apq == 0.0) continue;
        const double app = A[p * R + p], aqq = A[q * R + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        __syncwarp();
        // rotate rows p, q then columns p, q (A stays symmetric)
        for (int k = lane; k < R; k += 32) {
          const double akp = A[p * R + k], akq = A[q * R + k];
          A[p * R + k] = cs * akp - sn * akq;
          A[q * R + k] = sn * akp + cs * akq;
        }
        __syncwarp();
        for (int k = lane; k < R; k += 32) {
          const double akp = A[k * R + p], akq = A[k * R + q];
          A[k * R + p] = cs * akp - sn * akq;
          A[k * R + q] = sn * akp + cs * akq;
        }
        __syncwarp();
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    double big = A[0], small = A[0];
    for (int i = 1; i < R; ++i) {
      big = fmax(big, A[i * R + i]);
      small = fmin(small, A[i * R + i]);
    }
    small = fmax(small, 0.0);
    double lam;
    if (big <= 0.0) lam = 1.0;
    else if (small / big >= prox_floor) lam = 0.0;
    else lam = (prox_floor * big - small) / (1.0 - prox_floor);
    const double qv = (small + lam) / (big + lam);
    hyper[0] = lam;
    hyper[1] = 1.0 / (big + lam);
    hyper[2] = (1.0 - sqrt(qv)) / (1.0 + sqrt(qv));
  }
}

// One accelerated projected-gradient step (updaters.py:266-277) for every row:
//   grad = y S - m + lam (y - x*);  x' = max(y - alpha grad, 0);  y' = x' + beta (x' - x)
// plus the local max |x' - x| and max |x'| (maxes2) of the stopping test.
__global__ void __launch_bounds__(kRowWarps * 32)
    nes_step_kernel(const double* __restrict__ grams, int order, int mode, int R, const double* __restrict__ hyper,
                    const double* __restrict__ mrows, const double* __restrict__ y_in, const double* __restrict__ x_in,
                    const double* __restrict__ xstar, double* __restrict__ x_out, double* __restrict__ y_out,
                    int64_t rows, double* __restrict__ part, double* maxes2, unsigned int* ticket) {
  __shared__ double S[kMaxRank * kMaxRank];
  __shared__ double red[8][2];
  load_hadamard(S, grams, order, mode, R);
  __syncthreads();
  const double lam = hyper[0], alpha = hyper[1], beta = hyper[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double dmax = 0.0, xmax = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kRowWarps + warp; i < rows; i += int64_t(gridDim.x) * kRowWarps) {
    double y[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = lane + 32 * q;
      y[q] = (r < R) ? y_in[i * R + r] : 0.0;
    }
    double d[2] = {0.0, 0.0};
    for (int cc = 0; cc < R; ++cc) {
      const double yc = __shfl_sync(0xffffffffu, cc < 32 ? y[0] : y[1], cc & 31);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = lane + 32 * q;
        if (r < R) d[q] = fma(yc, S[cc * R + r], d[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = lane + 32 * q;
      if (r < R) {
        const int64_t e = i * R + r;
        const double grad = (d[q] - mrows[e]) + lam * (y[q] - xstar[e]);
        const double t = y[q] - alpha * grad;
        const double xn = (t < 0.0) ? 0.0 : t;
        const double xo = x_in[e];
        x_out[e] = xn;
        y_out[e] = xn + beta * (xn - xo);
        dmax = fmax(dmax, fabs(xn - xo));
        xmax = fmax(xmax, fabs(xn));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
  }
  if (lane == 0) {
    red[warp][0] = dmax;
    red[warp][1] = xmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = red[0][0], b = red[0][1];
    for (int w = 1; w < kRowWarps; ++w) {
      a = fmax(a, red[w][0]);
      b = fmax(b, red[w][1]);
    }
    part[size_t(blockIdx.x) * 2] = a;
    part[size_t(blockIdx.x) * 2 + 1] = b;
  }
  if (last_cta_ticket(ticket)) {
    if (threadIdx.x < 2) {
      double m = part[threadIdx.x];
      for (unsigned k = 1; k < gridDim.x; ++k) m = fmax(m, part[size_t(k) * 2 + threadIdx.x]);
      maxes2[threadIdx.x] = m;
    }
  }
}

// ----------------------------------------------------------- elementwise ----
__global__ void scale_columns_kernel(const double* __restrict__ in, const double* __restrict__ scale, int64_t rows,
                                     int R, double* __restrict__ out) {
  const int64_t n = rows * R;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    out[e] = in[e] * scale[e % R];
}

// driver.py:464-470: max(h + step (h - h_prev), 0)
__global__ void extrapolate_kernel(const double* __restrict__ cur, const double* __restrict__ prev, int64_t n,
                                   double step, double* __restrict__ out) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const double v = cur[e] + step * (cur[e] - prev[e]);
    out[e] = (v < 0.0) ? 0.0 : v;
  }
}

// driver.py:482-486: lam = cand_lam * prod_n sqrt(nsq_n)
__global__ void nes_lambda_kernel(const double* __restrict__ cand_lam, const double* __restrict__ nsq, int order,
                                  int R, double* __restrict__ lam) {
  const int r = threadIdx.x;
  if (r >= R) return;
  double p = 1.0;
  for (int n = 0; n < order; ++n) p = (n == 0) ? sqrt(nsq[r]) : p * sqrt(nsq[size_t(n) * R + r]);
  lam[r] = cand_lam[r] * p;
}

// column sums of squares (driver.py:479)
__global__ void __launch_bounds__(kRowWarps * 32)
    colsumsq_kernel(const double* __restrict__ h, int64_t rows, int R, double* __restrict__ part, double* nsq,
                    unsigned int* ticket) {
  __shared__ double red[kRowWarps * 64];
  __shared__ double colbuf[kMaxRank + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sq[2] = {0.0, 0.0};
  for (int64_t i = int64_t(blockIdx.x) * kRowWarps + warp; i < rows; i += int64_t(gridDim.x) * kRowWarps) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int r = lane + 32 * q;
      if (r < R) sq[q] = fma(h[i * R + r], h[i * R + r], sq[q]);
    }
  }
  colsum_epilogue<2>(sq, 0.0, R, red, colbuf, part, nsq, nullptr, ticket);
}

// ------------------------------------------------------------- host side ---
int row_blocks(int64_t rows);

static int grid_rows(int64_t rows) { return row_blocks(rows); }

int ucp(const double* grams, int order, int mode, int rank, const double* mrows, int64_t rows, double* hhat,
        double* nsq, double* beta, int* status, void* ws, size_t ws_bytes, cudaStream_t st, int64_t mld,
        const TailArgs* tail) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int blocks = grid_rows(rows);
  if (w.part_elems < size_t(blocks) * (rank + 1)) return fail(NNCP_ERR_VALUE, "workspace too small (ucp)");
  constexpr int smem = int(sizeof(double)) * (2 * kMaxRank * kMaxRank + kRowWarps * kMaxRank);
  if (int rc = set_max_smem_once<ucp_kernel>(smem)) return rc;
  ucp_kernel<<<blocks, kRowWarps * 32, smem, st>>>(grams, order, mode, rank, mrows, rows, hhat, w.part, nsq, beta,
                                                   status, w.tickets + T_UPDATE, mld, tail ? *tail : TailArgs{});
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int admm_step(const double* grams, int order, int mode, int rank, double rho, const double* mrows, const double* x_in,
              double* u, double* x_out, int64_t rows, double* sums5, int* status, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int blocks = grid_rows(rows);
  if (w.part_elems < size_t(blocks) * 5) return fail(NNCP_ERR_VALUE, "workspace too small (admm)");
  admm_step_kernel<<<blocks, kRowWarps * 32, 0, st>>>(grams, order, mode, rank, rho, mrows, x_in, u, x_out, rows,
                                                       w.part, sums5, status, w.tickets + T_ITER);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int nes_hyper(const double* grams, int order, int mode, int rank, double prox_floor, double* hyper, cudaStream_t st) {
  nes_hyper_kernel<<<1, 32, 0, st>>>(grams, order, mode, rank, prox_floor, hyper);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int nes_step(const double* grams, int order, int mode, int rank, const double* hyper, const double* mrows,
             const double* y_in, const double* x_in, const double* xstar, double* x_out, double* y_out, int64_t rows,
             double* maxes2, void* ws, size_t ws_bytes, cudaStream_t st) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int blocks = grid_rows(rows);
  if (w.part_elems < size_t(blocks) * 2) return fail(NNCP_ERR_VALUE, "workspace too small (nes)");
  nes_step_kernel<<<blocks, kRowWarps * 32, 0, st>>>(grams, order, mode, rank, hyper, mrows, y_in, x_in, xstar, x_out,
                                                      y_out, rows, w.part, maxes2, w.tickets + T_ITER);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

static int elem_blocks(int64_t n) { return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4096))); }

int scale_columns(const double* in, const double* scale, int64_t rows, int rank, double* out, cudaStream_t st) {
  if (rows * rank == 0) return NNCP_OK;
  scale_columns_kernel<<<elem_blocks(rows * rank), 256, 0, st>>>(in, scale, rows, rank, out);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int extrapolate(const double* cur, const double* prev, int64_t n, double step, double* out, cudaStream_t st) {
  if (n == 0) return NNCP_OK;
  extrapolate_kernel<<<elem_blocks(n), 256, 0, st>>>(cur, prev, n, step, out);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int nes_lambda(const double* cand_lam, const double* nsq, int order, int rank, double* lam, cudaStream_t st) {
  nes_lambda_kernel<<<1, 64, 0, st>>>(cand_lam, nsq, order, rank, lam);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int colsumsq(const double* h, int64_t rows, int rank, double* nsq, void* ws, size_t ws_bytes, cudaStream_t st) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int blocks = grid_rows(rows);
  if (w.part_elems < size_t(blocks) * (rank + 1)) return fail(NNCP_ERR_VALUE, "workspace too small (colsumsq)");
  colsumsq_kernel<<<blocks, kRowWarps * 32, 0, st>>>(h, rows, rank, w.part, nsq, w.tickets + T_COLSQ);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

}  // namespace nncp
