// Normal-equation side of the ALS step: Hadamard-of-Grams, MU / HALS / ANLS-BPP
// row updates, column norms, normalisation, Gram matrices, error terms.
// References: tensor_ops.py:140-155, updaters.py:91-164, driver.py:396-433.
//
// Every factor row is an independent NNLS problem (updaters.py:1-8), so the
// updates run one thread (MU, HALS) or one warp (BPP) per row with S = A^T A
// staged once per CTA in shared memory.  Column sums (norms, beta, Grams) use
// per-CTA partials plus a last-CTA fixed-order reduction: deterministic and a
// single launch.
#include <climits>

#include "nnls_common.cuh"

namespace nncp {

template <int ALGO, int RP>
__global__ void __launch_bounds__(kRowWarps * 32)
    update_rows_kernel(const double* __restrict__ grams, int order, int mode, int R,
                       const double* __restrict__ mrows, const double* __restrict__ owned,
                       const double* __restrict__ lam, int64_t rows, double* __restrict__ hhat,
                       double* __restrict__ part, double* nsq, double* beta, int* status, unsigned int* ticket,
                       double mu_eps, int64_t mld, TailArgs tail) {
  __shared__ double S[kMaxRank * kMaxRank];
  __shared__ double red[kRowWarps * 64];
  __shared__ double colbuf[kMaxRank + 1];
  __shared__ double inv_diag[kMaxRank];
  constexpr int NH = (RP + 31) / 32;   // column slots per lane
#ifdef NNCP_UPD_TIMING
  const long long tu0 = clock64();
#endif
  load_hadamard(S, grams, order, mode, R);
  __syncthreads();
  // HALS: 1 / S_rr once per CTA (the same quotient the row loop formed per column,
  // off the column chain)
  if (ALGO == NNCP_ALGO_HALS)
    for (int r = threadIdx.x; r < R; r += blockDim.x) inv_diag[r] = 1.0 / S[r * R + r];
  __syncthreads();
#ifdef NNCP_UPD_TIMING
  const long long tu1 = clock64();
#endif
  if (ALGO == NNCP_ALGO_HALS && blockIdx.x == 0) {
    for (int r = threadIdx.x; r < R; r += blockDim.x)
      if (S[r * R + r] <= 0.0) atomicOr(status + (r >> 5), int(1u << (r & 31)));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double sq[2] = {0.0, 0.0};
  double bsum = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * kRowWarps + warp; i < rows; i += int64_t(gridDim.x) * kRowWarps) {
    const double* orow = owned + i * R;
    const double* mr = mrows + i * R;
    double h[2] = {0.0, 0.0}, m[2] = {0.0, 0.0};
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int r = lane + 32 * q;
      h[q] = (r < R) ? (lam ? orow[r] * lam[r] : orow[r]) : 0.0;  // driver.py:403 current = owned * lam
      // M row-major, or (mld > 0) the dimension tree's column-major temporary itself
      m[q] = (r < R) ? load_m(mrows, mld, i, r, R, tail) : 0.0;
    }
    if (ALGO == NNCP_ALGO_MU) {
      // updaters.py:93-94: current * M / (current @ S + eps)
      double d[2] = {0.0, 0.0};
#pragma unroll
      for (int cc = 0; cc < RP; ++cc) {
        if (cc >= R) break;
        const double hc = __shfl_sync(0xffffffffu, cc < 32 ? h[0] : h[1], cc & 31);
#pragma unroll
        for (int q = 0; q < NH; ++q) {
          const int r = lane + 32 * q;
          if (r < R) d[q] = fma(hc, S[cc * R + r], d[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < NH; ++q) {
        const int r = lane + 32 * q;
        h[q] = (r < R) ? h[q] * m[q] / (d[q] + mu_eps) : 0.0;
      }
    } else {
      // updaters.py:107-118: Gauss-Seidel over columns with the latest values,
      // h_r <- max(0, h_r + (m_r - (h S)_r) / S_rr).  Instead of a fresh warp-reduced
      // dot product per column (a 5-level shuffle tree on the sequential column
      // chain), every lane keeps g_c = (h S)_c for its columns c, split the way the
      // reference's dot product sees h at column c: the old values of columns j >= c
      // (summed up front) plus the new values of columns j < c (added as each column
      // finishes: one broadcast and one FMA).  Never old-minus-new deltas: when a
      // column is wiped out its O(1) old value must leave g exactly, or the rounding
      // of the cancellation lands on the tiny survivors (tensors far below the initial
      // factors' scale).  The quotient is the reciprocal product plus one FMA residual
      // correction (the correctly rounded division in all but rare tie cases), the
      // reciprocal formed off the chain.
      double g[2] = {0.0, 0.0};
#pragma unroll
      for (int j = 0; j < RP; ++j) {
        if (j >= R) break;
        const double hj = __shfl_sync(0xffffffffu, j < 32 ? h[0] : h[1], j & 31);
#pragma unroll
        for (int q = 0; q < NH; ++q) {
          const int c = lane + 32 * q;
          if (c < R && j >= c) g[q] = fma(hj, S[j * R + c], g[q]);    // sum_{j >= c} h_j S[j][c]
        }
      }
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        if (r >= R) break;
        const double dg = S[r * R + r];
        const double idg = inv_diag[r];
        const int q = r >> 5;
        // every lane evaluates the column step on its own slot, branch-free; lane r % 32's
        // value is the one broadcast (no divergent region on the column chain)
        const double hv = q ? h[1] : h[0];
        const double num = (q ? m[1] : m[0]) - (q ? g[1] : g[0]);
        const double q0 = num * idg;
        const double quo = fma(fma(-q0, dg, num), idg, q0);
        const double col = hv + quo;
        double v = (dg > 0.0) ? ((col < 0.0) ? 0.0 : col) : hv;   // a skipped column (S_rr <= 0) keeps its value
        v = __shfl_sync(0xffffffffu, v, r & 31);
        if ((r & 31) == lane) {
          if (q) h[1] = v; else h[0] = v;
        }
        if (v != 0.0) {
#pragma unroll
          for (int qq = 0; qq < NH; ++qq) {
            const int c = lane + 32 * qq;
            if (c < R && c > r) g[qq] = fma(v, S[r * R + c], g[qq]);
          }
        }
      }
    }
    double* hr = hhat + i * R;
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int r = lane + 32 * q;
      if (r < R) {
        hr[r] = h[q];
        sq[q] = fma(h[q], h[q], sq[q]);
        bsum = fma(m[q], h[q], bsum);
      }
    }
  }
  tail.scratch = S;   // S is dead after the rows
#ifdef NNCP_UPD_TIMING
  const long long tu2 = clock64();
#endif
  colsum_epilogue<2>(sq, bsum, R, red, colbuf, part, nsq, beta, ticket, &tail);
#ifdef NNCP_UPD_TIMING
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("update cta %d/%d: hadamard %lld rows %lld epilogue %lld (start %lld)\n", blockIdx.x, gridDim.x, tu1 - tu0,
           tu2 - tu1, clock64() - tu2, tu0 % 1000000);
#endif
}

// ------------------------------------------------------------------ BPP ----
// One warp per row: block principal pivoting (updaters.py:121-155).
constexpr int kBppWarps = 4;   // warps per CTA at R > 48 (shared-memory bound)
// Warps per CTA: the block-level S^-1 is a 2R-step Gauss-Jordan chain -- latency-bound,
// so it wants many warps; every warp then solves its own rows.  The per-warp LU scratch
// (R x (R+1) doubles) caps the count at large R.
template <int RP>
constexpr int bpp_warps() { return RP <= 32 ? 16 : (RP <= 48 ? 8 : kBppWarps); }

// Warp LU with partial pivoting (first-max pivot, like dgesv) of the m x m system in A
// (pitch LP, right-hand side in column m); the solution overwrites column m.  False
// when a pivot is exactly zero (what makes np.linalg.solve raise LinAlgError).
template <int RP>
__device__ bool warp_lu_solve(double* A, int m, int LP) {
  constexpr int NH = (RP + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (int cidx = 0; cidx < m; ++cidx) {
    // pivot: max |A[i][c]| over i >= c, first index on ties (idamax).  Exact warp
    // argmax in three reductions: |v| >= 0 orders like its bit pattern, so max of the
    // high words, then of the low words among those, then the smallest row index
    // among the exact maxima.
    double bv = -1.0;
    int bi = INT_MAX;
    for (int a = cidx + lane; a < m; a += 32) {
      const double v = fabs(A[a * LP + cidx]);
      if (v > bv) {
        bv = v;
        bi = a;
      }
    }
    {
      const bool cand = bi != INT_MAX;
      const unsigned long long bits = cand ? (unsigned long long)__double_as_longlong(bv) : 0ull;
      const uint32_t mh = __reduce_max_sync(0xffffffffu, uint32_t(bits >> 32));
      const unsigned tie = __ballot_sync(0xffffffffu, cand && uint32_t(bits >> 32) == mh);
      if (__popc(tie) == 1) {   // one lane holds the high-word maximum: its (value, row) wins
        const int src = __ffs(tie) - 1;
        bi = __shfl_sync(0xffffffffu, bi, src);
        bv = __shfl_sync(0xffffffffu, bv, src);
      } else {
        const uint32_t ml =
            __reduce_max_sync(0xffffffffu, (cand && uint32_t(bits >> 32) == mh) ? uint32_t(bits) : 0u);
        const bool win = cand && uint32_t(bits >> 32) == mh && uint32_t(bits) == ml;
        bi = int(__reduce_min_sync(0xffffffffu, win ? uint32_t(bi) : 0xffffffffu));
        bv = __hiloint2double(int(mh), int(ml));
      }
    }
    if (!(bv > 0.0)) return false;
    // the pivot (row bi before the swap); its reciprocal overlaps the swap
    const double piv = A[bi * LP + cidx];
    __syncwarp();
    const double inv = 1.0 / piv;
    if (bi != cidx) {
      for (int b = lane; b <= m; b += 32) {
        const double t0 = A[cidx * LP + b];
        A[cidx * LP + b] = A[bi * LP + b];
        A[bi * LP + b] = t0;
      }
    }
    __syncwarp();
    for (int a = cidx + 1 + lane; a < m; a += 32) {
      const double l = A[a * LP + cidx] * inv;
      A[a * LP + cidx] = l;
      double* ra = A + a * LP;
      const double* rc = A + cidx * LP;
      int b = cidx + 1;
      // 8 columns per batch: all loads issued before the FMAs (same arithmetic,
      // eight independent shared-memory round trips in flight instead of one)
      for (; b + 8 <= m + 1; b += 8) {
        double x[8], y[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q] = rc[b + q];
          y[q] = ra[b + q];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) ra[b + q] = fma(-l, x[q], y[q]);
      }
      for (; b <= m; ++b) ra[b] = fma(-l, rc[b], ra[b]);
    }
    __syncwarp();
  }
  // back substitution in column (axpy) order, as dtrsm does it: the right-hand side
  // lives in registers (lane k holds rows k, k + 32); per step one division on the
  // owning lane, one broadcast, one FMA per remaining row.
  double bq[NH];
#pragma unroll
  for (int q = 0; q < NH; ++q) {
    const int k = lane + 32 * q;
    bq[q] = k < m ? A[k * LP + m] : 0.0;
  }
  for (int a = m - 1; a >= 0; --a) {
    const int src = a & 31, qa = a >> 5;
    double mine = 0.0;
#pragma unroll
    for (int q = 0; q < NH; ++q)
      if (q == qa) mine = bq[q];
    const double xa = __shfl_sync(0xffffffffu, mine / A[a * LP + a], src);
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int k = lane + 32 * q;
      if (k == a) bq[q] = xa;
      else if (k < a) bq[q] = fma(-A[k * LP + a], xa, bq[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NH; ++q) {
    const int k = lane + 32 * q;
    if (k < m) A[k * LP + m] = bq[q];
  }
  __syncwarp();
  return true;
}

// acc_i = sum_{j in P} M[i][j] x_j for every i, M given as M^T (lane i reads row j:
// lane-consecutive addresses); x broadcast from the registers of its lanes.  Fully
// unrolled over j so the shuffles and loads overlap (a loop over the set bits of P
// was one dependent round trip per term).
template <int RP>
__device__ void bpp_matvec(const double* MT, int R, unsigned long long P, const double (&xs)[(RP + 31) / 32],
                           double (&acc)[(RP + 31) / 32]) {
  constexpr int NH = (RP + 31) / 32;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < NH; ++q) acc[q] = 0.0;
#pragma unroll
  for (int j = 0; j < RP; ++j) {
    const double xj = __shfl_sync(0xffffffffu, xs[j >> 5], j & 31);
    if (j < R && ((P >> j) & 1ull)) {
#pragma unroll
      for (int q = 0; q < NH; ++q) {
        const int i = lane + 32 * q;
        if (i < R) acc[q] = fma(MT[j * R + i], xj, acc[q]);
      }
    }
  }
}

// y = S[~P,P] x_P - f[~P] on the active indices, 0 on the passive ones (updaters.py:153-154)
template <int RP>
__device__ void bpp_dual(const double* S, int R, unsigned long long P, const double (&xs)[(RP + 31) / 32],
                         const double (&fs)[(RP + 31) / 32], double (&ys)[(RP + 31) / 32]) {
  constexpr int NH = (RP + 31) / 32;
  const int lane = threadIdx.x & 31;
  double acc[NH];
  bpp_matvec<RP>(S, R, P, xs, acc);
#pragma unroll
  for (int q = 0; q < NH; ++q) {
    const int i = lane + 32 * q;
    ys[q] = (i < R && !((P >> i) & 1ull)) ? acc[q] - fs[q] : 0.0;
  }
}

// x, y for passive set P by the reference's direct solve: S[P,P] x_P = f_P (LU as
// np.linalg.solve), y from S.  False when S[P,P] is singular.
template <int RP>
__device__ bool bpp_eval_direct(const double* S, int R, const double* fr, unsigned long long P, double* A, int* pidx,
                                const double (&fs)[(RP + 31) / 32], double (&xs)[(RP + 31) / 32],
                                double (&ys)[(RP + 31) / 32]) {
  constexpr int NH = (RP + 31) / 32;
  constexpr int LP = RP + 1;
  const int lane = threadIdx.x & 31;
  const int p = __popcll(P);
#pragma unroll
  for (int q = 0; q < NH; ++q) xs[q] = 0.0;
  if (p > 0) {
    // passive index list: variable r in P is the popc(P below r)-th entry
    for (int r = lane; r < R; r += 32)
      if ((P >> r) & 1ull) pidx[__popcll(P & ((1ull << r) - 1ull))] = r;
    __syncwarp();
    for (int a = lane; a < p; a += 32) {
      const int ra = pidx[a];
      for (int b = 0; b < p; ++b) A[a * LP + b] = S[pidx[b] * R + ra];   // S^T[pb][ra] = S[ra][pb]
      A[a * LP + p] = fr[ra];
    }
    __syncwarp();
    if (!warp_lu_solve<RP>(A, p, LP)) return false;
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int r = lane + 32 * q;
      if (r < R && ((P >> r) & 1ull)) xs[q] = A[__popcll(P & ((1ull << r) - 1ull)) * LP + p];
    }
    __syncwarp();
  }
  bpp_dual<RP>(S, R, P, xs, fs, ys);
  return true;
}

// Warp solve of a symmetric positive definite m x m system (pitch LP, rhs in column m)
// by elimination without pivoting; the solution overwrites column m.  False when a
// pivot is not positive (the caller then solves directly).
__device__ bool warp_spd_solve(double* A, int m, int LP) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < m; ++c) {
    const double piv = A[c * LP + c];
    if (!(piv > 0.0)) return false;
    const double inv = 1.0 / piv;
    for (int a = c + 1 + lane; a < m; a += 32) {
      const double l = A[a * LP + c] * inv;
      for (int b = c + 1; b <= m; ++b) A[a * LP + b] = fma(-l, A[c * LP + b], A[a * LP + b]);
    }
    __syncwarp();
  }
  for (int a = m - 1; a >= 0; --a) {   // back substitution, one row per step
    if (lane == 0) {
      double v = A[a * LP + m];
      for (int b = a + 1; b < m; ++b) v = fma(-A[a * LP + b], A[b * LP + m], v);
      A[a * LP + m] = v / A[a * LP + a];
    }
    __syncwarp();
  }
  return true;
}

// x for passive set P from T = S^-1 (held as T^T) when few variables are active
// (q = R - p small): with Q the active set, the constrained solve is
//   x = T f~ - T[:,Q] w,  T[Q,Q] w = (T f~)_Q     (f~ = f on P, 0 on Q)
// -- block elimination of the KKT system: one q x q solve instead of a p x p one.
// False when T[Q,Q] is not numerically positive definite (the caller solves directly).
template <int RP>
__device__ bool bpp_schur(const double* TT, int R, unsigned long long P, double* A, int* qidx, double* zbuf,
                          const double (&rhs)[(RP + 31) / 32], double (&xs)[(RP + 31) / 32]) {
  constexpr int NH = (RP + 31) / 32;
  constexpr int LP = RP + 1;
  const int lane = threadIdx.x & 31;
  const unsigned long long all = R < 64 ? ((1ull << R) - 1ull) : ~0ull;
  const unsigned long long Q = all & ~P;
  const int q = __popcll(Q);
  double z[NH];
  bpp_matvec<RP>(TT, R, P, rhs, z);     // z = T f~
  if (q > 0) {
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      const int i = lane + 32 * k;
      if (i < R) zbuf[i] = z[k];
    }
    for (int r = lane; r < R; r += 32)
      if ((Q >> r) & 1ull) qidx[__popcll(Q & ((1ull << r) - 1ull))] = r;
    __syncwarp();
    for (int e = lane; e < q * q; e += 32) {
      const int a = e / q, b = e - (e / q) * q;
      A[a * LP + b] = TT[qidx[b] * R + qidx[a]];   // T[qa][qb]
    }
    for (int a = lane; a < q; a += 32) A[a * LP + q] = zbuf[qidx[a]];
    __syncwarp();
    if (!warp_spd_solve(A, q, LP)) return false;
    for (int a = 0; a < q; ++a) {
      const double wa = A[a * LP + q];
      const int ra = qidx[a];
#pragma unroll
      for (int k = 0; k < NH; ++k) {
        const int i = lane + 32 * k;
        if (i < R) z[k] = fma(-TT[ra * R + i], wa, z[k]);   // T[i][ra]
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < NH; ++k) {
    const int i = lane + 32 * k;
    xs[k] = (i < R && ((P >> i) & 1ull)) ? z[k] : 0.0;
  }
  return true;
}

// T^T = (S^-1)^T for the block-elimination passes, by Gauss-Jordan on [S | I] without
// pivoting (S = Hadamard of Grams is symmetric positive definite when nonsingular: the
// pivots are Schur complements).  Block-cooperative, one barrier per step; returns
// false (uniformly) when a pivot is not comfortably positive -- the kernel then solves
// every pass directly.  (A Newton-Schulz refresh from the previous sweep's inverse was
// measured slower: S moves by 1e-2..1 between sweeps early on, and each R^3 product in
// shared memory cost about as much as the whole elimination.)
template <int RP>
__device__ bool block_inverse(const double* S, int R, double* aug, double* TT, double* gj) {
  constexpr int W = 2 * RP;   // [S | I] with row pitch 2 RP; warp w owns rows w, w + nw, ...
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // the step's pivot row and column (unscaled, as the previous step left them) in
  // double-buffered shared rows: whoever writes an element of the next pivot row or
  // column also stores it there, so each step needs ONE block barrier
  double* rowb[2] = {gj, gj + 2 * RP};            // 2 RP each
  double* colb[2] = {gj + 4 * RP, gj + 5 * RP};   // RP each
  for (int i = warp; i < R; i += nw)
    for (int j = lane; j < 2 * R; j += 32) {
      const double v = j < R ? S[j * R + i] : (j - R == i ? 1.0 : 0.0);
      aug[i * W + j] = v;
      if (i == 0) rowb[0][j] = v;
      if (j == 0) colb[0][i] = v;
    }
  __syncthreads();
  for (int c = 0; c < R; ++c) {
    const double* row = rowb[c & 1];
    const double* col = colb[c & 1];
    double* nrow = rowb[(c + 1) & 1];
    double* ncol = colb[(c + 1) & 1];
    const double piv = row[c];
    if (!(piv > 1e-8 * fabs(S[c * R + c]))) return false;   // uniform: every thread reads the same piv
    const double inv = 1.0 / piv;
    for (int i = warp; i < R; i += nw) {
      const double f = col[i];
      for (int j = lane; j < 2 * R; j += 32) {
        const double pr = row[j] * inv;
        const double v = (i == c) ? pr : fma(-f, pr, aug[i * W + j]);
        aug[i * W + j] = v;
        if (i == c + 1) nrow[j] = v;
        if (j == c + 1) ncol[i] = v;
      }
    }
    __syncthreads();
  }
  for (int i = warp; i < R; i += nw)
    for (int j = lane; j < R; j += 32) TT[j * R + i] = aug[i * W + R + j];
  __syncthreads();
  return true;
}

// BPP's S and S^-1 prepared ahead of the update (nncp_bpp_prepare, launched on another
// stream while the mode's MTTKRP runs -- S needs only the Grams): a block after the
// caller's passive sets, uint64 sets[rows rounded up to 2], then
//   [0] key (0 = none), [1] t_ok, [2..3] unused, S^T (R x R), S^-1 transposed (R x R).
// The update takes S and S^-1 from it when the key matches (order, mode, R) and its
// last CTA clears the key: a block is used at most once.
__host__ __device__ inline unsigned long long bpp_prep_key(int order, int mode, int R) {
  return (0x4250ull << 48) | (unsigned long long)(order + 1) << 32 | (unsigned long long)(mode + 1) << 16 |
         (unsigned long long)R;
}
__host__ __device__ inline int64_t bpp_prep_offset(int64_t rows) { return (rows + 1) / 2 * 2; }
inline size_t bpp_prep_words(int rank) { return 4 + 2 * size_t(rank) * rank; }

template <int RP>
__global__ void __launch_bounds__(bpp_warps<RP>() * 32)
    bpp_prepare_kernel(const double* __restrict__ grams, int order, int mode, int R, double* __restrict__ blk) {
  extern __shared__ __align__(16) double dsm[];
  double* S = dsm;                 // RP*RP (S^T, as bpp_kernel holds it)
  double* TT = S + RP * RP;        // RP*RP
  double* gj = TT + RP * RP;       // 6 RP
  double* aug = gj + 6 * RP;       // RP * 2 RP
  load_hadamard<true>(S, grams, order, mode, R);
  __syncthreads();
  const bool t_ok = block_inverse<RP>(S, R, aug, TT, gj);   // bpp_kernel's own elimination: the same bits
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    blk[4 + e] = S[e];
    blk[4 + R * R + e] = TT[e];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    reinterpret_cast<unsigned long long*>(blk)[1] = t_ok ? 1ull : 0ull;
    reinterpret_cast<unsigned long long*>(blk)[0] = bpp_prep_key(order, mode, R);
  }
}

template <int RP>
__global__ void __launch_bounds__(bpp_warps<RP>() * 32)
    bpp_kernel(const double* __restrict__ grams, int order, int mode, int R, const double* __restrict__ mrows,
               int64_t rows, double* __restrict__ hhat, double* __restrict__ part, double* nsq, double* beta,
               int* status, unsigned int* ticket, unsigned long long* __restrict__ psets, int64_t mld,
               TailArgs tail) {
  extern __shared__ __align__(16) double dsm[];
  constexpr int LP = RP + 1;  // LU pitch (augmented column at index p)
  constexpr int NH = (RP + 31) / 32;  // entries per lane
  constexpr int NW = bpp_warps<RP>();
  double* S = dsm;                                    // RP*RP (holds S^T)
  double* TT = S + RP * RP;                           // RP*RP (T^T, T = S^-1)
  double* red = TT + RP * RP;                         // NW * 64
  double* colbuf = red + NW * 64;                     // RP + 1
  double* zall = colbuf + RP + 1;                     // NW * RP
  double* gj = zall + NW * RP;                        // 6 * RP (Gauss-Jordan row / column buffers)
  double* fall = gj + 6 * RP;                         // NW * RP (each warp's right-hand side f)
  double* lu = fall + NW * RP;                        // NW * RP * LP (the inverse's work space at the start)
  int* pidx_all = reinterpret_cast<int*>(lu + size_t(NW) * RP * LP);   // NW * 64
  int* qidx_all = pidx_all + NW * 64;                                  // NW * 64
#ifdef NNCP_BPP_TIMING
  const long long tk0 = clock64();
#endif
  // S and S^-1 prepared ahead (nncp_bpp_prepare), else formed here
  unsigned long long* prep = psets != nullptr && order > 0 ? psets + bpp_prep_offset(rows) : nullptr;
  const bool use_prep = prep != nullptr && prep[0] == bpp_prep_key(order, mode, R);
  bool t_ok;
  if (use_prep) {
    const double* blk = reinterpret_cast<const double*>(prep);
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      S[e] = blk[4 + e];
      TT[e] = blk[4 + R * R + e];
    }
    t_ok = prep[1] != 0ull;
    __syncthreads();
  }
#ifdef NNCP_BPP_TIMING
  const long long tk1 = clock64();
#endif
  if (!use_prep) {
    load_hadamard<true>(S, grams, order, mode, R);   // S^T: the gathers below walk columns across lanes
    __syncthreads();
    // the block-elimination passes need S^-1; order 0 (an explicit S from bpp_update)
    // need not be symmetric: solve those directly, like the reference
    t_ok = order > 0 && block_inverse<RP>(S, R, lu, TT, gj);
  }
#ifdef NNCP_BPP_TIMING
  const long long tk2 = clock64();
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = lu + size_t(warp) * RP * LP;
  int* pidx = pidx_all + warp * 64;   // pidx[a] = index of the a-th passive variable
  int* qidx = qidx_all + warp * 64;   // qidx[a] = index of the a-th active variable
  double* zbuf = zall + warp * RP;
  double* fbuf = fall + warp * RP;
  double xs[NH], ys[NH], fs[NH];
  double sq2[NH];
#pragma unroll
  for (int q = 0; q < NH; ++q) sq2[q] = 0.0;
  double bsum = 0.0;

  // rows spread evenly over the CTAs (one or two per warp up to ~2400 rows): the kernel's
  // latency is the per-CTA S^-1 plus one row's passes, so more CTAs, not more rows per CTA
  const int64_t rpc = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t row_lo = int64_t(blockIdx.x) * rpc, row_hi = min(rows, row_lo + rpc);
  for (int64_t i = row_lo + warp; i < row_hi; i += NW) {
    // f = this row of M: row-major, or (mld > 0) the dimension tree's column-major temporary
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int r = lane + 32 * q;
      fs[q] = (r < R) ? load_m(mrows, mld, i, r, R, tail) : 0.0;
      xs[q] = 0.0;
      ys[q] = -fs[q];
      if (r < R) fbuf[r] = fs[q];
    }
    __syncwarp();
    const double* fr = fbuf;
    // warm start (psets): the passive set this row ended with in the previous outer
    // iteration.  The first pass then only evaluates it; the exchange rules below are
    // the reference's from there on (the NNLS minimiser is unique for SPD S).  A row
    // whose fast attempt (warm start and/or block-elimination passes) fails is redone
    // exactly as the reference does it: cold start, direct solves -- so failures
    // (BppCyclingError, singular solves) are the reference's.
    const unsigned long long warm_set = psets ? psets[i] & (R < 64 ? ((1ull << R) - 1ull) : ~0ull) : 0ull;
    unsigned long long P = 0ull;
    bool done = false;
    int fail_kind = 0;
    for (int attempt = (warm_set != 0ull || t_ok) ? 0 : 1; attempt < 2 && !done; ++attempt) {
      const bool fast = attempt == 0;
      P = fast ? warm_set : 0ull;
#pragma unroll
      for (int q = 0; q < NH; ++q) {
        xs[q] = 0.0;
        ys[q] = -fs[q];
      }
      bool pending = P != 0ull;       // x, y of P not evaluated yet
      bool direct_only = !(fast && t_ok);
      int best = R + 1, backup = 3;
      fail_kind = 0;
      for (int it = 0; it < 5 * R + 1; ++it) {
        if (!pending) {
          unsigned long long viol = 0ull;
#pragma unroll
          for (int q = 0; q < NH; ++q) {
            const int r = lane + 32 * q;
            const bool pr = (P >> r) & 1ull;
            const bool v = (r < R) && ((pr && xs[q] < 0.0) || (!pr && ys[q] < 0.0));
            viol |= (unsigned long long)__ballot_sync(0xffffffffu, v) << (32 * q);
          }
          const int k = __popcll(viol);
          if (k == 0) {
            done = true;
            break;
          }
          if (k < best) {
            best = k;
            backup = 3;
            P ^= viol;
          } else if (backup > 0) {
            --backup;
            P ^= viol;
          } else {
            P ^= 1ull << (63 - __clzll(viol));
          }
        }
        pending = false;
        // ---- x_P for the new passive set (updaters.py:152), y = S[~P,P] x_P - f[~P].
        // Few active variables: block elimination through S^-1 (a q x q solve); many:
        // the reference's direct solve of S[P,P] (a p x p solve).  Same minimiser.
        const int p = __popcll(P);
        if (!direct_only && 2 * p > R) {
          if (bpp_schur<RP>(TT, R, P, A, qidx, zbuf, fs, xs)) {
            bpp_dual<RP>(S, R, P, xs, fs, ys);
            continue;
          }
          direct_only = true;     // T[Q,Q] not positive definite: this row continues directly
        }
        if (!bpp_eval_direct<RP>(S, R, fr, P, A, pidx, fs, xs, ys)) {
          fail_kind = 2;
          break;
        }
      }
    }
    if (!done && fail_kind == 0) fail_kind = 1;
    if (fail_kind) {
      if (lane == 0) {
        atomicMin(status + 2, int(i));
        atomicMax(status + 3, fail_kind);
      }
    }
    if (psets && lane == 0) psets[i] = fail_kind ? 0ull : P;
    double* hr = hhat + i * R;
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const int r = lane + 32 * q;
      if (r < R) {
        hr[r] = xs[q];
        if (beta) bsum = fma(fs[q], xs[q], bsum);
      }
    }
#pragma unroll
    for (int q = 0; q < NH; ++q) sq2[q] = fma(xs[q], xs[q], sq2[q]);
  }
#ifdef NNCP_BPP_TIMING
  const long long tk3 = clock64();
#endif
  __syncthreads();
  tail.scratch = lu;   // the per-warp scratch is dead after the rows
  colsum_epilogue<NH>(sq2, bsum, R, red, colbuf, part, nsq, beta, ticket, &tail, use_prep ? prep : nullptr);
#ifdef NNCP_BPP_TIMING
  if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("bpp cta %d warp %d t_ok %d: hadamard %lld inverse %lld rows %lld epilogue %lld\n", blockIdx.x,
           warp, int(t_ok), tk1 - tk0, tk2 - tk1, tk3 - tk2, clock64() - tk3);
#endif
}

// --------------------------------------------------- normalise + Gram ------
constexpr int kGramRows = 64;
template <int RP>
constexpr int gram_rows() {   // rows per normalise+Gram CTA
  return RP <= 32 ? 128 : kGramRows;
}

template <int RP>
__global__ void __launch_bounds__(256)
    normalize_gram_kernel(const double* __restrict__ hhat, const double* __restrict__ nsq, int64_t rows, int R,
                          double* __restrict__ owned, double* __restrict__ lam, double* __restrict__ gram,
                          double* __restrict__ part, unsigned int* ticket, const PublishArgs pub) {
  // rows per CTA: 128 up to R = 32 (half the per-CTA Gram partials the last CTA sums)
  constexpr int GR = gram_rows<RP>();
  __shared__ __align__(16) double tile[GR * RP];
  __shared__ double scale[RP];
  __shared__ double rscale[RP];
#ifdef NNCP_UPD_TIMING
  const long long tn0 = clock64();
#endif
  if (threadIdx.x < R) {
    double s = 1.0;
    if (nsq) {
      const double w = sqrt(nsq[threadIdx.x]);
      s = (w > 0.0) ? w : 1.0;
      if (blockIdx.x == 0 && lam) lam[threadIdx.x] = w;
    }
    scale[threadIdx.x] = s;
    rscale[threadIdx.x] = 1.0 / s;
  }
  __syncthreads();
#ifdef NNCP_UPD_TIMING
  const long long tn1 = clock64();
#endif
  // the launch picks the CTA count (<= GR rows each): few rows -> more, shorter CTAs
  const int64_t grk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = int64_t(blockIdx.x) * grk;
  const int nr = int(rows - r0 < grk ? rows - r0 : grk);   // <= 0: an empty CTA (zero partial)
  // every load of the tile issued before the first use (a load-use loop serialised
  // PER global-memory latencies; this kernel is latency-bound at these sizes)
  constexpr int PER = (GR * RP + 255) / 256;
  double v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = int(threadIdx.x) + 256 * k, il = e / RP, r = e % RP;
    v[k] = (il < nr && r < R) ? hhat[(r0 + il) * R + r] : 0.0;
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = int(threadIdx.x) + 256 * k, il = e / RP, r = e % RP;
    if (il < nr) {
      double x = v[k];   // 0 in the padding columns r >= R
      if (nsq && r < R) {
        // x / w (driver.py:416-418) as the product with the column's reciprocal plus one
        // FMA residual correction: the correctly rounded quotient bar rare ties, without
        // a full division per element (the divisions were most of this kernel's row phase)
        const double w = scale[r], iw = rscale[r];
        const double q0 = x * iw;
        x = fma(fma(-q0, w, x), iw, q0);
        owned[(r0 + il) * R + r] = x;
      }
      tile[il * RP + r] = x;
    }
  }
  __syncthreads();
#ifdef NNCP_UPD_TIMING
  const long long tn2 = clock64();
#endif
  if (gram == nullptr) return;  // row scaling only
  const int RR = R * R;
  double* mypart = part + size_t(blockIdx.x) * RR;
  // 2 x 2 register blocks of G: per row one 16-byte load of the block's two a-values and
  // one of its two b-values feed four FMA chains (one entry per chain read two 8-byte
  // words per FMA: shared-memory bound); every entry still sums its rows in order
  constexpr int NB2 = RP / 2;
  for (int blk = threadIdx.x; blk < NB2 * NB2; blk += blockDim.x) {
    const int a0 = 2 * (blk / NB2), b0 = 2 * (blk % NB2);
    if (a0 >= R || b0 >= R) continue;
    double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;
#pragma unroll 8
    for (int il = 0; il < nr; ++il) {
      const double2 xa = *reinterpret_cast<const double2*>(tile + il * RP + a0);
      const double2 xb = *reinterpret_cast<const double2*>(tile + il * RP + b0);
      s00 = fma(xa.x, xb.x, s00);
      s01 = fma(xa.x, xb.y, s01);
      s10 = fma(xa.y, xb.x, s10);
      s11 = fma(xa.y, xb.y, s11);
    }
    mypart[a0 * R + b0] = s00;
    if (b0 + 1 < R) mypart[a0 * R + b0 + 1] = s01;
    if (a0 + 1 < R) {
      mypart[(a0 + 1) * R + b0] = s10;
      if (b0 + 1 < R) mypart[(a0 + 1) * R + b0 + 1] = s11;
    }
  }
#ifdef NNCP_UPD_TIMING
  const long long tn3 = clock64();
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("normalize cta %d/%d: scale %lld rows %lld gram %lld\n", blockIdx.x, gridDim.x, tn1 - tn0, tn2 - tn1,
           tn3 - tn2);
#endif
  if (last_cta_ticket(ticket)) {
#ifdef NNCP_UPD_TIMING
    const long long tn4 = clock64();
#endif
    finish_partials<8>(part, gridDim.x, RR, gram);
#ifdef NNCP_UPD_TIMING
    if (threadIdx.x == 0) printf("normalize last cta %d: ticket %lld finish %lld\n", blockIdx.x, tn4 - tn3, clock64() - tn4);
#endif
    if (pub.gamma != nullptr) {
      // the sweep's last normalisation also produces gamma and hands the status off
      // (a single context: no All-Reduce of the Gram in between) -- one launch fewer
      __threadfence();
      __syncthreads();
      gamma_publish_body(pub, R, tile, scale);
    }
  }
}

// Normalisation from the All-Reduced Gram of the UNnormalised rows (the grid path's
// merged collective): nsq = diag(G^), w = sqrt(nsq) (driver.py:411-418),
// H = H^ / (w > 0 ? w : 1), lam = w, and the Gram of the normalised factor
// G = sym(G^) / (w' w'^T) (driver.py:419-422) without a second pass over the rows.
__global__ void __launch_bounds__(256)
    normalize_from_gram_kernel(const double* __restrict__ hhat, const double* __restrict__ graw, int64_t rows,
                               int R, double* __restrict__ owned, double* __restrict__ lam,
                               double* __restrict__ gram) {
  __shared__ double scale[kMaxRank];
  if (threadIdx.x < R) {
    const double w = sqrt(graw[threadIdx.x * R + threadIdx.x]);
    scale[threadIdx.x] = (w > 0.0) ? w : 1.0;
    if (blockIdx.x == 0 && lam) lam[threadIdx.x] = w;
  }
  __syncthreads();
  const int64_t n = rows * R;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x)
    owned[e] = hhat[e] / scale[int(e % R)];
  if (blockIdx.x == 0 && gram) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int a = e / R, b = e - (e / R) * R;
      gram[e] = 0.5 * (graw[a * R + b] + graw[b * R + a]) / (scale[a] * scale[b]);
    }
  }
}

__global__ void __launch_bounds__(256) gamma_kernel(const PublishArgs a, int R) {
  __shared__ double W[kMaxRank * kMaxRank];
  __shared__ double v[kMaxRank];
  gamma_publish_body(a, R, W, v);
}

__global__ void __launch_bounds__(256)
    inner_kernel(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ lam,
                 int64_t rows, int R, double* __restrict__ part, double* out, unsigned int* ticket) {
  __shared__ double red[8];
  const int64_t n = rows * R;
  double s = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    double bv = b[e];
    if (lam) bv = bv * lam[e % R];
    s = fma(a[e], bv, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (last_cta_ticket(ticket)) finish_partials(part, gridDim.x, 1, out);
}

// out[0] = sum x^2 (fixed-order reduction); with out_min, in the same pass:
// out_min[0] = min x (the reference's negative-entry warning, driver.py:571-573),
// out_min[1] = max |x| and out_min[2] = min over the nonzero |x| (INFINITY if none):
// the dynamic range the sliced MTTKRP engine's "auto" choice checks.
__device__ __forceinline__ void minmax_acc(double v, double& mn, double& amax, double& anz) {
  const double a = fabs(v);
  mn = fmin(mn, v);
  amax = fmax(amax, a);
  anz = fmin(anz, a > 0.0 ? a : INFINITY);
}

__global__ void __launch_bounds__(512)
    norm_sq_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part, double* out,
                   double* out_min, unsigned int* ticket) {
  __shared__ double red[16];
  __shared__ double redm[3][16];
  double s0 = 0.0, s1 = 0.0, mn = INFINITY, amax = 0.0, anz = INFINITY;
  const int64_t n2 = n / 2;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  bool nonfinite = false;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n2; e += int64_t(gridDim.x) * blockDim.x) {
    const double2 v = __ldcs(x2 + e);
    s0 = fma(v.x, v.x, s0);
    s1 = fma(v.y, v.y, s1);
    if (out_min != nullptr) {
      minmax_acc(v.x, mn, amax, anz);
      minmax_acc(v.y, mn, amax, anz);
      nonfinite |= !isfinite(v.x) || !isfinite(v.y);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    s0 = fma(x[n - 1], x[n - 1], s0);
    minmax_acc(x[n - 1], mn, amax, anz);
    nonfinite |= !isfinite(x[n - 1]);
  }
  // fmin/fmax drop NaN: a non-finite entry poisons the max so callers can see it
  if (nonfinite) amax = NAN;
  const double s = block_sum(s0 + s1, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (out_min != nullptr) {
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
      double m = redm[0][0], a = redm[1][0], z = redm[2][0];
      bool nan = isnan(a);
      for (int w = 1; w < int(blockDim.x >> 5); ++w) {
        m = fmin(m, redm[0][w]);
        nan |= isnan(redm[1][w]);
        a = fmax(a, redm[1][w]);
        z = fmin(z, redm[2][w]);
      }
      part[gridDim.x + blockIdx.x] = m;
      part[2 * gridDim.x + blockIdx.x] = nan ? NAN : a;
      part[3 * gridDim.x + blockIdx.x] = z;
    }
  }
  if (last_cta_ticket(ticket)) {
    finish_partials(part, gridDim.x, 1, out);
    if (out_min != nullptr && threadIdx.x == 0) {
      double m = part[gridDim.x], a = part[2 * gridDim.x], z = part[3 * gridDim.x];
      bool nan = isnan(a);
      for (int b = 1; b < int(gridDim.x); ++b) {
        m = fmin(m, part[gridDim.x + b]);
        nan |= isnan(part[2 * gridDim.x + b]);
        a = fmax(a, part[2 * gridDim.x + b]);
        z = fmin(z, part[3 * gridDim.x + b]);
      }
      out_min[0] = m;
      out_min[1] = nan ? NAN : a;
      out_min[2] = z;
    }
  }
}

__global__ void status_reset_kernel(int* status, int count) {
  for (int b = threadIdx.x; b < count; b += blockDim.x) {
    int* s = status + b * NNCP_STATUS_WORDS;
    s[0] = 0;
    s[1] = 0;
    s[2] = INT_MAX;
    s[3] = 0;
  }
}

// ------------------------------------------------------------- host side ---
#define NNCP_RP_CASES(RPV, ...)            \
  switch (RPV) {                            \
    case 8: { constexpr int RP = 8; __VA_ARGS__; } break;   \
    case 16: { constexpr int RP = 16; __VA_ARGS__; } break; \
    case 24: { constexpr int RP = 24; __VA_ARGS__; } break; \
    case 32: { constexpr int RP = 32; __VA_ARGS__; } break; \
    case 40: { constexpr int RP = 40; __VA_ARGS__; } break; \
    case 48: { constexpr int RP = 48; __VA_ARGS__; } break; \
    case 56: { constexpr int RP = 56; __VA_ARGS__; } break; \
    case 64: { constexpr int RP = 64; __VA_ARGS__; } break; \
    default: return fail(NNCP_ERR_UNSUPPORTED, "rank above NNCP_MAX_RANK"); \
  }

int row_blocks(int64_t rows) {
  return int(std::max<int64_t>(1, std::min<int64_t>((rows + kRowWarps - 1) / kRowWarps, int64_t(num_sms()) * 4)));
}

size_t row_update_part_elems(int64_t rows, int rank) {
  const int64_t blocks_rows = row_blocks(rows);
  const int64_t blocks_bpp = std::min<int64_t>((rows + kBppWarps - 1) / kBppWarps, int64_t(num_sms()) * 4);
  const int64_t blocks_gram = (rows + 31) / 32;   // normalise+Gram: >= 32 rows per CTA
  size_t e = std::max<int64_t>(blocks_rows, blocks_bpp) * (rank + 6);  // + ADMM/NES step partials
  e = std::max<size_t>(e, size_t(std::max<int64_t>(blocks_gram, 1)) * rank * rank);
  e = std::max<size_t>(e, size_t(num_sms()) * 8 * 4);   // norm_squared(_min): <= 8 blocks/SM, sum + 3 extrema
  return e;
}

int update(int algo, const double* grams, int order, int mode, int rank, const double* mrows, const double* owned,
           const double* lam, int64_t rows, double* hhat, double* nsq, double* beta, int* status, void* ws,
           size_t ws_bytes, cudaStream_t st, double mu_eps, void* bpp_sets, int64_t mld, const TailArgs* tail) {
  const TailArgs tl = tail ? *tail : TailArgs{};
  if (rows <= 0) {
    // an empty row block still owes its (zero) column sums
    if (nsq) NNCP_CUDA_TRY(cudaMemsetAsync(nsq, 0, sizeof(double) * rank, st));
    if (beta) NNCP_CUDA_TRY(cudaMemsetAsync(beta, 0, sizeof(double), st));
    return NNCP_OK;
  }
  WsLayout w = ws_layout(ws, ws_bytes);
  const int rp = pad8(rank);
  (void)rp;
  if (tl.mgroups > 1) {
    // group partials may live in the same workspace (the sliced MTTKRP's): they must not
    // meet the tickets and per-CTA partials this launch writes
    const char* m0 = reinterpret_cast<const char*>(mrows);
    const char* m1 = m0 + sizeof(double) * size_t(tl.mgroups) * size_t(tl.mgstride);
    const char* w0 = static_cast<const char*>(ws);
    const char* w1 = reinterpret_cast<const char*>(w.part + size_t(std::max<int64_t>(row_blocks(rows), num_sms())) *
                                                   (rank + 1));
    if (m0 < w1 && w0 < m1) return fail(NNCP_ERR_VALUE, "group partials overlap the update's workspace");
    if (mld < rows || tl.mgstride < mld * rank) return fail(NNCP_ERR_VALUE, "bad group partial layout");
  }
  if (algo == NNCP_ALGO_MU || algo == NNCP_ALGO_HALS) {
    const int blocks = row_blocks(rows);
    if (w.part_elems < size_t(blocks) * (rank + 1)) return fail(NNCP_ERR_VALUE, "workspace too small (update)");
    const int rp32 = rank <= 16 ? 16 : rank <= 32 ? 32 : 64;   // unrolled column loops
    auto launch = [&](auto kern) {
      kern<<<blocks, kRowWarps * 32, 0, st>>>(grams, order, mode, rank, mrows, owned, lam, rows, hhat, w.part, nsq,
                                              beta, status, w.tickets + T_UPDATE, mu_eps, mld, tl);
    };
    if (algo == NNCP_ALGO_MU) {
      if (rp32 == 16) launch(update_rows_kernel<NNCP_ALGO_MU, 16>);
      else if (rp32 == 32) launch(update_rows_kernel<NNCP_ALGO_MU, 32>);
      else launch(update_rows_kernel<NNCP_ALGO_MU, 64>);
    } else {
      if (rp32 == 16) launch(update_rows_kernel<NNCP_ALGO_HALS, 16>);
      else if (rp32 == 32) launch(update_rows_kernel<NNCP_ALGO_HALS, 32>);
      else launch(update_rows_kernel<NNCP_ALGO_HALS, 64>);
    }
  } else if (algo == NNCP_ALGO_BPP) {
    NNCP_RP_CASES(rp, {
      constexpr int NW = bpp_warps<RP>();
      const int blocks = int(std::min<int64_t>(rows, int64_t(num_sms())));
      if (w.part_elems < size_t(blocks) * (rank + 1)) return fail(NNCP_ERR_VALUE, "workspace too small (bpp)");
      const size_t smem = sizeof(double) * (2 * size_t(RP) * RP + NW * 64 + RP + 1 + 2 * NW * RP + 6 * RP +
                                            size_t(NW) * RP * (RP + 1)) +
                          sizeof(int) * NW * 128;
      if (int rc = set_max_smem_once<bpp_kernel<RP>>(int(smem))) return rc;
      bpp_kernel<RP><<<blocks, NW * 32, smem, st>>>(grams, order, mode, rank, mrows, rows, hhat, w.part, nsq,
                                                           beta, status, w.tickets + T_UPDATE,
                                                           static_cast<unsigned long long*>(bpp_sets), mld, tl);
    });
  } else {
    return fail(NNCP_ERR_VALUE, "algorithm must be MU, HALS or BPP");
  }
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

size_t bpp_sets_words(int64_t rows, int rank) {
  return size_t(bpp_prep_offset(std::max<int64_t>(rows, 0))) + bpp_prep_words(rank);
}

int bpp_prepare(const double* grams, int order, int mode, int rank, void* sets, int64_t rows, cudaStream_t st) {
  if (order < 1) return fail(NNCP_ERR_VALUE, "bpp_prepare needs the Grams of an order >= 1 tensor");
  if (sets == nullptr) return fail(NNCP_ERR_VALUE, "bpp_prepare needs the passive-set buffer");
  double* blk = reinterpret_cast<double*>(static_cast<unsigned long long*>(sets) + bpp_prep_offset(rows));
  const int rp = pad8(rank);
  NNCP_RP_CASES(rp, {
    constexpr int NW = bpp_warps<RP>();
    const size_t smem = sizeof(double) * (4 * size_t(RP) * RP + 6 * RP);
    if (int rc = set_max_smem_once<bpp_prepare_kernel<RP>>(int(smem))) return rc;
    bpp_prepare_kernel<RP><<<1, NW * 32, smem, st>>>(grams, order, mode, rank, blk);
  });
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

static int normalize_gram_impl(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned, double* lam,
                   double* gram, void* ws, size_t ws_bytes, cudaStream_t st, int ticket_slot,
                   const PublishArgs* pub) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int rp = pad8(rank);
  // rows per CTA: 32 up to 512 rows, 64 up to 1024, then the kernel's maximum (measured:
  // the Gram chain and the partial count trade off)
  NNCP_RP_CASES(rp, const int64_t gr = std::min<int64_t>(gram_rows<RP>(), rows <= 512 ? 32 : rows <= 1024 ? 64 : 128);
                const int blocks = int(std::max<int64_t>(1, (rows + gr - 1) / gr));
                if (gram && w.part_elems < size_t(blocks) * rank * rank)
                  return fail(NNCP_ERR_VALUE, "workspace too small (gram)");
                (normalize_gram_kernel<RP><<<blocks, 256, 0, st>>>(hhat, nsq, std::max<int64_t>(rows, 0), rank,
                                                                      owned, lam, gram, w.part,
                                                                      w.tickets + ticket_slot,
                                                                      pub ? *pub : PublishArgs{})));
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int normalize_gram(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned, double* lam,
                   double* gram, void* ws, size_t ws_bytes, cudaStream_t st, int ticket_slot) {
  return normalize_gram_impl(hhat, nsq, rows, rank, owned, lam, gram, ws, ws_bytes, st, ticket_slot, nullptr);
}

int normalize_from_gram(const double* hhat, const double* graw, int64_t rows, int rank, double* owned, double* lam,
                        double* gram, cudaStream_t st) {
  const int64_t n = std::max<int64_t>(rows, 0) * rank;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 4)));
  normalize_from_gram_kernel<<<blocks, 256, 0, st>>>(hhat, graw, std::max<int64_t>(rows, 0), rank, owned, lam, gram);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int gamma(const double* grams, int order, int rank, const double* lam, double* out, cudaStream_t st) {
  PublishArgs a{grams, order, lam, out, nullptr, 0, nullptr, 0, 0, nullptr};
  gamma_kernel<<<1, 256, 0, st>>>(a, rank);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int normalize_gram_publish(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned, double* lam,
                           double* gram, void* ws, size_t ws_bytes, const double* grams, int order, double* gamma_out,
                           int* status, int count, double* codes, int nslots, int offset, int* masks,
                           cudaStream_t st) {
  PublishArgs a{grams, order, lam, gamma_out, status, count, codes, nslots, offset, masks};
  return normalize_gram_impl(hhat, nsq, rows, rank, owned, lam, gram, ws, ws_bytes, st, 2, &a);
}

int gamma_publish(const double* grams, int order, int rank, const double* lam, double* out, int* status, int count,
                  double* codes, int nslots, int offset, int* masks, cudaStream_t st) {
  PublishArgs a{grams, order, lam, out, status, count, codes, nslots, offset, masks};
  gamma_kernel<<<1, 256, 0, st>>>(a, rank);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int inner(const double* a, const double* b, const double* lam, int64_t rows, int rank, double* out, void* ws,
          size_t ws_bytes, cudaStream_t st) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int64_t n = rows * rank;
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 4)));
  if (w.part_elems < size_t(blocks)) return fail(NNCP_ERR_VALUE, "workspace too small (inner)");
  inner_kernel<<<blocks, 256, 0, st>>>(a, b, lam, rows, rank, w.part, out, w.tickets + T_INNER);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int norm_squared(const double* x, int64_t n, double* out, double* out_min, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  WsLayout w = ws_layout(ws, ws_bytes);
  const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((n / 2 + 511) / 512, int64_t(num_sms()) * 8)));
  if (w.part_elems < size_t(blocks) * (out_min ? 4 : 1)) return fail(NNCP_ERR_VALUE, "workspace too small (norm)");
  if (reinterpret_cast<uintptr_t>(x) % 16) return fail(NNCP_ERR_VALUE, "tensor must be 16-byte aligned");
  if (out_min != nullptr && n < 1) return fail(NNCP_ERR_VALUE, "min of an empty tensor");
  norm_sq_kernel<<<blocks, 512, 0, st>>>(x, n, w.part, out, out_min, w.tickets + T_NORM);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

int status_reset(int* status, int count, cudaStream_t st) {
  status_reset_kernel<<<1, 32, 0, st>>>(status, count);
  NNCP_LAUNCH_CHECK();
  return NNCP_OK;
}

}  // namespace nncp
