// Device helpers shared by the NNLS-side translation units (nnls.cu, nnls_iter.cu).
#pragma once

#include "common.cuh"

namespace nncp {

// --------------------------------------------------------------- helpers --
// S[a][b] = prod_{m != mode} 0.5 (G_m[a][b] + G_m[b][a]); order==0: S = grams.
// TRANSPOSED: store S^T instead (identical for order > 0, where S is symmetric bit
// for bit), so kernels that walk a column of S across lanes read a row instead:
// lane-consecutive addresses, no 32-way shared-memory bank conflict at R = 32.
template <bool TRANSPOSED = false>
static __device__ void load_hadamard(double* S, const double* __restrict__ grams, int order, int mode, int R) {
  // Latency-bound prologue of every update kernel.  Each thread takes up to EPT
  // elements at a time and walks the Grams in ascending order with the NEXT Gram's
  // entries already in flight, so a 3-way mode costs one L2 round trip per EPT
  // elements (the element-at-a-time loop cost one per element: 4 at R = 32, ~8k
  // cycles, measured).  Products in ascending m, as before: the same bits.
  constexpr int EPT = 4;
  const int RR = R * R, T = int(blockDim.x);
  if (order == 0) {
    for (int e = threadIdx.x; e < RR; e += T) {
      const int a = e / R, b = e - (e / R) * R;
      S[TRANSPOSED ? b * R + a : e] = grams[e];
    }
    return;
  }
  int m0 = 0;
  while (m0 < order && m0 == mode) ++m0;
  for (int e0 = threadIdx.x; e0 < RR; e0 += EPT * T) {
    int pa[EPT], pb[EPT];
    double acc[EPT], x[EPT], y[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = min(e0 + k * T, RR - 1);
      const int a = e / R, b = e - (e / R) * R;
      pa[k] = a * R + b;
      pb[k] = b * R + a;
      acc[k] = 1.0;
    }
    int m = m0;
    if (m < order) {
      const double* g = grams + size_t(m) * RR;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        x[k] = __ldg(g + pa[k]);
        y[k] = __ldg(g + pb[k]);
      }
    }
    while (m < order) {
      int mn = m + 1;
      if (mn == mode) ++mn;
      double xn[EPT], yn[EPT];
      if (mn < order) {
        const double* g = grams + size_t(mn) * RR;
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          xn[k] = __ldg(g + pa[k]);
          yn[k] = __ldg(g + pb[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k) acc[k] *= 0.5 * (x[k] + y[k]);
      if (mn >= order) break;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        x[k] = xn[k];
        y[k] = yn[k];
      }
      m = mn;
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int e = e0 + k * T;
      if (e < RR) S[TRANSPOSED ? pb[k] : pa[k]] = acc[k];
    }
  }
}

static __device__ double block_sum(double v, double* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    s = red[0];
    for (int w = 1; w < nw; ++w) s += red[w];
  }
  __syncthreads();
  return s;
}

// Final fixed-order reduction of per-CTA partials [nblk][n] -> out[n], run by the
// last CTA.  Latency-bound if done naively (one thread walking nblk partials), so
// the loads are issued in independent batches: with n <= blockDim.x each output
// is split into `segs` strided segments with eight accumulators, then the segments
// are summed in order; otherwise a thread owns four outputs and issues 4 x 4 loads
// per step.  Deterministic for a given launch configuration.
// DEPTH: partial blocks in flight per entry when n exceeds the block size (the Gram's
// R x R entries): each round is one L2 round trip for the last CTA.
template <int DEPTH = 4>
static __device__ void finish_partials(const double* part, int nblk, int n, double* out) {
  __shared__ double seg_sum[1024];
  const int T = blockDim.x;
  int segs = T / max(n, 1);
  segs = max(1, min(segs, min(32, nblk)));
  if (n * segs <= T) {
    const int t = threadIdx.x;
    if (t < n * segs) {
      const int e = t % n, sg = t / n;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = 0.0;
      int b = sg;
      for (; b + 7 * segs < nblk; b += 8 * segs) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = part[size_t(b + q * segs) * n + e];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] += v[q];
      }
      for (; b < nblk; b += segs) a[0] += part[size_t(b) * n + e];
      seg_sum[sg * n + e] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += T) {
      double s = seg_sum[e];
      for (int sg = 1; sg < segs; ++sg) s += seg_sum[sg * n + e];
      out[e] = s;
    }
  } else {
    for (int e0 = threadIdx.x; e0 < n; e0 += 4 * T) {
      double a[4][DEPTH];
#pragma unroll
      for (int o = 0; o < 4; ++o)
#pragma unroll
        for (int q = 0; q < DEPTH; ++q) a[o][q] = 0.0;
      for (int b = 0; b < nblk; b += DEPTH) {
        double v[4][DEPTH];
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
          for (int q = 0; q < DEPTH; ++q) {
            const int e = e0 + o * T;
            v[o][q] = (e < n && b + q < nblk) ? part[size_t(b + q) * n + e] : 0.0;
          }
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
          for (int q = 0; q < DEPTH; ++q) a[o][q] += v[o][q];
      }
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        // pairwise, fixed order
#pragma unroll
        for (int w = 1; w < DEPTH; w *= 2)
#pragma unroll
          for (int q = 0; q + w < DEPTH; q += 2 * w) a[o][q] += a[o][q + w];
        if (e0 + o * T < n) out[e0 + o * T] = a[o][0];
      }
    }
  }
}

// Workspace carve-up (bytes): [0,256) tickets, then partial buffers.
struct WsLayout {
  unsigned int* tickets;
  double* part;
  size_t part_elems;
};
inline WsLayout ws_layout(void* ws, size_t bytes) {
  WsLayout w;
  w.tickets = static_cast<unsigned int*>(ws);
  w.part = reinterpret_cast<double*>(static_cast<char*>(ws) + 256);
  w.part_elems = bytes > 256 ? (bytes - 256) / sizeof(double) : 0;
  return w;
}
enum Ticket { T_NORM = 0, T_UPDATE = 1, T_NORMGRAM = 2, T_GRAM = 3, T_INNER = 4, T_ITER = 5, T_COLSQ = 6 };

// ------------------------------------------------------------- scalars -----
// End-of-sweep scalars: gamma = lam^T (prod_m sym(G_m)) lam (driver.py:431), and the
// status hand-off.  codes[0..nslots) is the rank-slotted vector that one SUM
// All-Reduce combines: every slot is zeroed, then this rank's slot [offset, offset +
// count) gets, per mode, failure kind * 2^32 + failing row (0 = none; exact in fp64);
// masks[2n..2n+1] = the warning bits; the status words are reset for the next sweep
// (the reset the caller would otherwise launch separately).  Block-cooperative;
// W (R*R) and v (R) are shared-memory scratch.
struct PublishArgs {
  const double* grams;
  int order;
  const double* lam;
  double* gamma;
  int* status;
  int count;
  double* codes;
  int nslots;
  int offset;
  int* masks;
};

static __device__ void gamma_publish_body(const PublishArgs& a, int R, double* W, double* v) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e / R, c = e - (e / R) * R;
    double p = 1.0;
    for (int m = 0; m < a.order; ++m) {
      const double* g = a.grams + size_t(m) * R * R;
      const double sym = 0.5 * (g[r * R + c] + g[c * R + r]);
      p = (m == 0) ? sym : p * sym;
    }
    W[e] = p * a.lam[c];
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double s = 0.0;
    for (int c = 0; c < R; ++c) s += W[threadIdx.x * R + c];
    v[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < R; ++k) s = fma(a.lam[k], v[k], s);
    a.gamma[0] = s;
  }
  if (a.status == nullptr) return;
  for (int e = threadIdx.x; e < a.nslots; e += blockDim.x) a.codes[e] = 0.0;
  __syncthreads();
  if (int(threadIdx.x) < a.count) {
    int* st = a.status + threadIdx.x * NNCP_STATUS_WORDS;
    const int kind = st[3], row = st[2];
    a.codes[a.offset + threadIdx.x] = kind ? double(kind) * 4294967296.0 + double(row) : 0.0;
    if (a.masks != nullptr) {
      a.masks[2 * threadIdx.x] = st[0];
      a.masks[2 * threadIdx.x + 1] = st[1];
    }
    st[0] = 0;
    st[1] = 0;
    st[2] = INT_MAX;
    st[3] = 0;
  }
}

// Single-context fusion of the normalisation into the update kernel's last CTA
// (driver.py:411-422 after the column sums): w = sqrt(nsq), owned = hhat / (w > 0 ? w
// : 1), lam = w, gram = H^T H of the normalised rows (rows staged 64 at a time in
// `scratch`), and for the sweep's last mode also gamma + the status hand-off.  Only
// for small row blocks (the host checks rows * R^2): one CTA does it all, in place
// of the normalise (+ gamma) launches.
struct TailArgs {
  const double* hhat;     // nullptr: no fused tail
  int64_t rows;
  double* owned;
  double* lam;
  double* gram;
  double* scratch;        // >= max(64 R, R^2 + R) doubles of shared memory
  PublishArgs pub;        // pub.gamma == nullptr: no gamma / hand-off
  // M as split-K group partials left by the sliced partial MTTKRP (column-major,
  // m_ld apart per column, mgstride apart per group): the update sums them in group
  // order while loading its rows (group_reduce_kernel's arithmetic, one launch fewer)
  int mgroups;            // <= 1: M itself
  int64_t mgstride;
};

// Element (i, r) of M: row-major (mld == 0), or column-major with leading dimension
// mld, optionally the sum over t.mgroups group partials in group order.
__device__ __forceinline__ double load_m(const double* __restrict__ mrows, int64_t mld, int64_t i, int r, int R,
                                         const TailArgs& t) {
  if (!mld) return mrows[i * R + r];
  const double* p = mrows + i + mld * r;
  double s = p[0];
  for (int g = 1; g < t.mgroups; ++g) s += p[g * t.mgstride];
  return s;
}

static __device__ void fused_tail(const TailArgs& t, int R, const double* nsq_s /* shared, R */, double* scale) {
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const double w = sqrt(nsq_s[r]);
    scale[r] = (w > 0.0) ? w : 1.0;
    if (t.lam) t.lam[r] = w;
  }
  __syncthreads();
  const int RR = R * R;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};     // entries threadIdx.x + k * blockDim.x
  double* tile = t.scratch;
  for (int64_t r0 = 0; r0 < t.rows; r0 += 64) {
    const int nr = int(t.rows - r0 < 64 ? t.rows - r0 : 64);
    for (int e = threadIdx.x; e < nr * R; e += blockDim.x) {
      const int il = e / R, c = e - (e / R) * R;
      const int64_t gi = (r0 + il) * R + c;
      const double v = t.hhat[gi] / scale[c];
      t.owned[gi] = v;
      tile[il * R + c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < RR) {
        const int a = e / R, b = e - (e / R) * R;
        double sacc = acc[k];
        for (int il = 0; il < nr; ++il) sacc = fma(tile[il * R + a], tile[il * R + b], sacc);
        acc[k] = sacc;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int e = threadIdx.x + k * blockDim.x;
    if (e < RR) t.gram[e] = acc[k];
  }
  if (t.pub.gamma != nullptr) {
    __threadfence();
    __syncthreads();
    gamma_publish_body(t.pub, R, t.scratch, t.scratch + RR);
  }
}

// ------------------------------------------------------------ MU / HALS ----
// One warp per row; lane l holds columns l and l+32 (R <= 64).
constexpr int kRowWarps = 8;

// Per-CTA column sums of squares (+ beta) -> partials, last CTA reduces in order.
template <int NH>
__device__ void colsum_epilogue(const double (&sq)[NH], double bsum, int R, double* red /* [nw][64] */,
                                double* colbuf, double* part, double* nsq, double* beta, unsigned int* ticket,
                                const TailArgs* tail = nullptr, unsigned long long* clear_last = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NH; ++q) red[warp * 64 + lane + 32 * q] = sq[q];
  __syncthreads();
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    double s = red[r];
    for (int w = 1; w < nw; ++w) s += red[w * 64 + r];
    colbuf[r] = s;
  }
  __syncthreads();
  if (beta) {
    const double b = block_sum(bsum, red);
    if (threadIdx.x == 0) colbuf[R] = b;
    __syncthreads();
  }
  const int stride = R + 1;
  for (int e = threadIdx.x; e < stride; e += blockDim.x) part[size_t(blockIdx.x) * stride + e] = colbuf[e];
  if (last_cta_ticket(ticket)) {
    if (clear_last != nullptr && threadIdx.x == 0) *clear_last = 0ull;   // every CTA is past its reads
    finish_partials(part, gridDim.x, stride, colbuf);
    __syncthreads();
    for (int e = threadIdx.x; e < stride; e += blockDim.x) {
      if (e < R) {
        if (nsq) nsq[e] = colbuf[e];
      } else if (beta) {
        beta[0] = colbuf[e];
      }
    }
    if (tail != nullptr && tail->hhat != nullptr) {
      // every CTA's rows are written (last ticket); red (>= 4 * 64 doubles) holds the scales
      __threadfence();
      __syncthreads();
      fused_tail(*tail, R, colbuf, red);
    }
  }
}

}  // namespace nncp
