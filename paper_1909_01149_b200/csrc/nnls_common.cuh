// Device helpers shared by the NNLS-side translation units (nnls.cu, nnls_iter.cu).
#pragma once

#include "common.cuh"

namespace nncp {

// --------------------------------------------------------------- helpers --
// S[a][b] = prod_{m != mode} 0.5 (G_m[a][b] + G_m[b][a]); order==0: S = grams.
static __device__ void load_hadamard(double* S, const double* __restrict__ grams, int order, int mode, int R) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e - (e / R) * R;
    double v;
    if (order == 0) {
      v = grams[e];
    } else {
      v = 1.0;
      for (int m = 0; m < order; ++m) {
        if (m == mode) continue;
        const double* g = grams + size_t(m) * R * R;
        v *= 0.5 * (g[a * R + b] + g[b * R + a]);
      }
    }
    S[e] = v;
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
// each output is split into `segs` strided segments with four independent
// accumulators, then the segments are summed in order: deterministic for a given
// launch configuration.  Needs blockDim.x doubles of shared scratch.
static __device__ void finish_partials(const double* part, int nblk, int n, double* out) {
  __shared__ double seg_sum[1024];
  const int T = blockDim.x;
  int segs = T / max(n, 1);
  segs = max(1, min(segs, min(32, nblk)));
  if (n * segs <= T) {
    const int t = threadIdx.x;
    if (t < n * segs) {
      const int e = t % n, sg = t / n;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int b = sg;
      for (; b + 3 * segs < nblk; b += 4 * segs) {
        a0 += part[size_t(b) * n + e];
        a1 += part[size_t(b + segs) * n + e];
        a2 += part[size_t(b + 2 * segs) * n + e];
        a3 += part[size_t(b + 3 * segs) * n + e];
      }
      for (; b < nblk; b += segs) a0 += part[size_t(b) * n + e];
      seg_sum[sg * n + e] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n; e += T) {
      double s = seg_sum[e];
      for (int sg = 1; sg < segs; ++sg) s += seg_sum[sg * n + e];
      out[e] = s;
    }
  } else {
    for (int e = threadIdx.x; e < n; e += T) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int b = 0;
      for (; b + 3 < nblk; b += 4) {
        a0 += part[size_t(b) * n + e];
        a1 += part[size_t(b + 1) * n + e];
        a2 += part[size_t(b + 2) * n + e];
        a3 += part[size_t(b + 3) * n + e];
      }
      for (; b < nblk; ++b) a0 += part[size_t(b) * n + e];
      out[e] = (a0 + a1) + (a2 + a3);
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

// ------------------------------------------------------------ MU / HALS ----
// One warp per row; lane l holds columns l and l+32 (R <= 64).
constexpr int kRowWarps = 8;

// Per-CTA column sums of squares (+ beta) -> partials, last CTA reduces in order.
template <int NH>
__device__ void colsum_epilogue(const double (&sq)[NH], double bsum, int R, double* red /* [nw][64] */,
                                double* colbuf, double* part, double* nsq, double* beta, unsigned int* ticket) {
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
    finish_partials(part, gridDim.x, stride, colbuf);
    __syncthreads();
    for (int e = threadIdx.x; e < stride; e += blockDim.x) {
      if (e < R) {
        if (nsq) nsq[e] = colbuf[e];
      } else if (beta) {
        beta[0] = colbuf[e];
      }
    }
  }
}

}  // namespace nncp
