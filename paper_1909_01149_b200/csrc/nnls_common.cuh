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

// Final fixed-order reduction of per-CTA partials [nblk][n] -> out[n] by the last CTA.
static __device__ void finish_partials(const double* part, int nblk, int n, double* out) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) {
    double s = part[e];
    for (int b = 1; b < nblk; ++b) s += part[size_t(b) * n + e];
    out[e] = s;
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
    const int nblk = gridDim.x;
    for (int e = threadIdx.x; e < stride; e += blockDim.x) {
      if (e == R && !beta) continue;
      double s = part[e];
      for (int b = 1; b < nblk; ++b) s += part[size_t(b) * stride + e];
      if (e < R) {
        if (nsq) nsq[e] = s;
      } else {
        beta[0] = s;
      }
    }
  }
}

}  // namespace nncp
