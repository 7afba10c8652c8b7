/*
 * nncp_b200.h -- C ABI of the B200-native dense NNCP hot path.
 *
 * Drop-in boundary for the reference package `nncp` (/root/reference/pkg/src/nncp),
 * whose hot path is the alternating-update loop of driver.py:331-449.  Each entry
 * point below replaces one numeric call site of that loop; the replaced reference
 * interface is cited on every declaration.  The reference is pure Python, so the
 * binding a maintainer adds is a ctypes stub (INTEGRATION.md shows it); this
 * repository's own Python mirror (paper_1909_01149_b200/) binds exactly these
 * symbols.
 *
 * Conventions (identical to the reference, tensor_ops.py:1-13):
 *   - tensors: flat float64, mode-1 index fastest (column-major generalisation);
 *   - factor matrices: row-major (I_n, R) float64;
 *   - dimension-tree temporaries: retained-mode indices fastest, rank slowest
 *     (dimtree.py:68-99), i.e. column-major (prod(retained), R);
 *   - Gram buffers hold the RAW H^T H (R x R, row-major); every consumer reads the
 *     symmetrised 0.5 (G + G^T) exactly as driver.py:353,422 stores it.
 * All pointers are DEVICE pointers (caller-owned, e.g. torch CUDA tensors) unless
 * the parameter is documented as host.  Every call is asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream) and returns NNCP_OK or an error
 * code; nncp_last_error() returns the thread-local message.  Workspaces must be
 * zero-filled once at allocation (they carry self-resetting reduction tickets).
 */
#ifndef NNCP_B200_H
#define NNCP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNCP_ABI_VERSION 1
#define NNCP_MAX_ORDER 8
#define NNCP_MAX_RANK 64
#define NNCP_STATUS_WORDS 4

/* return codes; the Python mirror maps VALUE -> ValueError, RUNTIME -> RuntimeError */
#define NNCP_OK 0
#define NNCP_ERR_VALUE 1
#define NNCP_ERR_RUNTIME 2
#define NNCP_ERR_CUDA 3
#define NNCP_ERR_UNSUPPORTED 4

#define NNCP_SIDE_LEFT 0      /* dimtree.py:111-117: T = X_(1:S)   . KRP(H_{S+1..N}) */
#define NNCP_SIDE_RIGHT 1     /* dimtree.py:118-124: T = X_(1:S)^T . KRP(H_{1..S})   */
#define NNCP_TTV_TRAILING 0   /* dimtree.py:159-165 */
#define NNCP_TTV_LEADING 1    /* dimtree.py:166-172 */
#define NNCP_ALGO_MU 1        /* updaters.py:91-94   */
#define NNCP_ALGO_HALS 2      /* updaters.py:97-118  */
#define NNCP_ALGO_BPP 3       /* updaters.py:121-164 */
#define NNCP_ALGO_UCP 4       /* updaters.py:77-88 (status[0] bit 0: ridge applied; still singular with the ridge:
                                 the minimum-norm lstsq solution through a Jacobi eigendecomposition) */

/* status words (device int32[NNCP_STATUS_WORDS]) written by nncp_update:
 *   [0],[1]  HALS: bit r set when gram diagonal r <= 0 (updaters.py:110-113)
 *   [2]      BPP : smallest failing row, INT32_MAX when none (updaters.py:155,163)
 *   [3]      BPP : failure kind, 0 none, 1 cycling (BppCyclingError), 2 singular solve
 * The caller zero-fills [0],[1],[3] and sets [2]=INT32_MAX before the call
 * (nncp_status_reset does it on the stream). */

int nncp_abi_version(void);
const char* nncp_last_error(void);
/* SM count of the current device, for host-side bookkeeping */
int nncp_device_sms(void);
/* Number of kernels this library has launched in the process (evidence counter). */
unsigned long long nncp_launch_count(void);

/* dimtree.py:25-39 choose_split_mode.  dims: host array. */
int nncp_choose_split(int order, const int64_t* dims, int strict, int* split_out);

/* Workspace bytes that covers every call below for this local tensor shape/rank. */
size_t nncp_workspace_bytes(int order, const int64_t* dims, int split, int rank);

/* tensor_ops.py:76-78 norm_squared: out[0] = sum x^2 (deterministic reduction). */
int nncp_norm_squared(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream);
/* Same sum (bitwise), plus in the same pass (out_min: 3 doubles): out_min[0] = min x,
 * the negative-entry UserWarning of driver.py:571-573 without a second read of the
 * tensor; out_min[1] = max |x| (NaN if any entry is NaN or +-Inf); out_min[2] = the
 * smallest nonzero |x| (+Inf if none) -- the sign / dynamic-range facts the engine's
 * "auto" MTTKRP choice needs before slicing the tensor.  n >= 1. */
int nncp_norm_squared_min(const double* x, int64_t n, double* out_sum, double* out_min, void* ws, size_t ws_bytes,
                          void* stream);

/* dimtree.py:102-127 partial_mttkrp.  dims: host.  factors: host array of `order`
 * device pointers (row-major (dims[n], R)); only the contracted side's factors are
 * read.  out: column-major (prod(retained), R).  The Khatri-Rao rows are generated
 * on the fly (never materialised); FP64 tensor cores (DMMA) fed by TMA. */
int nncp_partial_mttkrp(const double* x, int order, const int64_t* dims, int split, int side,
                        const double* const* factors, int rank, double* out, void* ws,
                        size_t ws_bytes, void* stream);

/* Sliced-tensor partial MTTKRP (same contraction as nncp_partial_mttkrp, on the
 * int8 tensor cores: tcgen05.mma kind::i8, Ozaki-scheme digit slices).
 * The tensor is sliced ONCE (nncp_slice_tensor) for a fixed split; every later
 * partial reads `levels` int8 digit planes (levels bytes per element) instead of
 * the fp64 tensor.  levels: 6 (46-bit operands) or 7 (54-bit).
 * nncp_sliced_tensor_bytes: device buffer size for nncp_slice_tensor (host out).
 * nncp_sliced_workspace_bytes: workspace of nncp_partial_mttkrp_sliced (both sides),
 * 0 for an invalid shape.  Buffers are used from their first 1 KB boundary on. */
int nncp_sliced_tensor_bytes(int order, const int64_t* dims, int split, int levels, size_t* bytes);
int nncp_slice_tensor(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                      size_t bytes, void* stream);
/* nncp_slice_tensor in two steps, so a run that slices reads the 8-byte tensor once
 * before the planes pass instead of twice: nncp_norm_rowmax takes the row maxima
 * into `sliced` AND, in the same read, nncp_norm_squared_min's outputs (out_sum[0] =
 * sum x^2, out_min[0..2] = min x, max |x|, min nonzero |x|; the facts the engine
 * choice needs, driver.py:338-345); nncp_slice_tensor_planes then writes the digit
 * planes from those row maxima (same bits as nncp_slice_tensor). */
int nncp_norm_rowmax(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                     size_t bytes, double* out_sum, double* out_min, void* ws, size_t ws_bytes, void* stream);
int nncp_slice_tensor_planes(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                             size_t bytes, void* stream);
size_t nncp_sliced_workspace_bytes(int order, const int64_t* dims, int split, int rank, int levels);
int nncp_partial_mttkrp_sliced(const void* sliced, int order, const int64_t* dims, int split, int side,
                               const double* const* factors, int rank, int levels, double* out, void* ws,
                               size_t ws_bytes, void* stream);

/* nncp_partial_mttkrp_sliced without the final split-K group reduction: when the
 * contraction was split into groups (*groups_out > 1) the group partials stay in the
 * workspace at *parts_out (column-major (rows, R) each, *gstride_out doubles apart) for a
 * consumer that sums them itself (nncp_update_grouped: the last mode's MTTKRP of a
 * 3-way tree is the right partial itself); otherwise out is written and
 * *parts_out = out, *groups_out = 1.  One launch fewer per sweep. */
int nncp_partial_mttkrp_sliced_deferred(const void* sliced, int order, const int64_t* dims, int split, int side,
                                        const double* const* factors, int rank, int levels, double* out, void* ws,
                                        size_t ws_bytes, const double** parts_out, int* groups_out,
                                        int64_t* gstride_out, void* stream);

/* The left sliced partial plus the dimension tree's first trailing multi-TTV in one
 * pass (dimtree.py:241-250 mode 1: out_trailing = multi_ttv(T_L, H_2, trailing)),
 * accumulated in the GEMM epilogue instead of re-reading T_L.  Supported for split 2,
 * dims[0] a multiple of 128, rank <= 32 and long row tiles (nncp_sliced_trailing_supported);
 * NNCP_ERR_UNSUPPORTED otherwise (use nncp_partial_mttkrp_sliced + nncp_multi_ttv).  out_temp as for the left partial;
 * out_trailing: column-major (dims[0], R). */
/* 1 when nncp_partial_mttkrp_sliced_trailing supports (and is worth it for) this shape. */
int nncp_sliced_trailing_supported(int order, const int64_t* dims, int split, int rank, int levels);
int nncp_partial_mttkrp_sliced_trailing(const void* sliced, int order, const int64_t* dims, int split,
                                        const double* const* factors, int rank, int levels, double* out_temp,
                                        double* out_trailing, void* ws, size_t ws_bytes, void* stream);

/* dimtree.py:135-175 multi_ttv.  temp: column-major (prod(ret_dims), R).
 * TRAILING: coeff = KRP(coeff[0..ncoeff)) with coeff_rows[k] rows each, whose
 *   product must equal prod(ret_dims[1:]); out retains ret_dims[0].
 * LEADING : ncoeff == 1, coeff[0] is (ret_dims[0], R); out retains ret_dims[1:].
 * ret_dims, coeff, coeff_rows: host arrays. */
int nncp_multi_ttv(const double* temp, int nret, const int64_t* ret_dims, int rank, int side,
                   const double* const* coeff, const int64_t* coeff_rows, int ncoeff, double* out,
                   void* stream);

/* tensor_ops.py:121-137 khatri_rao, materialised (the hot path never does this):
 * out (prod(rows) x rank, row-major) row (i_1..i_m) = prod_f factors[f][i_f, :], the first
 * factor's index fastest.  factors: host array of `count` (1..8) device pointers. */
int nncp_khatri_rao(const double* const* factors, const int64_t* rows, int count, int rank, double* out,
                    void* stream);

/* dimtree.py:287 np.ascontiguousarray(temp.as_matrix()): column-major -> row-major. */
int nncp_temp_to_rows(const double* temp, int64_t rows, int rank, double* out_rows, void* stream);

/* Status reset on the stream (see status words above). */
int nncp_status_reset(int* status, void* stream);
/* The same for `count` consecutive status blocks (one per mode) in one launch. */
int nncp_status_reset_n(int* status, int count, void* stream);

/* Fused NNLS factor update (driver.py:396-418 first half + updaters.py):
 *   S = prod_{m != mode} sym(G_m)          (tensor_ops.py:146-155), or when order == 0
 *       `grams` is S itself (R x R, used as given: UpdateInputs.gram);
 *   current = owned * lam (lam may be NULL -> ones)                (driver.py:403);
 *   hhat = MU / HALS / BPP(S, mttkrp_rows, current)                (updaters.py);
 *   nsq[r] = sum_i hhat[i,r]^2 (may be NULL)                       (driver.py:413);
 *   beta[0] = <mttkrp_rows, hhat> when beta != NULL                (driver.py:428).
 * mttkrp_rows, owned, hhat: row-major (rows, R). */
int nncp_update(int algo, const double* grams, int order, int mode, int rank,
                const double* mttkrp_rows, const double* owned, const double* lam, int64_t rows,
                double* hhat, double* nsq, double* beta, int* status, void* ws, size_t ws_bytes,
                void* stream);
/* nncp_update with extra inputs.  mu_eps: the MU epsilon (mu_update(inp, eps),
 * updaters.py:91-94; nncp_update uses MU_EPSILON = 1e-16, updaters.py:27).
 * bpp_sets (BPP only, may be NULL = the reference's cold start from P = {}): device
 * uint64[rows], per row the passive-set bit mask to start from, overwritten with the
 * final one (0 after a failure).  The NNLS minimiser is unique for SPD S, so a warm
 * start from the previous outer iteration's sets reaches the same solution in fewer
 * passes.  m_ld: 0 = mttkrp_rows is row-major (rows x rank); > 0 = column-major with
 * that leading dimension (>= rows), i.e. the dimension tree's temporary
 * (dimtree.py:68-99) consumed in place, without the np.ascontiguousarray transpose
 * (dimtree.py:287). */
int nncp_update_ex(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                   const double* owned, const double* lam, int64_t rows, double* hhat, double* nsq, double* beta,
                   int* status, double mu_eps, void* bpp_sets, int64_t m_ld, void* ws, size_t ws_bytes,
                   void* stream);
/* BPP's S = prod_{m != mode} sym(G_m) and S^-1 formed ahead of the update -- they need
 * only the Grams, so a caller can launch this on a second stream while the mode's
 * MTTKRP runs and join before nncp_update_ex / _grouped / _normalize (driver.py:396-418:
 * the Gram Hadamard + the solves of updaters.py:121-164).  The result goes into a
 * block after the passive sets of `bpp_sets` (allocate nncp_bpp_sets_words(rows, rank)
 * uint64 words instead of rows); the next BPP update of that buffer with the same
 * (order, mode, rank) takes S and S^-1 from it instead of forming them (the same
 * bits: it is the update's own elimination) and marks the block used. */
size_t nncp_bpp_sets_words(int64_t rows, int rank);
int nncp_bpp_prepare(const double* grams, int order, int mode, int rank, void* bpp_sets, int64_t rows,
                     void* stream);
/* nncp_update_ex with M given as m_groups column-major partials (leading dimension
 * m_ld >= rows, m_gstride >= m_ld * rank doubles apart) summed in group order while the
 * rows are loaded -- the output of nncp_partial_mttkrp_sliced_deferred.  MU, HALS, BPP.
 * The partials must not overlap the workspace's tickets and per-CTA partials. */
int nncp_update_grouped(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_parts,
                        int64_t m_ld, int m_groups, int64_t m_gstride, const double* owned, const double* lam,
                        int64_t rows, double* hhat, double* nsq, double* beta, int* status, double mu_eps,
                        void* bpp_sets, void* ws, size_t ws_bytes, void* stream);
/* nncp_update_ex followed, in the same launch, by the normalisation of
 * nncp_normalize_gram (driver.py:411-422) for a single context: the kernel's last CTA
 * turns the column sums into w = sqrt(nsq), writes owned = hhat / (w > 0 ? w : 1),
 * lam = w (owned / lam may be the inputs: they are read before the last CTA starts)
 * and gram_out = H^T H of the normalised rows; with gamma_out it also does
 * nncp_gamma_publish over status_all (the sweep's `status_count` per-mode blocks;
 * grams: all `order` Grams, this mode's being gram_out).  Small
 * row blocks only (one CTA does it; the host keeps rows * rank^2 <= 2^20), rank <= 32. */
int nncp_update_normalize(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                          double* owned, double* lam, int64_t rows, double* hhat, double* nsq, double* beta,
                          int* status, double mu_eps, void* bpp_sets, int64_t m_ld, double* gram_out, double* gamma_out,
                          int* status_all, int status_count, double* codes, int nslots, int offset, int* masks_out,
                          void* ws, size_t ws_bytes, void* stream);

/* driver.py:414-420: w = sqrt(nsq); owned = hhat / (w > 0 ? w : 1); lam = w;
 * gram = owned^T owned (raw, local rows).  owned may alias hhat; lam and gram may be NULL. */
int nncp_normalize_gram(const double* hhat, const double* nsq, int64_t rows, int rank,
                        double* owned, double* lam, double* gram, void* ws, size_t ws_bytes,
                        void* stream);

/* driver.py:351 local Gram h^T h (raw). */
int nncp_gram(const double* h, int64_t rows, int rank, double* gram, void* ws, size_t ws_bytes,
              void* stream);

/* driver.py:411-422 from the All-Reduced Gram of the UNnormalised rows (one collective
 * instead of the norm and Gram All-Reduces): w = sqrt(diag(gram_raw)),
 * owned = hhat / (w > 0 ? w : 1), lam = w, gram = sym(gram_raw) / (w' w'^T).
 * gram must not alias gram_raw. */
int nncp_normalize_from_gram(const double* hhat, const double* gram_raw, int64_t rows, int rank, double* owned,
                             double* lam, double* gram, void* stream);

/* driver.py:368,431 gamma = lam^T (prod_m sym(G_m)) lam over all `order` Grams. */
int nncp_gamma(const double* grams, int order, int rank, const double* lam, double* gamma,
               void* stream);
/* nncp_normalize_gram for the sweep's last mode, whose last CTA then also does
 * nncp_gamma_publish (grams: all `order` Grams, this mode's being the one written):
 * one launch instead of two when no All-Reduce of the Gram sits in between (a
 * single context). */
int nncp_normalize_gram_publish(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned,
                                double* lam, double* gram, void* ws, size_t ws_bytes, const double* grams, int order,
                                double* gamma_out, int* status, int count, double* codes, int nslots, int offset,
                                int* masks_out, void* stream);

/* The same gamma, plus the end-of-sweep status hand-off (grid.py:172-203 failure
 * propagation).  codes[0..nslots) is a rank-slotted vector: every slot is zeroed, then
 * for n < count codes[offset + n] = kind * 2^32 + failing row of status n (0 when the
 * update succeeded; exact in fp64) and masks_out[2n..2n+1] = its warning bits (may be
 * NULL); then status n is reset (replaces nncp_status_reset_n inside a sweep).  One
 * SUM All-Reduce of `codes` then gives every rank every rank's failures. */
int nncp_gamma_publish(const double* grams, int order, int rank, const double* lam, double* gamma_out, int* status,
                       int count, double* codes, int nslots, int offset, int* masks_out, void* stream);

/* tensor_ops.py:208-212 matrix_inner_product <a, b * lam> (lam may be NULL). */
int nncp_inner(const double* a, const double* b, const double* lam, int64_t rows, int rank,
               double* out, void* ws, size_t ws_bytes, void* stream);

/* ---- the remaining update rules -------------------------- */

/* One ADMM inner step for all rows (updaters.py:196-215): xhat = (S + rho I)^-1 (m + rho (x + u)),
 * x_out = max(xhat - u, 0), u += x_out - xhat (in place); sums5 = local [|x-xhat|^2, |x|^2,
 * |xhat|^2, |x-xprev|^2, |u|^2] for the hook, sums5[5] = the rho used (6 doubles).
 * rho <= 0: tr(S)/R (updaters.py:167-170).
 * S as in nncp_update (Grams + mode, or order == 0 and S given). */
int nncp_admm_step(const double* grams, int order, int mode, int rank, double rho, const double* mttkrp_rows,
                   const double* x_in, double* u, double* x_out, int64_t rows, double* sums5, int* status,
                   void* ws, size_t ws_bytes, void* stream);

/* nesterov_hyperparams (updaters.py:223-243): hyper3 = (lam, alpha, beta) from the extreme
 * eigenvalues of S (device Jacobi). */
int nncp_nes_hyper(const double* grams, int order, int mode, int rank, double prox_floor, double* hyper3,
                   void* stream);

/* One accelerated projected-gradient step (updaters.py:266-277) for all rows; maxes2 = local
 * [max |x_out - x_in|, max |x_out|] for the max-hook. */
int nncp_nes_step(const double* grams, int order, int mode, int rank, const double* hyper3,
                  const double* mttkrp_rows, const double* y_in, const double* x_in, const double* xstar,
                  double* x_out, double* y_out, int64_t rows, double* maxes2, void* ws, size_t ws_bytes,
                  void* stream);

/* Elementwise helpers of the driver (driver.py:403, 464-486). */
int nncp_scale_columns(const double* in, const double* colscale, int64_t rows, int rank, double* out,
                       void* stream);
int nncp_extrapolate(const double* cur, const double* prev, int64_t n, double step, double* out, void* stream);
int nncp_nes_lambda(const double* cand_lam, const double* nsq, int order, int rank, double* lam, void* stream);
int nncp_colsumsq(const double* h, int64_t rows, int rank, double* nsq, void* ws, size_t ws_bytes, void* stream);

/* Synthetic input (BASELINE.json configs; tensor_io.py:103-125 generalised with noise):
 * x[i] = sum_r prod_n H_n(i_n, r) + noise_scale * |N(0,1)|_i, the Gaussian drawn from
 * Philox4x32-10 keyed by (seed) and counted by the GLOBAL linear index, so every grid
 * block is bit-identical to the matching slice of the global tensor.
 * local_dims/offsets/global_dims: host.  factors: host array of device pointers to the
 * LOCAL row blocks (local_dims[n] x R). */
int nncp_synthetic(double* x, int order, const int64_t* local_dims, const int64_t* offsets,
                   const int64_t* global_dims, const double* const* factors, int rank,
                   double noise_scale, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* NNCP_B200_H */
