// extern "C" boundary (include/nncp_b200.h): argument validation, error
// reporting and dispatch to the kernels.  Validation messages mirror the
// reference's ValueError / RuntimeError texts where one exists.
#include <atomic>
#include <string>

#include "nnls_common.cuh"

namespace nncp {

thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// kernels (defined in the other translation units)
struct PartialPlan;
int partial_mttkrp(const double*, int, const int64_t*, int, int, const double* const*, int, double*, void*, size_t,
                   cudaStream_t);
size_t partial_ws_bytes(int order, const int64_t* dims, int split, int side, int rank);
int multi_ttv(const double*, int, const int64_t*, int, int, const double* const*, const int64_t*, int, double*,
              cudaStream_t);
int temp_to_rows(const double*, int64_t, int, double*, cudaStream_t);
int khatri_rao(const double* const*, const int64_t*, int, int, double*, cudaStream_t);
int update(int, const double*, int, int, int, const double*, const double*, const double*, int64_t, double*, double*,
           double*, int*, void*, size_t, cudaStream_t, double, void*, int64_t, const TailArgs*);
int normalize_gram(const double*, const double*, int64_t, int, double*, double*, double*, void*, size_t, cudaStream_t,
                   int);
int gamma(const double*, int, int, const double*, double*, cudaStream_t);
int normalize_from_gram(const double*, const double*, int64_t, int, double*, double*, double*, cudaStream_t);
int gamma_publish(const double*, int, int, const double*, double*, int*, int, double*, int, int, int*, cudaStream_t);
int normalize_gram_publish(const double*, const double*, int64_t, int, double*, double*, double*, void*, size_t,
                           const double*, int, double*, int*, int, double*, int, int, int*, cudaStream_t);
int inner(const double*, const double*, const double*, int64_t, int, double*, void*, size_t, cudaStream_t);
int norm_squared(const double*, int64_t, double*, double*, void*, size_t, cudaStream_t);
int status_reset(int*, int, cudaStream_t);
size_t row_update_part_elems(int64_t rows, int rank);
size_t bpp_sets_words(int64_t rows, int rank);
int bpp_prepare(const double*, int, int, int, void*, int64_t, cudaStream_t);
int ucp(const double*, int, int, int, const double*, int64_t, double*, double*, double*, int*, void*, size_t,
        cudaStream_t, int64_t, const TailArgs*);
int admm_step(const double*, int, int, int, double, const double*, const double*, double*, double*, int64_t, double*,
              int*, void*, size_t, cudaStream_t);
int nes_hyper(const double*, int, int, int, double, double*, cudaStream_t);
int nes_step(const double*, int, int, int, const double*, const double*, const double*, const double*, const double*,
             double*, double*, int64_t, double*, void*, size_t, cudaStream_t);
int scale_columns(const double*, const double*, int64_t, int, double*, cudaStream_t);
int extrapolate(const double*, const double*, int64_t, double, double*, cudaStream_t);
int nes_lambda(const double*, const double*, int, int, double*, cudaStream_t);
int colsumsq(const double*, int64_t, int, double*, void*, size_t, cudaStream_t);
int synthetic(double*, int, const int64_t*, const int64_t*, const int64_t*, const double* const*, int, double,
              uint64_t, cudaStream_t);

size_t sliced_tensor_bytes(int order, const int64_t* dims, int split, int levels);
size_t sliced_ws_bytes(int order, const int64_t* dims, int split, int rank, int levels);
bool sliced_trailing_supported(int order, const int64_t* dims, int split, int rank, int levels);
int slice_tensor(const double*, int, const int64_t*, int, int, void*, size_t, cudaStream_t);
int norm_rowmax(const double*, int, const int64_t*, int, int, void*, size_t, double*, double*, void*, size_t,
                cudaStream_t);
int slice_tensor_planes(const double*, int, const int64_t*, int, int, void*, size_t, cudaStream_t);
int sliced_partial_mttkrp(const void*, int, const int64_t*, int, int, const double* const*, int, int, double*, double*,
                          void*, size_t, cudaStream_t, const double** parts_out = nullptr, int* groups_out = nullptr,
                          int64_t* gstride_out = nullptr);

// caller buffers for the sliced path are used from the next 1 KB boundary on
static inline void* align1k(const void* p, size_t bytes, size_t* avail) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023);
  const size_t skip = a - reinterpret_cast<uintptr_t>(p);
  *avail = bytes > skip ? bytes - skip : 0;
  return reinterpret_cast<void*>(a);
}

static int check_common(int order, const int64_t* dims, int rank) {
  if (order < 2 || order > kMaxOrder) return fail(NNCP_ERR_VALUE, "tensor order must be in [2, 8]");
  if (rank < 1) return fail(NNCP_ERR_VALUE, "rank must be at least 1");
  if (rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank above 64 is not supported on the device path");
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return fail(NNCP_ERR_VALUE, "dims must be positive");
  return NNCP_OK;
}

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace nncp

using namespace nncp;

extern "C" {

int nncp_abi_version(void) { return NNCP_ABI_VERSION; }
const char* nncp_last_error(void) { return g_last_error.c_str(); }
int nncp_device_sms(void) { return num_sms(); }
unsigned long long nncp_launch_count(void) { return g_launches.load(); }

int nncp_choose_split(int order, const int64_t* dims, int strict, int* split_out) {
  if (order < 2) return fail(NNCP_ERR_VALUE, "need at least 2 modes");
  for (int s = 1; s < order; ++s) {
    // products can exceed int64 only for absurd shapes; use long double to compare safely
    long double left = 1, right = 1;
    for (int n = 0; n < s; ++n) left *= (long double)dims[n];
    for (int n = s; n < order; ++n) right *= (long double)dims[n];
    if (left > right || (!strict && left == right)) {
      *split_out = s;
      return NNCP_OK;
    }
  }
  *split_out = order - 1;
  return NNCP_OK;
}

size_t nncp_workspace_bytes(int order, const int64_t* dims, int split, int rank) {
  size_t b = 0;
  b = std::max(b, partial_ws_bytes(order, dims, split, NNCP_SIDE_LEFT, rank));
  b = std::max(b, partial_ws_bytes(order, dims, split, NNCP_SIDE_RIGHT, rank));
  int64_t maxrows = 1;
  for (int n = 0; n < order; ++n) maxrows = std::max<int64_t>(maxrows, dims[n]);
  b = std::max(b, 256 + sizeof(double) * row_update_part_elems(maxrows, rank));
  return 256 + b;
}

int nncp_norm_squared(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0) return fail(NNCP_ERR_VALUE, "negative length");
  return norm_squared(x, n, out, nullptr, ws, ws_bytes, S(stream));
}

int nncp_norm_squared_min(const double* x, int64_t n, double* out_sum, double* out_min, void* ws, size_t ws_bytes,
                          void* stream) {
  if (n < 1) return fail(NNCP_ERR_VALUE, "empty tensor");
  if (!out_min) return fail(NNCP_ERR_VALUE, "null min output");
  return norm_squared(x, n, out_sum, out_min, ws, ws_bytes, S(stream));
}

int nncp_partial_mttkrp(const double* x, int order, const int64_t* dims, int split, int side,
                        const double* const* factors, int rank, double* out, void* ws, size_t ws_bytes,
                        void* stream) {
  int rc = check_common(order, dims, rank);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (side != NNCP_SIDE_LEFT && side != NNCP_SIDE_RIGHT)
    return fail(NNCP_ERR_VALUE, "side must be 'left' or 'right'");
  // the partial kernels use the first 256 bytes of nothing: split-K partials start at ws
  return partial_mttkrp(x, order, dims, split, side, factors, rank, out, ws ? static_cast<char*>(ws) + 256 : nullptr,
                        ws_bytes > 256 ? ws_bytes - 256 : 0, S(stream));
}

int nncp_sliced_tensor_bytes(int order, const int64_t* dims, int split, int levels, size_t* bytes) {
  int rc = check_common(order, dims, 1);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (levels != 6 && levels != 7) return fail(NNCP_ERR_UNSUPPORTED, "sliced MTTKRP supports 6 or 7 digit levels");
  *bytes = 1024 + sliced_tensor_bytes(order, dims, split, levels);
  return NNCP_OK;
}

int nncp_slice_tensor(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                      size_t bytes, void* stream) {
  int rc = check_common(order, dims, 1);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (!x || !sliced) return fail(NNCP_ERR_VALUE, "null tensor or sliced buffer");
  size_t avail = 0;
  void* base = align1k(sliced, bytes, &avail);
  return slice_tensor(x, order, dims, split, levels, base, avail, S(stream));
}

int nncp_norm_rowmax(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                     size_t bytes, double* out_sum, double* out_min, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_common(order, dims, 1);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (!x || !sliced) return fail(NNCP_ERR_VALUE, "null tensor or sliced buffer");
  size_t avail = 0;
  void* base = align1k(sliced, bytes, &avail);
  return norm_rowmax(x, order, dims, split, levels, base, avail, out_sum, out_min, ws, ws_bytes, S(stream));
}

int nncp_slice_tensor_planes(const double* x, int order, const int64_t* dims, int split, int levels, void* sliced,
                             size_t bytes, void* stream) {
  int rc = check_common(order, dims, 1);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (!x || !sliced) return fail(NNCP_ERR_VALUE, "null tensor or sliced buffer");
  size_t avail = 0;
  void* base = align1k(sliced, bytes, &avail);
  return slice_tensor_planes(x, order, dims, split, levels, base, avail, S(stream));
}

size_t nncp_sliced_workspace_bytes(int order, const int64_t* dims, int split, int rank, int levels) {
  if (order < 2 || order > kMaxOrder || rank < 1 || rank > kMaxRank || split < 1 || split >= order) return 0;
  return 256 + 1024 + sliced_ws_bytes(order, dims, split, rank, levels);
}

int nncp_partial_mttkrp_sliced(const void* sliced, int order, const int64_t* dims, int split, int side,
                               const double* const* factors, int rank, int levels, double* out, void* ws,
                               size_t ws_bytes, void* stream) {
  int rc = check_common(order, dims, rank);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (side != NNCP_SIDE_LEFT && side != NNCP_SIDE_RIGHT)
    return fail(NNCP_ERR_VALUE, "side must be 'left' or 'right'");
  if (!sliced) return fail(NNCP_ERR_VALUE, "null sliced tensor");
  size_t dummy = 0, avail = 0;
  const void* base = align1k(sliced, 1024, &dummy);
  // the first 256 workspace bytes hold the reduction tickets of the other kernels
  void* w = (ws && ws_bytes > 256) ? align1k(static_cast<char*>(ws) + 256, ws_bytes - 256, &avail) : nullptr;
  return sliced_partial_mttkrp(base, order, dims, split, side, factors, rank, levels, out, nullptr, w, avail,
                               S(stream));
}

int nncp_partial_mttkrp_sliced_deferred(const void* sliced, int order, const int64_t* dims, int split, int side,
                                        const double* const* factors, int rank, int levels, double* out, void* ws,
                                        size_t ws_bytes, const double** parts_out, int* groups_out,
                                        int64_t* gstride_out, void* stream) {
  int rc = check_common(order, dims, rank);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (side != NNCP_SIDE_LEFT && side != NNCP_SIDE_RIGHT)
    return fail(NNCP_ERR_VALUE, "side must be 'left' or 'right'");
  if (!sliced || !parts_out || !groups_out || !gstride_out) return fail(NNCP_ERR_VALUE, "null argument");
  size_t dummy = 0, avail = 0;
  const void* base = align1k(sliced, 1024, &dummy);
  void* w = (ws && ws_bytes > 256) ? align1k(static_cast<char*>(ws) + 256, ws_bytes - 256, &avail) : nullptr;
  return sliced_partial_mttkrp(base, order, dims, split, side, factors, rank, levels, out, nullptr, w, avail,
                               S(stream), parts_out, groups_out, gstride_out);
}

int nncp_sliced_trailing_supported(int order, const int64_t* dims, int split, int rank, int levels) {
  if (order < 2 || order > kMaxOrder || rank < 1 || rank > kMaxRank || split < 1 || split >= order) return 0;
  for (int n = 0; n < order; ++n)
    if (dims[n] < 1) return 0;
  if (levels != 6 && levels != 7) return 0;
  return sliced_trailing_supported(order, dims, split, rank, levels) ? 1 : 0;
}

int nncp_partial_mttkrp_sliced_trailing(const void* sliced, int order, const int64_t* dims, int split,
                                        const double* const* factors, int rank, int levels, double* out_temp,
                                        double* out_trailing, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_common(order, dims, rank);
  if (rc) return rc;
  if (split < 1 || split >= order) return fail(NNCP_ERR_VALUE, "split must be in [1, order-1]");
  if (!sliced || !out_trailing) return fail(NNCP_ERR_VALUE, "null sliced tensor or trailing output");
  size_t dummy = 0, avail = 0;
  const void* base = align1k(sliced, 1024, &dummy);
  void* w = (ws && ws_bytes > 256) ? align1k(static_cast<char*>(ws) + 256, ws_bytes - 256, &avail) : nullptr;
  return sliced_partial_mttkrp(base, order, dims, split, NNCP_SIDE_LEFT, factors, rank, levels, out_temp,
                               out_trailing, w, avail, S(stream));
}

int nncp_multi_ttv(const double* temp, int nret, const int64_t* ret_dims, int rank, int side,
                   const double* const* coeff, const int64_t* coeff_rows, int ncoeff, double* out, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_VALUE, "bad rank");
  return multi_ttv(temp, nret, ret_dims, rank, side, coeff, coeff_rows, ncoeff, out, S(stream));
}

int nncp_khatri_rao(const double* const* factors, const int64_t* rows, int count, int rank, double* out,
                    void* stream) {
  if (rank < 1) return fail(NNCP_ERR_VALUE, "rank must be positive");
  return khatri_rao(factors, rows, count, rank, out, S(stream));
}

int nncp_temp_to_rows(const double* temp, int64_t rows, int rank, double* out_rows, void* stream) {
  return temp_to_rows(temp, rows, rank, out_rows, S(stream));
}

int nncp_status_reset(int* status, void* stream) { return status_reset(status, 1, S(stream)); }

int nncp_status_reset_n(int* status, int count, void* stream) {
  if (count < 1) return fail(NNCP_ERR_VALUE, "status block count must be positive");
  return status_reset(status, count, S(stream));
}

static int update_dispatch(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                           const double* owned, const double* lam, int64_t rows, double* hhat, double* nsq,
                           double* beta, int* status, double mu_eps, void* bpp_sets, int64_t m_ld, const TailArgs* tail,
                           void* ws, size_t ws_bytes, void* stream, int m_groups = 1, int64_t m_gstride = 0) {
  if (m_ld < 0 || (m_ld > 0 && m_ld < rows)) return fail(NNCP_ERR_VALUE, "m_ld must be 0 (row-major) or >= rows");
  if (m_groups < 1 || (m_groups > 1 && (m_ld == 0 || m_gstride < m_ld * rank)))
    return fail(NNCP_ERR_VALUE, "group partials need m_ld > 0 and m_gstride >= m_ld * rank");
  if (m_groups > 1 && algo != NNCP_ALGO_MU && algo != NNCP_ALGO_HALS && algo != NNCP_ALGO_BPP)
    return fail(NNCP_ERR_UNSUPPORTED, "group partials: MU, HALS or BPP");
  TailArgs targs = tail ? *tail : TailArgs{};
  targs.mgroups = m_groups;
  targs.mgstride = m_gstride;
  tail = &targs;
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64] on the device path");
  if (order < 0 || order > kMaxOrder) return fail(NNCP_ERR_VALUE, "bad order");
  if (order > 0 && (mode < 0 || mode >= order)) return fail(NNCP_ERR_VALUE, "exclude index out of range");
  if (!status) return fail(NNCP_ERR_VALUE, "status buffer required");
  if (algo == NNCP_ALGO_UCP) {
    if (rows <= 0) {
      if (nsq) NNCP_CUDA_TRY(cudaMemsetAsync(nsq, 0, sizeof(double) * rank, S(stream)));
      if (beta) NNCP_CUDA_TRY(cudaMemsetAsync(beta, 0, sizeof(double), S(stream)));
      return NNCP_OK;
    }
    return ucp(grams, order, mode, rank, mttkrp_rows, rows, hhat, nsq, beta, status, ws, ws_bytes, S(stream), m_ld,
               tail);
  }
  return update(algo, grams, order, mode, rank, mttkrp_rows, owned, lam, rows, hhat, nsq, beta, status, ws, ws_bytes,
                S(stream), mu_eps, bpp_sets, m_ld, tail);
}

int nncp_update_ex(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                   const double* owned, const double* lam, int64_t rows, double* hhat, double* nsq, double* beta,
                   int* status, double mu_eps, void* bpp_sets, int64_t m_ld, void* ws, size_t ws_bytes,
                   void* stream) {
  return update_dispatch(algo, grams, order, mode, rank, mttkrp_rows, owned, lam, rows, hhat, nsq, beta, status, mu_eps,
                         bpp_sets, m_ld, nullptr, ws, ws_bytes, stream);
}

size_t nncp_bpp_sets_words(int64_t rows, int rank) { return bpp_sets_words(rows, rank); }

int nncp_bpp_prepare(const double* grams, int order, int mode, int rank, void* bpp_sets, int64_t rows, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  if (order > kMaxOrder || mode < 0 || mode >= order) return fail(NNCP_ERR_VALUE, "exclude index out of range");
  if (rows < 0) return fail(NNCP_ERR_VALUE, "negative row count");
  return bpp_prepare(grams, order, mode, rank, bpp_sets, rows, S(stream));
}

int nncp_update_grouped(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_parts,
                        int64_t m_ld, int m_groups, int64_t m_gstride, const double* owned, const double* lam,
                        int64_t rows, double* hhat, double* nsq, double* beta, int* status, double mu_eps,
                        void* bpp_sets, void* ws, size_t ws_bytes, void* stream) {
  return update_dispatch(algo, grams, order, mode, rank, mttkrp_parts, owned, lam, rows, hhat, nsq, beta, status,
                         mu_eps, bpp_sets, m_ld, nullptr, ws, ws_bytes, stream, m_groups, m_gstride);
}

int nncp_update_normalize(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                          double* owned, double* lam, int64_t rows, double* hhat, double* nsq, double* beta,
                          int* status, double mu_eps, void* bpp_sets, int64_t m_ld, double* gram_out, double* gamma_out,
                          int* status_all, int status_count, double* codes, int nslots, int offset, int* masks_out,
                          void* ws, size_t ws_bytes, void* stream) {
  if (rank > 32) return fail(NNCP_ERR_UNSUPPORTED, "the fused normalisation takes rank <= 32");
  if (rows < 1) return fail(NNCP_ERR_VALUE, "the fused normalisation needs rows");
  if (!owned || !lam || !nsq || !gram_out || order < 1) return fail(NNCP_ERR_VALUE, "owned, lam, nsq and gram required");
  if (gamma_out && (!codes || !status_all || status_count < 0 || status_count > kMaxOrder || offset < 0 ||
                    offset + status_count > nslots))
    return fail(NNCP_ERR_VALUE, "bad status hand-off arguments");
  TailArgs t{};
  t.hhat = hhat;
  t.rows = rows;
  t.owned = owned;
  t.lam = lam;
  t.gram = gram_out;
  t.pub = PublishArgs{grams, order, lam, gamma_out, gamma_out ? status_all : nullptr, status_count, codes, nslots,
                      offset, masks_out};
  return update_dispatch(algo, grams, order, mode, rank, mttkrp_rows, owned, lam, rows, hhat, nsq, beta, status, mu_eps,
                         bpp_sets, m_ld, &t, ws, ws_bytes, stream);
}

int nncp_update(int algo, const double* grams, int order, int mode, int rank, const double* mttkrp_rows,
                const double* owned, const double* lam, int64_t rows, double* hhat, double* nsq, double* beta,
                int* status, void* ws, size_t ws_bytes, void* stream) {
  return nncp_update_ex(algo, grams, order, mode, rank, mttkrp_rows, owned, lam, rows, hhat, nsq, beta, status,
                        1e-16, nullptr, 0, ws, ws_bytes, stream);   // MU_EPSILON (updaters.py:27)
}

int nncp_normalize_gram(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned, double* lam,
                        double* gram, void* ws, size_t ws_bytes, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  if (!nsq) return fail(NNCP_ERR_VALUE, "nsq required");
  return normalize_gram(hhat, nsq, rows, rank, owned, lam, gram, ws, ws_bytes, S(stream), 2);
}

int nncp_gram(const double* h, int64_t rows, int rank, double* gram, void* ws, size_t ws_bytes, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  return normalize_gram(h, nullptr, rows, rank, nullptr, nullptr, gram, ws, ws_bytes, S(stream), 3);
}

int nncp_gamma(const double* grams, int order, int rank, const double* lam, double* gamma_out, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  return gamma(grams, order, rank, lam, gamma_out, S(stream));
}

int nncp_normalize_from_gram(const double* hhat, const double* gram_raw, int64_t rows, int rank, double* owned,
                             double* lam, double* gram, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  if (!gram_raw) return fail(NNCP_ERR_VALUE, "raw gram required");
  if (gram == gram_raw) return fail(NNCP_ERR_VALUE, "gram output must not alias the raw gram");
  return normalize_from_gram(hhat, gram_raw, rows, rank, owned, lam, gram, S(stream));
}

int nncp_normalize_gram_publish(const double* hhat, const double* nsq, int64_t rows, int rank, double* owned,
                                double* lam, double* gram, void* ws, size_t ws_bytes, const double* grams, int order,
                                double* gamma_out, int* status, int count, double* codes, int nslots, int offset,
                                int* masks_out, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  if (!nsq || !gram || !grams || !gamma_out || !status || !codes)
    return fail(NNCP_ERR_VALUE, "nsq, gram, grams, gamma, status and codes are required");
  if (count < 0 || count > kMaxOrder) return fail(NNCP_ERR_VALUE, "status count must be in [0, max order]");
  if (offset < 0 || offset + count > nslots) return fail(NNCP_ERR_VALUE, "status slot outside the codes vector");
  return normalize_gram_publish(hhat, nsq, rows, rank, owned, lam, gram, ws, ws_bytes, grams, order, gamma_out, status,
                                count, codes, nslots, offset, masks_out, S(stream));
}

int nncp_gamma_publish(const double* grams, int order, int rank, const double* lam, double* gamma_out, int* status,
                       int count, double* codes, int nslots, int offset, int* masks_out, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  if (!status || !codes) return fail(NNCP_ERR_VALUE, "status and codes buffers required");
  if (count < 0 || count > kMaxOrder) return fail(NNCP_ERR_VALUE, "status count must be in [0, max order]");
  if (offset < 0 || offset + count > nslots) return fail(NNCP_ERR_VALUE, "status slot outside the codes vector");
  return gamma_publish(grams, order, rank, lam, gamma_out, status, count, codes, nslots, offset, masks_out,
                       S(stream));
}

int nncp_inner(const double* a, const double* b, const double* lam, int64_t rows, int rank, double* out, void* ws,
               size_t ws_bytes, void* stream) {
  return inner(a, b, lam, rows, rank, out, ws, ws_bytes, S(stream));
}

static int check_rank_mode(int order, int mode, int rank) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64] on the device path");
  if (order < 0 || order > kMaxOrder) return fail(NNCP_ERR_VALUE, "bad order");
  if (order > 0 && (mode < 0 || mode >= order)) return fail(NNCP_ERR_VALUE, "exclude index out of range");
  return NNCP_OK;
}

int nncp_admm_step(const double* grams, int order, int mode, int rank, double rho, const double* mttkrp_rows,
                   const double* x_in, double* u, double* x_out, int64_t rows, double* sums5, int* status, void* ws,
                   size_t ws_bytes, void* stream) {
  int rc = check_rank_mode(order, mode, rank);
  if (rc) return rc;
  return admm_step(grams, order, mode, rank, rho, mttkrp_rows, x_in, u, x_out, std::max<int64_t>(rows, 0), sums5,
                   status, ws, ws_bytes, S(stream));
}

int nncp_nes_hyper(const double* grams, int order, int mode, int rank, double prox_floor, double* hyper3,
                   void* stream) {
  int rc = check_rank_mode(order, mode, rank);
  if (rc) return rc;
  return nes_hyper(grams, order, mode, rank, prox_floor, hyper3, S(stream));
}

int nncp_nes_step(const double* grams, int order, int mode, int rank, const double* hyper3, const double* mttkrp_rows,
                  const double* y_in, const double* x_in, const double* xstar, double* x_out, double* y_out,
                  int64_t rows, double* maxes2, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_rank_mode(order, mode, rank);
  if (rc) return rc;
  return nes_step(grams, order, mode, rank, hyper3, mttkrp_rows, y_in, x_in, xstar, x_out, y_out,
                  std::max<int64_t>(rows, 0), maxes2, ws, ws_bytes, S(stream));
}

int nncp_scale_columns(const double* in, const double* colscale, int64_t rows, int rank, double* out, void* stream) {
  return scale_columns(in, colscale, rows, rank, out, S(stream));
}

int nncp_extrapolate(const double* cur, const double* prev, int64_t n, double step, double* out, void* stream) {
  return extrapolate(cur, prev, n, step, out, S(stream));
}

int nncp_nes_lambda(const double* cand_lam, const double* nsq, int order, int rank, double* lam, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  return nes_lambda(cand_lam, nsq, order, rank, lam, S(stream));
}

int nncp_colsumsq(const double* h, int64_t rows, int rank, double* nsq, void* ws, size_t ws_bytes, void* stream) {
  if (rank < 1 || rank > kMaxRank) return fail(NNCP_ERR_UNSUPPORTED, "rank must be in [1, 64]");
  return colsumsq(h, std::max<int64_t>(rows, 0), rank, nsq, ws, ws_bytes, S(stream));
}

int nncp_synthetic(double* x, int order, const int64_t* local_dims, const int64_t* offsets,
                   const int64_t* global_dims, const double* const* factors, int rank, double noise_scale,
                   uint64_t seed, void* stream) {
  int rc = check_common(order, local_dims, rank);
  if (rc) return rc;
  return synthetic(x, order, local_dims, offsets, global_dims, factors, rank, noise_scale, seed, S(stream));
}

}  // extern "C"
