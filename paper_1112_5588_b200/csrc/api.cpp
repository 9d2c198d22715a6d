// C ABI of libpjds (include/pjds.h): single-GPU pJDS / ELLPACK-R handles.
#include <algorithm>
#include <cstring>
#include <new>
#include "internal.h"

namespace pjds {

static thread_local std::string g_err;
int set_error(int status, const std::string& msg) {
  g_err = msg;
  return status;
}

template <typename P>
static int dmalloc_copy(P** dst, const void* src, size_t bytes) {
  *dst = nullptr;
  // empty arrays still get a (16-byte, zeroed) allocation so the kernels see a valid pointer;
  // only the `bytes` that exist on the host are copied
  PJDS_CUDA_TRY(cudaMalloc((void**)dst, bytes ? bytes : 16));
  if (!bytes) PJDS_CUDA_TRY(cudaMemset(*dst, 0, 16));
  if (src && bytes) PJDS_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return PJDS_OK;
}

int free_pjds_device(pjds_mat* A) {
  cudaFree(A->d_val); dev_free(A->d_col); cudaFree(A->d_col_start); cudaFree(A->d_block_len);
  dev_free(A->d_perm); cudaFree(A->d_xs); cudaFree(A->d_ys); cudaFree(A->d_wcs_off); cudaFree(A->d_sched);
  A->d_wcs_off = nullptr;
  A->d_sched = nullptr;
  for (int b = 0; b < 2; ++b) {
    cudaFree(A->d_bx[b]); cudaFree(A->d_by[b]); cudaFree(A->d_bp[b]);
    A->d_bx[b] = A->d_by[b] = A->d_bp[b] = nullptr;
  }
  if (A->s_h2d) cudaStreamDestroy(A->s_h2d);
  if (A->s_d2h) cudaStreamDestroy(A->s_d2h);
  A->s_h2d = A->s_d2h = nullptr;
  for (auto& e : A->ev_b) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
  for (auto& o : A->d_order) {
    cudaFree(o);
    o = nullptr;
  }
  for (auto& o : A->d_worder) {
    cudaFree(o);
    o = nullptr;
  }
  A->d_val = A->d_xs = A->d_ys = nullptr;
  A->d_col = A->d_block_len = A->d_perm = nullptr;
  A->d_col_start = nullptr;
  A->on_device = false;
  return PJDS_OK;
}

// Upload the host arrays; the per-row store target is perm[k] (or store_map[perm[k]] when a
// composition is requested, e.g. A_nl rows -> local rows).  Host val/col are released afterwards.
int upload_pjds(pjds_mat* A, const int32_t* store_map) {
  auto& h = A->h;
  PJDS_CUDA_TRY(cudaGetDevice(&A->device));
  std::vector<int32_t> target;
  const int32_t* tp = h.perm.data();
  if (store_map) {
    target.resize(h.n);
    for (int64_t k = 0; k < h.n; ++k) target[k] = store_map[h.perm[k]];
    tp = target.data();
  }
  // kernel view of col_start: per window w, wstart[w] + col_start_w[j] - w * sigma, so that the
  // slot of sorted row k in column j is cs[j] + k for every window
  // (n = 0 has no window: its col_start is the single entry {0})
  std::vector<int64_t> cs_abs(h.col_start.size());
  const bool windowed = h.n_windows >= 1 && (int64_t)h.wcs_off.size() == h.n_windows + 1;
  for (int64_t w = 0; w < (windowed ? h.n_windows : 1); ++w) {
    const int64_t a0 = windowed ? h.wcs_off[w] : 0;
    const int64_t a1 = windowed ? h.wcs_off[w + 1] : (int64_t)cs_abs.size();
    const int64_t add = (windowed ? h.wstart[w] : 0) - w * h.sigma;
    for (int64_t i = a0; i < a1; ++i) cs_abs[i] = h.col_start[i] + add;
  }
  std::vector<int64_t> woff = windowed ? h.wcs_off : std::vector<int64_t>{0, (int64_t)cs_abs.size()};
  int s = PJDS_OK;
  if ((s = dmalloc_copy(&A->d_val, h.val.data(), h.val.size())) ||
      (s = dalloc_index(&A->d_col, h.col.data(), h.col.size() * 4)) ||
      (s = dmalloc_copy(&A->d_col_start, cs_abs.data(), cs_abs.size() * 8)) ||
      (s = dmalloc_copy(&A->d_wcs_off, woff.data(), woff.size() * 8)) ||
      (s = dmalloc_copy(&A->d_block_len, h.block_len.data(), h.block_len.size() * 4)) ||
      (s = dalloc_index(&A->d_perm, tp, (size_t)h.n * 4)) ||
      (s = dmalloc_copy(&A->d_sched, nullptr, 0))) {  // 16 zeroed bytes: the dynamic-schedule counters
    free_pjds_device(A);
    return s;
  }
  {
    int64_t mx = 0;
    for (int64_t c : h.hist) mx = std::max(mx, c);
    A->mixed_classes = h.n > 0 && (double)mx < 0.9 * (double)h.n;
  }
  if ((s = build_tile_orders(A)) != PJDS_OK) {
    free_pjds_device(A);
    return s;
  }
  A->on_device = true;
  std::vector<int32_t>().swap(h.col);
  std::vector<uint8_t>().swap(h.val);
  return PJDS_OK;
}

}  // namespace pjds

using namespace pjds;

extern "C" {

const char* pjds_last_error(void) { return g_err.c_str(); }
const char* pjds_version(void) { return "libpjds 0.1 (sm_100a)"; }

int pjds_create_from_crs_ex(pjds_t* out, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                            int dtype, int32_t block_rows, int64_t sigma, uint32_t flags);

int pjds_create_from_crs(pjds_t* out, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                         int dtype, int32_t block_rows, uint32_t flags) {
  return pjds_create_from_crs_ex(out, n, rowptr, col, val, dtype, block_rows, 0, flags);
}

int pjds_create_from_crs_ex(pjds_t* out, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                            int dtype, int32_t block_rows, int64_t sigma, uint32_t flags) {
  if (!out) return set_error(PJDS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (flags & ~(uint32_t)(PJDS_PERM_SYMMETRIC | PJDS_HOST_ONLY)) return set_error(PJDS_ERR_INVALID_ARG, "unknown flags");
  if (block_rows == 0) block_rows = 32;
  pjds_mat* A = new (std::nothrow) pjds_mat();
  if (!A) return set_error(PJDS_ERR_OOM, "handle allocation failed");
  A->flags = flags;
  int s = convert_pjds(A->h, n, n, rowptr, col, val, dtype, block_rows, flags & PJDS_PERM_SYMMETRIC, sigma);
  if (s == PJDS_OK && !(flags & PJDS_HOST_ONLY)) {
    // permuted basis: y_perm[k] is stored at k; the kernel does not read perm at all
    A->direct_store = flags & PJDS_PERM_SYMMETRIC;
    s = upload_pjds(A, nullptr);
  }
  if (s != PJDS_OK) {
    delete A;
    return s;
  }
  A->ncols = n;
  *out = A;
  return PJDS_OK;
}

int pjds_destroy(pjds_t A) {
  if (!A) return PJDS_OK;
  if (A->on_device) {
    DeviceGuard dg(A->device);
    free_pjds_device(A);
  }
  delete A;
  return PJDS_OK;
}

int pjds_spmv(pjds_t A, void* y, const void* x, void* stream) {
  if (!A || (A->h.n > 0 && (!y || !x))) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv: NULL argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv: handle is host-only");
  if (y == x && A->h.n > 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv: y aliases x");
  DeviceGuard dg(A->device);
  return launch_pjds_spmv(A, y, x, (cudaStream_t)stream, false);
}

int pjds_spmv_accum(pjds_t A, void* y, const void* x, void* stream) {
  if (!A || (A->h.n > 0 && (!y || !x))) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_accum: NULL argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_accum: handle is host-only");
  if (y == x && A->h.n > 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_accum: y aliases x");
  if (A->direct_store)
    return set_error(PJDS_ERR_UNSUPPORTED, "pjds_spmv_accum: permuted-basis (symmetric) handles store y[k] = only");
  DeviceGuard dg(A->device);
  return launch_pjds_spmv(A, y, x, (cudaStream_t)stream, true);
}

// Staging of pjds_spmv_host / pjds_spmv_host_batch is all-or-nothing: on any failure everything
// created so far is released and the pointers are reset, so a later call retries from scratch
// instead of launching on a half-allocated set.
static void free_host_staging(pjds_mat* A) {
  cudaFree(A->d_xs); cudaFree(A->d_ys);
  A->d_xs = A->d_ys = nullptr;
}
static void free_batch_staging(pjds_mat* A) {
  for (int b = 0; b < 2; ++b) {
    cudaFree(A->d_bx[b]); cudaFree(A->d_by[b]); cudaFree(A->d_bp[b]);
    A->d_bx[b] = A->d_by[b] = A->d_bp[b] = nullptr;
  }
  if (A->s_h2d) cudaStreamDestroy(A->s_h2d);
  if (A->s_d2h) cudaStreamDestroy(A->s_d2h);
  A->s_h2d = A->s_d2h = nullptr;
  for (auto& e : A->ev_b) {
    if (e) cudaEventDestroy(e);
    e = nullptr;
  }
}
static int alloc_host_staging(pjds_mat* A, size_t bx, size_t by) {
  if (A->d_xs && A->d_ys) return PJDS_OK;
  free_host_staging(A);
  if (cudaMalloc(&A->d_xs, bx) != cudaSuccess || cudaMalloc(&A->d_ys, by) != cudaSuccess) {
    cudaGetLastError();
    free_host_staging(A);
    return set_error(PJDS_ERR_OOM, "pjds_spmv_host: staging allocation failed");
  }
  return PJDS_OK;
}
static int alloc_batch_staging(pjds_mat* A, size_t bx, size_t by, bool sym) {
  bool ok = true;
  for (int b = 0; b < 2 && ok; ++b) {
    ok = cudaMalloc(&A->d_bx[b], bx) == cudaSuccess && cudaMalloc(&A->d_by[b], by) == cudaSuccess &&
         (!sym || cudaMalloc(&A->d_bp[b], std::max(bx, by)) == cudaSuccess);
  }
  ok = ok && cudaStreamCreateWithFlags(&A->s_h2d, cudaStreamNonBlocking) == cudaSuccess &&
       cudaStreamCreateWithFlags(&A->s_d2h, cudaStreamNonBlocking) == cudaSuccess;
  for (auto& e : A->ev_b) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    free_batch_staging(A);
    return set_error(PJDS_ERR_OOM, "pjds_spmv_host_batch: staging allocation failed");
  }
  return PJDS_OK;
}

int pjds_spmv_host(pjds_t A, void* y_host, const void* x_host, void* stream) {
  if (!A || !y_host || !x_host) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_host: NULL argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_host: handle is host-only");
  const size_t bytes_x = (size_t)A->ncols * dtype_size(A->h.dtype), bytes_y = (size_t)A->h.n * dtype_size(A->h.dtype);
  const bool sym = A->direct_store;
  // symmetric: a second vector each for the basis change, at a 256-byte aligned offset
  const size_t off_x = ((bytes_x ? bytes_x : 16) + 255) & ~size_t(255), off_y = ((bytes_y ? bytes_y : 16) + 255) & ~size_t(255);
  DeviceGuard dg(A->device);
  PJDS_TRY(alloc_host_staging(A, sym ? 2 * off_x : off_x, sym ? 2 * off_y : off_y));
  cudaStream_t s = (cudaStream_t)stream;
  PJDS_CUDA_TRY(cudaMemcpyAsync(A->d_xs, x_host, bytes_x, cudaMemcpyHostToDevice, s));
  if (sym) {  // host vectors are in the ORIGINAL basis: permute once before and once after
    char* xp = (char*)A->d_xs + off_x;
    char* yp = (char*)A->d_ys + off_y;
    PJDS_TRY(launch_permute(A->d_perm, A->h.n, A->d_xs, xp, A->h.dtype, 0, s));
    PJDS_TRY(launch_pjds_spmv(A, yp, xp, s, false));
    PJDS_TRY(launch_permute(A->d_perm, A->h.n, yp, A->d_ys, A->h.dtype, 1, s));
  } else {
    PJDS_TRY(launch_pjds_spmv(A, A->d_ys, A->d_xs, s, false));
  }
  PJDS_CUDA_TRY(cudaMemcpyAsync(y_host, A->d_ys, bytes_y, cudaMemcpyDeviceToHost, s));
  PJDS_CUDA_TRY(cudaStreamSynchronize(s));
  return PJDS_OK;
}

int pjds_spmv_host_batch(pjds_t A, void* const* y_host, const void* const* x_host, int32_t count, void* stream) {
  if (!A || count < 0 || (count > 0 && (!y_host || !x_host)))
    return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_host_batch: bad argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_host_batch: handle is host-only");
  const size_t vs = dtype_size(A->h.dtype);
  const size_t bx = std::max<size_t>((size_t)A->ncols * vs, 16), by = std::max<size_t>((size_t)A->h.n * vs, 16);
  const bool sym = A->direct_store;
  DeviceGuard dg(A->device);
  if (!A->ev_b[8]) PJDS_TRY(alloc_batch_staging(A, bx, by, sym));  // the last object created
  cudaStream_t cs = (cudaStream_t)stream;
  cudaEvent_t *ev_x = A->ev_b, *ev_y = A->ev_b + 2, *ev_xf = A->ev_b + 4, *ev_yf = A->ev_b + 6, ev0 = A->ev_b[8];
  // the copy streams start after everything already queued on the caller's stream
  PJDS_CUDA_TRY(cudaEventRecord(ev0, cs));
  PJDS_CUDA_TRY(cudaStreamWaitEvent(A->s_h2d, ev0, 0));
  PJDS_CUDA_TRY(cudaStreamWaitEvent(A->s_d2h, ev0, 0));
  for (int32_t i = 0; i < count; ++i) {
    const int b = i & 1;
    if (!x_host[i] || !y_host[i]) return set_error(PJDS_ERR_INVALID_ARG, "pjds_spmv_host_batch: NULL vector");
    if (i >= 2) PJDS_CUDA_TRY(cudaStreamWaitEvent(A->s_h2d, ev_xf[b], 0));  // product i-2 done reading
    PJDS_CUDA_TRY(cudaMemcpyAsync(A->d_bx[b], x_host[i], (size_t)A->ncols * vs, cudaMemcpyHostToDevice, A->s_h2d));
    PJDS_CUDA_TRY(cudaEventRecord(ev_x[b], A->s_h2d));
    PJDS_CUDA_TRY(cudaStreamWaitEvent(cs, ev_x[b], 0));
    if (i >= 2) PJDS_CUDA_TRY(cudaStreamWaitEvent(cs, ev_yf[b], 0));  // y of product i-2 copied out
    if (sym) {
      PJDS_TRY(launch_permute(A->d_perm, A->h.n, A->d_bx[b], A->d_bp[b], A->h.dtype, 0, cs));
      PJDS_TRY(launch_pjds_spmv(A, A->d_bx[b], A->d_bp[b], cs, false));  // x slot reused for y_perm
      PJDS_TRY(launch_permute(A->d_perm, A->h.n, A->d_bx[b], A->d_by[b], A->h.dtype, 1, cs));
    } else {
      PJDS_TRY(launch_pjds_spmv(A, A->d_by[b], A->d_bx[b], cs, false));
    }
    PJDS_CUDA_TRY(cudaEventRecord(ev_xf[b], cs));
    PJDS_CUDA_TRY(cudaEventRecord(ev_y[b], cs));
    PJDS_CUDA_TRY(cudaStreamWaitEvent(A->s_d2h, ev_y[b], 0));
    PJDS_CUDA_TRY(cudaMemcpyAsync(y_host[i], A->d_by[b], (size_t)A->h.n * vs, cudaMemcpyDeviceToHost, A->s_d2h));
    PJDS_CUDA_TRY(cudaEventRecord(ev_yf[b], A->s_d2h));
  }
  PJDS_CUDA_TRY(cudaEventRecord(ev0, A->s_d2h));
  PJDS_CUDA_TRY(cudaStreamWaitEvent(cs, ev0, 0));
  PJDS_CUDA_TRY(cudaStreamSynchronize(cs));
  return PJDS_OK;
}

int pjds_permute(pjds_t A, void* dst, const void* src, int32_t direction, void* stream) {
  if (!A || (A->h.n > 0 && (!dst || !src))) return set_error(PJDS_ERR_INVALID_ARG, "pjds_permute: NULL argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_permute: handle is host-only");
  if (dst == src && A->h.n > 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_permute: dst aliases src");
  if (direction != 0 && direction != 1) return set_error(PJDS_ERR_INVALID_ARG, "pjds_permute: direction 0 or 1");
  DeviceGuard dg(A->device);
  return launch_permute(A->d_perm, A->h.n, src, dst, A->h.dtype, direction, (cudaStream_t)stream);
}

int pjds_info(pjds_t A, pjds_info_t* o) {
  if (!A || !o) return set_error(PJDS_ERR_INVALID_ARG, "pjds_info: NULL argument");
  const auto& h = A->h;
  std::memset(o, 0, sizeof(*o));
  o->n = h.n; o->nnz = h.nnz; o->n_pad = h.n_pad; o->n_blocks = h.n_blocks; o->stored = h.stored;
  o->block_rows = h.br; o->width = h.width; o->dtype = h.dtype; o->flags = (int32_t)A->flags;
  o->len_min = h.len_min; o->len_max = h.len_max;
  o->len_mean = h.n ? (double)h.nnz / (double)h.n : 0.0;
  o->useful_fma = h.nnz;
  o->padded_fma = h.stored - h.nnz;
  o->idle_lane_slots = 0;
  o->bytes_values = h.stored * (int64_t)dtype_size(h.dtype);
  o->bytes_indices = h.stored * 4;
  o->bytes_aux = (int64_t)h.col_start.size() * 8 + h.n_blocks * 4 + h.n * 4 +
                 (h.n_windows > 1 ? (h.n_windows + 1) * 16 : 0);
  o->bytes_total = o->bytes_values + o->bytes_indices + o->bytes_aux;
  const int64_t ell = (h.n + 31) / 32 * 32 * (int64_t)h.width;
  o->data_reduction_vs_ellpack = ell ? 1.0 - (double)h.stored / (double)ell : 0.0;
  o->on_device = A->on_device;
  o->device = A->device;
  o->sigma = h.sigma;
  o->n_windows = h.n_windows;
  o->col_start_len = (int64_t)h.col_start.size();
  o->col_compressible = A->on_device && is_compressible(A->d_col);
  return PJDS_OK;
}

int pjds_export_windows(pjds_t A, int64_t* wstart, int64_t* wcs_off) {
  if (!A) return set_error(PJDS_ERR_INVALID_ARG, "pjds_export_windows: NULL handle");
  const auto& h = A->h;
  if (wstart) std::memcpy(wstart, h.wstart.data(), h.wstart.size() * 8);
  if (wcs_off) std::memcpy(wcs_off, h.wcs_off.data(), h.wcs_off.size() * 8);
  return PJDS_OK;
}

int pjds_histogram(pjds_t A, int64_t* counts, int32_t nbins) {
  if (!A || !counts || nbins < 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_histogram: bad argument");
  for (int32_t L = 0; L < nbins; ++L) counts[L] = L < (int32_t)A->h.hist.size() ? A->h.hist[L] : 0;
  return PJDS_OK;
}

int pjds_export(pjds_t A, int32_t* perm, int32_t* block_len, int64_t* col_start, int32_t* col, void* val) {
  if (!A) return set_error(PJDS_ERR_INVALID_ARG, "pjds_export: NULL handle");
  const auto& h = A->h;
  if (perm) std::memcpy(perm, h.perm.data(), (size_t)h.n * 4);
  if (block_len) std::memcpy(block_len, h.block_len.data(), (size_t)h.n_blocks * 4);
  if (col_start) std::memcpy(col_start, h.col_start.data(), h.col_start.size() * 8);
  const size_t vb = (size_t)h.stored * dtype_size(h.dtype);
  if (A->on_device) {
    if (col) PJDS_CUDA_TRY(cudaMemcpy(col, A->d_col, (size_t)h.stored * 4, cudaMemcpyDeviceToHost));
    if (val) PJDS_CUDA_TRY(cudaMemcpy(val, A->d_val, vb, cudaMemcpyDeviceToHost));
  } else {
    if (col) std::memcpy(col, h.col.data(), (size_t)h.stored * 4);
    if (val) std::memcpy(val, h.val.data(), vb);
  }
  return PJDS_OK;
}

// ---- ELLPACK-R ------------------------------------------------------------------------------
int ellr_create_from_crs(ellr_t* out, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                         int dtype, uint32_t flags) {
  if (!out) return set_error(PJDS_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (flags & ~(uint32_t)PJDS_HOST_ONLY) return set_error(PJDS_ERR_INVALID_ARG, "unknown flags");
  ellr_mat* A = new (std::nothrow) ellr_mat();
  if (!A) return set_error(PJDS_ERR_OOM, "handle allocation failed");
  A->flags = flags;
  int s = convert_ellr(A->h, n, rowptr, col, val, dtype);
  if (s == PJDS_OK && !(flags & PJDS_HOST_ONLY)) {
    auto& h = A->h;
    cudaGetDevice(&A->device);
    if ((s = dmalloc_copy(&A->d_val, h.val.data(), h.val.size())) ||
        (s = dalloc_index(&A->d_col, h.col.data(), h.col.size() * 4)) ||
        (s = dalloc_index(&A->d_rowmax, h.rowmax.data(), h.rowmax.size() * 4))) {
      cudaFree(A->d_val); dev_free(A->d_col); dev_free(A->d_rowmax);
    } else {
      A->on_device = true;
      std::vector<int32_t>().swap(h.col);
      std::vector<uint8_t>().swap(h.val);
    }
  }
  if (s != PJDS_OK) {
    delete A;
    return s;
  }
  *out = A;
  return PJDS_OK;
}

int ellr_destroy(ellr_t A) {
  if (!A) return PJDS_OK;
  if (A->on_device) {
    DeviceGuard dg(A->device);
    cudaFree(A->d_val); dev_free(A->d_col); dev_free(A->d_rowmax);
  }
  delete A;
  return PJDS_OK;
}

int ellr_spmv(ellr_t A, void* y, const void* x, void* stream) {
  if (!A || (A->h.n > 0 && (!y || !x))) return set_error(PJDS_ERR_INVALID_ARG, "ellr_spmv: NULL argument");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "ellr_spmv: handle is host-only");
  if (y == x && A->h.n > 0) return set_error(PJDS_ERR_INVALID_ARG, "ellr_spmv: y aliases x");
  DeviceGuard dg(A->device);
  return launch_ellr_spmv(A, y, x, (cudaStream_t)stream);
}

int ellr_info(ellr_t A, ellr_info_t* o) {
  if (!A || !o) return set_error(PJDS_ERR_INVALID_ARG, "ellr_info: NULL argument");
  const auto& h = A->h;
  std::memset(o, 0, sizeof(*o));
  o->n = h.n; o->nnz = h.nnz; o->n_pad = h.n_pad; o->stored = h.stored; o->width = h.width; o->dtype = h.dtype;
  o->useful_fma = h.nnz; o->padded_fma = 0; o->idle_lane_slots = h.idle;
  o->bytes_values = h.stored * (int64_t)dtype_size(h.dtype);
  o->bytes_indices = h.stored * 4;
  o->bytes_aux = h.n_pad * 4;
  o->bytes_total = o->bytes_values + o->bytes_indices + o->bytes_aux;
  o->on_device = A->on_device;
  o->device = A->device;
  o->col_compressible = A->on_device && is_compressible(A->d_col);
  return PJDS_OK;
}

int pjds_footprint(pjds_t A, pjds_footprint_t* o) {
  if (!A || !o) return set_error(PJDS_ERR_INVALID_ARG, "pjds_footprint: NULL argument");
  const auto& h = A->h;
  std::memset(o, 0, sizeof(*o));
  o->bytes_values = h.stored * (int64_t)dtype_size(h.dtype);
  o->bytes_indices = h.stored * 4;
  o->bytes_col_start = (int64_t)h.col_start.size() * 8 + (h.n_windows > 1 ? (h.n_windows + 1) * 16 : 0);
  o->bytes_block_len = h.n_blocks * 4;
  o->bytes_perm = h.n * 4;
  o->bytes_total = o->bytes_values + o->bytes_indices + o->bytes_col_start + o->bytes_block_len + o->bytes_perm;
  o->stored = h.stored; o->nnz = h.nnz; o->n_pad = h.n_pad;
  return PJDS_OK;
}

int pjds_stats(pjds_t A, pjds_stats_t* o) {
  if (!A || !o) return set_error(PJDS_ERR_INVALID_ARG, "pjds_stats: NULL argument");
  pjds_info_t i;
  PJDS_TRY(pjds_info(A, &i));
  std::memset(o, 0, sizeof(*o));
  o->n = i.n; o->nnz = i.nnz; o->n_pad = i.n_pad; o->n_blocks = i.n_blocks; o->padding = i.stored - i.nnz;
  o->width = i.width; o->block_rows = i.block_rows; o->len_min = i.len_min; o->len_max = i.len_max;
  o->len_mean = i.len_mean; o->reduction_vs_ellpack = i.data_reduction_vs_ellpack;
  o->useful_fma = i.useful_fma; o->padded_fma = i.padded_fma; o->idle_lane_slots = i.idle_lane_slots;
  return PJDS_OK;
}

int ellr_footprint(ellr_t A, pjds_footprint_t* o) {
  if (!A || !o) return set_error(PJDS_ERR_INVALID_ARG, "ellr_footprint: NULL argument");
  const auto& h = A->h;
  std::memset(o, 0, sizeof(*o));
  o->bytes_values = h.stored * (int64_t)dtype_size(h.dtype);
  o->bytes_indices = h.stored * 4;
  o->bytes_rowmax = h.n_pad * 4;
  o->bytes_total = o->bytes_values + o->bytes_indices + o->bytes_rowmax;
  o->stored = h.stored; o->nnz = h.nnz; o->n_pad = h.n_pad;
  return PJDS_OK;
}

int ellr_export(ellr_t A, int32_t* rowmax, int32_t* col, void* val) {
  if (!A) return set_error(PJDS_ERR_INVALID_ARG, "ellr_export: NULL handle");
  const auto& h = A->h;
  if (rowmax) std::memcpy(rowmax, h.rowmax.data(), (size_t)h.n_pad * 4);
  const size_t vb = (size_t)h.stored * dtype_size(h.dtype);
  if (A->on_device) {
    if (col) PJDS_CUDA_TRY(cudaMemcpy(col, A->d_col, (size_t)h.stored * 4, cudaMemcpyDeviceToHost));
    if (val) PJDS_CUDA_TRY(cudaMemcpy(val, A->d_val, vb, cudaMemcpyDeviceToHost));
  } else {
    if (col) std::memcpy(col, h.col.data(), (size_t)h.stored * 4);
    if (val) std::memcpy(val, h.val.data(), vb);
  }
  return PJDS_OK;
}

int pjds_set_kernel_variant(int32_t rows_per_thread, int32_t unroll) {
  return set_kernel_variant(rows_per_thread, unroll);
}

int pjds_set_cache_policy(int32_t stream_kind, int32_t x_kind) { return set_cache_policy(stream_kind, x_kind); }

int pjds_set_y_store(pjds_t A, int32_t kind) {
  if (!A) return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_y_store: NULL handle");
  if (kind < -1 || kind > 4) return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_y_store: kind in -1 .. 4");
  A->y_store = kind;
  return PJDS_OK;
}
int pjds_set_tile_order(int32_t mode) { return set_tile_order(mode); }
int pjds_set_schedule(int32_t mode) { return set_schedule(mode); }
int pjds_set_launch_overlap(int32_t mode, int32_t prefetch_cols) { return set_launch_overlap(mode, prefetch_cols); }
int pjds_set_compression(int32_t mode) { return set_compression(mode); }

int pjds_set_tile_keys(pjds_t A, const int64_t* key, int64_t n) {
  if (!A) return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_tile_keys: NULL handle");
  if (!A->on_device) return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_tile_keys: handle is host-only");
  if (key && n != A->h.n) return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_tile_keys: need one key per row");
  DeviceGuard dg(A->device);
  return build_tile_orders(A, key);
}

int pjds_bw_probe(int64_t bytes, int32_t reps, double* copy_gbs, double* read_gbs) {
  if (!copy_gbs || !read_gbs) return set_error(PJDS_ERR_INVALID_ARG, "pjds_bw_probe: NULL argument");
  return bw_probe(bytes, reps, copy_gbs, read_gbs);
}

}  // extern "C"
