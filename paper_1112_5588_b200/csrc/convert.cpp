// Host conversion CRS -> pJDS and CRS -> ELLPACK-R (§2.1).
//
// pJDS steps:
//   a1 len[i] = rowptr[i+1] - rowptr[i]
//   a2 "sort": stable descending counting sort of rows by len (ties: ascending row), perm[new]=old
//   a3 "pad": n_pad = ceil(n/b_r)*b_r; block_len[b] = len of the first (= longest) row of block b
//   a4 col_start[j+1] = col_start[j] + b_r * #{b : block_len[b] > j}
//   a5 fill val/col jagged column-major: slot col_start[j] + k holds entry j of sorted row k
// All steps are O(n + stored) and parallel (OpenMP); the result is independent of the thread
// count (bit-exact, deterministic).
#include <algorithm>
#include <cstring>
#include <new>
#include <omp.h>
#include "internal.h"

namespace pjds {

int validate_crs(int64_t n, int64_t ncols, const int64_t* rowptr, const int32_t* col) {
  if (n < 0 || n >= (int64_t(1) << 31) || ncols < 0 || ncols >= (int64_t(1) << 31))
    return set_error(PJDS_ERR_INVALID_ARG, "n must satisfy 0 <= n < 2^31");
  if (!rowptr) return set_error(PJDS_ERR_INVALID_ARG, "rowptr is NULL");
  if (rowptr[0] != 0) return set_error(PJDS_ERR_BAD_CSR, "rowptr[0] != 0");
  int64_t bad_row = -1;
#pragma omp parallel for reduction(max : bad_row)
  for (int64_t i = 0; i < n; ++i) {
    int64_t l = rowptr[i + 1] - rowptr[i];
    if (l < 0 || l > INT32_MAX) bad_row = std::max(bad_row, i);
  }
  if (bad_row >= 0) return set_error(PJDS_ERR_BAD_CSR, "rowptr decreasing (or row too long) at row " + std::to_string(bad_row));
  int64_t nnz = rowptr[n];
  if (nnz > 0 && !col) return set_error(PJDS_ERR_INVALID_ARG, "col is NULL");
  int64_t bad = -1;
#pragma omp parallel for reduction(max : bad)
  for (int64_t k = 0; k < nnz; ++k)
    if (col[k] < 0 || (int64_t)col[k] >= ncols) bad = std::max(bad, k);
  if (bad >= 0) return set_error(PJDS_ERR_BAD_CSR, "column index out of range at entry " + std::to_string(bad));
  return PJDS_OK;
}

namespace {

// Stable descending counting sort by length.  Rows are split into T contiguous chunks; every
// thread counts its chunk, per-(length, thread) start offsets are a scan over lengths in
// descending order then threads in ascending order, so the placement equals the sequential
// stable sort.
void sort_rows(int64_t n, const int32_t* len, int32_t maxlen, int32_t* perm) {
  int T = omp_get_max_threads();
  if (n < (1 << 16)) T = 1;
  const int64_t L = (int64_t)maxlen + 1;
  std::vector<int64_t> cnt((size_t)T * L, 0);
#pragma omp parallel num_threads(T)
  {
    int t = omp_get_thread_num();
    int64_t a = n * t / T, b = n * (t + 1) / T;
    int64_t* c = &cnt[(size_t)t * L];
    for (int64_t i = a; i < b; ++i) c[len[i]]++;
#pragma omp barrier
#pragma omp single
    {
      int64_t pos = 0;
      for (int64_t l = maxlen; l >= 0; --l)
        for (int tt = 0; tt < T; ++tt) {
          int64_t v = cnt[(size_t)tt * L + l];
          cnt[(size_t)tt * L + l] = pos;
          pos += v;
        }
    }
    for (int64_t i = a; i < b; ++i) perm[c[len[i]]++] = (int32_t)i;
  }
}

}  // namespace

int convert_pjds(PjdsHost& o, int64_t n, int64_t ncols, const int64_t* rowptr, const int32_t* col,
                 const void* val, int dtype, int32_t br, bool symmetric, int64_t sigma) {
  if (dtype != PJDS_F32 && dtype != PJDS_F64) return set_error(PJDS_ERR_INVALID_ARG, "dtype must be PJDS_F32 or PJDS_F64");
  if (br <= 0 || br % 32 != 0) return set_error(PJDS_ERR_INVALID_ARG, "block_rows must be a positive multiple of 32");
  if (sigma < 0 || (sigma > 0 && (sigma % 1024 != 0 || sigma % br != 0)))
    return set_error(PJDS_ERR_INVALID_ARG, "sigma must be 0 (global sort) or a multiple of 1024 and of block_rows");
  if (symmetric && ncols != n) return set_error(PJDS_ERR_INVALID_ARG, "symmetric permutation needs a square matrix");
  PJDS_TRY(validate_crs(n, ncols, rowptr, col));
  const int64_t nnz = rowptr[n];
  if (nnz > 0 && !val) return set_error(PJDS_ERR_INVALID_ARG, "val is NULL");
  const size_t vs = dtype_size(dtype);
  try {
    o = PjdsHost();
    o.n = n; o.ncols = ncols; o.nnz = nnz; o.br = br; o.dtype = dtype;
    // a1 row lengths
    std::vector<int32_t> len(n);
    int32_t mx = 0, mn = n ? INT32_MAX : 0;
#pragma omp parallel for reduction(max : mx) reduction(min : mn)
    for (int64_t i = 0; i < n; ++i) {
      len[i] = (int32_t)(rowptr[i + 1] - rowptr[i]);
      mx = std::max(mx, len[i]);
      mn = std::min(mn, len[i]);
    }
    o.len_max = mx; o.len_min = mn;
    o.hist.assign((size_t)mx + 1, 0);
    for (int64_t i = 0; i < n; ++i) o.hist[len[i]]++;
    // a2 sort (within windows of sigma rows; one window = the paper's global sort)
    o.n_blocks = (n + br - 1) / br;
    o.n_pad = o.n_blocks * br;
    o.sigma = (sigma <= 0 || sigma >= o.n_pad) ? std::max<int64_t>(o.n_pad, br) : sigma;
    o.n_windows = o.n_pad ? (o.n_pad + o.sigma - 1) / o.sigma : 0;
    o.perm.resize(n);
    for (int64_t w = 0; w < o.n_windows; ++w) {
      const int64_t r0 = w * o.sigma, r1 = std::min(n, r0 + o.sigma);
      if (r1 <= r0) continue;
      sort_rows(r1 - r0, len.data() + r0, mx, o.perm.data() + r0);
      if (r0)
        for (int64_t k = r0; k < r1; ++k) o.perm[k] += (int32_t)r0;
    }
    // a3 pad: block_len[b] = length of the first (longest) row of block b in its window
    o.block_len.resize(o.n_blocks);
    for (int64_t b = 0; b < o.n_blocks; ++b) o.block_len[b] = b * br < n ? len[o.perm[b * br]] : 0;
    // a4 col_start per window: nb_gt[j] = #blocks of the window with block_len > j (non-increasing)
    o.wstart.assign(o.n_windows + 1, 0);
    o.wcs_off.assign(o.n_windows + 1, 0);
    o.col_start.clear();
    o.width = 0;
    const int64_t bpw = o.sigma / br;  // blocks per window
    for (int64_t w = 0; w < o.n_windows; ++w) {
      const int64_t b0 = w * bpw, b1 = std::min(o.n_blocks, b0 + bpw);
      const int32_t ww = b1 > b0 ? o.block_len[b0] : 0;
      o.width = std::max(o.width, ww);
      std::vector<int64_t> nb_at((size_t)ww + 2, 0);
      for (int64_t b = b0; b < b1; ++b) nb_at[o.block_len[b]]++;
      const size_t base = o.col_start.size();
      o.col_start.resize(base + ww + 1, 0);
      int64_t gt = (b1 - b0) - nb_at[0];
      for (int32_t j = 0; j < ww; ++j) {
        o.col_start[base + j + 1] = o.col_start[base + j] + (int64_t)br * gt;
        gt -= nb_at[j + 1];
      }
      o.wcs_off[w + 1] = (int64_t)o.col_start.size();
      o.wstart[w + 1] = o.wstart[w] + o.col_start[base + ww];
    }
    if (o.n_windows == 0) o.col_start.assign(1, 0);
    o.stored = o.wstart[o.n_windows];
    // a5 fill
    o.col.assign(o.stored, 0);
    o.val.assign((size_t)o.stored * vs, 0);  // +0.0 bit pattern for padding
    std::vector<int32_t> inv;
    if (symmetric) {
      inv.resize(n);
#pragma omp parallel for
      for (int64_t k = 0; k < n; ++k) inv[o.perm[k]] = (int32_t)k;
    }
    int32_t* oc = o.col.data();
    uint8_t* ov = o.val.data();
    const uint8_t* iv = (const uint8_t*)val;
    const int64_t sg = o.sigma;
#pragma omp parallel for schedule(static, 1024)
    for (int64_t k = 0; k < n; ++k) {
      const int64_t w = k / sg;
      const int64_t* cs = o.col_start.data() + o.wcs_off[w];
      const int64_t kk = o.wstart[w] + (k - w * sg);  // slot of row k in jagged column 0 of its window
      const int64_t r = o.perm[k];
      const int64_t base = rowptr[r];
      const int32_t l = len[r];
      for (int32_t j = 0; j < l; ++j) {
        const int64_t dst = cs[j] + kk;
        const int32_t c = col[base + j];
        oc[dst] = symmetric ? inv[c] : c;
        std::memcpy(ov + dst * vs, iv + (base + j) * vs, vs);
      }
    }
  } catch (const std::bad_alloc&) {
    return set_error(PJDS_ERR_OOM, "host allocation failed during pJDS conversion");
  }
  return PJDS_OK;
}

int convert_ellr(EllrHost& o, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val, int dtype) {
  if (dtype != PJDS_F32 && dtype != PJDS_F64) return set_error(PJDS_ERR_INVALID_ARG, "dtype must be PJDS_F32 or PJDS_F64");
  PJDS_TRY(validate_crs(n, n, rowptr, col));
  const int64_t nnz = rowptr[n];
  if (nnz > 0 && !val) return set_error(PJDS_ERR_INVALID_ARG, "val is NULL");
  const size_t vs = dtype_size(dtype);
  try {
    o = EllrHost();
    o.n = n; o.nnz = nnz; o.dtype = dtype;
    o.n_pad = (n + 31) / 32 * 32;  // footnote PAPER.md L153-155
    int32_t mx = 0;
#pragma omp parallel for reduction(max : mx)
    for (int64_t i = 0; i < n; ++i) mx = std::max(mx, (int32_t)(rowptr[i + 1] - rowptr[i]));
    o.width = mx;
    o.stored = o.n_pad * (int64_t)mx;
    o.rowmax.assign(o.n_pad, 0);
    o.col.assign(o.stored, 0);
    o.val.assign((size_t)o.stored * vs, 0);
    int64_t idle = 0;
    const int64_t NP = o.n_pad;
#pragma omp parallel for reduction(+ : idle) schedule(static)
    for (int64_t w = 0; w < NP / 32; ++w) {
      int32_t wmax = 0;
      for (int64_t i = w * 32; i < w * 32 + 32; ++i) {
        int32_t l = i < n ? (int32_t)(rowptr[i + 1] - rowptr[i]) : 0;
        o.rowmax[i] = l;
        wmax = std::max(wmax, l);
        for (int32_t j = 0; j < l; ++j) {
          o.col[j * NP + i] = col[rowptr[i] + j];
          std::memcpy(&o.val[(size_t)(j * NP + i) * vs], (const uint8_t*)val + (rowptr[i] + j) * vs, vs);
        }
      }
      for (int64_t i = w * 32; i < w * 32 + 32; ++i) idle += wmax - o.rowmax[i];
    }
    o.idle = idle;
  } catch (const std::bad_alloc&) {
    return set_error(PJDS_ERR_OOM, "host allocation failed during ELLPACK-R conversion");
  }
  return PJDS_OK;
}

}  // namespace pjds
