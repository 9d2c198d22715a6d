// Internal declarations shared by the libpjds translation units (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "pjds.h"

namespace pjds {

// ---- errors -------------------------------------------------------------------------------
int set_error(int status, const std::string& msg);
inline int ok() { return PJDS_OK; }
#define PJDS_CUDA_TRY(expr)                                                                   \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return ::pjds::set_error(_e == cudaErrorMemoryAllocation ? PJDS_ERR_OOM : PJDS_ERR_CUDA, \
                               std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)
#define PJDS_TRY(expr)          \
  do {                          \
    int _s = (expr);            \
    if (_s != PJDS_OK) return _s; \
  } while (0)

inline size_t dtype_size(int dt) { return dt == PJDS_F64 ? 8 : 4; }

// Makes the handle's device current for the scope of an entry point and restores the caller's
// device afterwards (handles may be used from any current device; launches and allocations must
// land on the device that owns the handle's memory).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev < 0 || cudaGetDevice(&prev) != cudaSuccess) { prev = -1; return; }
    if (prev == dev) prev = -1;
    else cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// ---- host-side pJDS arrays (conversion result) ---------------------------------------------
struct PjdsHost {
  int64_t n = 0, ncols = 0, nnz = 0, n_pad = 0, n_blocks = 0, stored = 0;
  int32_t br = 32, width = 0, dtype = PJDS_F64, len_min = 0, len_max = 0;
  std::vector<int32_t> perm;       // [n]  perm[new] = old
  std::vector<int32_t> block_len;  // [n_blocks]
  std::vector<int64_t> col_start;  // per window: [width_w+1] offsets relative to the window start
  int64_t sigma = 0, n_windows = 0;  // sort scope (rows per window; n_pad = one global window)
  std::vector<int64_t> wstart;     // [n_windows+1] first stored slot of each window
  std::vector<int64_t> wcs_off;    // [n_windows+1] start of each window's col_start in col_start
  std::vector<int32_t> col;        // [stored]
  std::vector<uint8_t> val;        // [stored * dtype_size]
  std::vector<int64_t> hist;       // [len_max+1]
};

// CRS (rows x ncols) -> pJDS host arrays.  `val_src` optional gather index (val[k] = val_in[src[k]]).
// Validates CRS; cols must be < ncols.  symmetric: columns -> invperm[col] (requires ncols == n).
int convert_pjds(PjdsHost& out, int64_t n, int64_t ncols, const int64_t* rowptr, const int32_t* col,
                 const void* val, int dtype, int32_t br, bool symmetric, int64_t sigma = 0);

struct EllrHost {
  int64_t n = 0, nnz = 0, n_pad = 0, stored = 0, idle = 0;
  int32_t width = 0, dtype = PJDS_F64;
  std::vector<int32_t> rowmax, col;
  std::vector<uint8_t> val;
};
int convert_ellr(EllrHost& out, int64_t n, const int64_t* rowptr, const int32_t* col, const void* val,
                 int dtype);

int validate_crs(int64_t n, int64_t ncols, const int64_t* rowptr, const int32_t* col);

}  // namespace pjds

// ---- handles --------------------------------------------------------------------------------
struct pjds_mat {
  pjds::PjdsHost h;  // arrays are cleared (vectors freed) after upload unless host-only
  uint32_t flags = 0;
  bool on_device = false;
  int device = -1;
  void* d_val = nullptr;
  int32_t* d_col = nullptr;
  int64_t* d_col_start = nullptr;  // per window: wstart[w] + col_start_w[j] - w*sigma (kernel view)
  int64_t* d_wcs_off = nullptr;
  int32_t* d_block_len = nullptr;
  int32_t* d_perm = nullptr;  // store target per sorted row (orig row; or local row for A_nl)
  void* d_xs = nullptr;       // staging for pjds_spmv_host
  void* d_ys = nullptr;
  // pipelined host batch (pjds_spmv_host_batch): double-buffered staging, copy streams, events
  void* d_bx[2] = {nullptr, nullptr};
  void* d_by[2] = {nullptr, nullptr};
  void* d_bp[2] = {nullptr, nullptr};  // permuted-basis scratch (x then y) per slot
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_b[9] = {};            // x ready[2], y ready[2], x free[2], y free[2], start
  int64_t ncols = 0;
  bool direct_store = false;  // permuted basis: y[k] stored contiguously, perm not read
  int32_t* d_order[3] = {nullptr, nullptr, nullptr};  // CTA tile execution orders (R = 1, 2, 4)
  int32_t* d_worder[3] = {nullptr, nullptr, nullptr};  // warp-tile (32 R rows) execution orders
  // fused remote-gather dist matrix (PJDS_TRANSPORT_DIRECT): column codes (owner << win_shift) |
  // position; d_win = device table of 64 x-window base pointers (owned by the dist handle)
  void** d_win = nullptr;
  int win_shift = 0;
  unsigned long long* d_sched = nullptr;  // dynamic warp-tile schedule: {next tile, CTAs done}
  // y-store override of the permuted-basis kernel for this handle (-1: the global policy; else
  // 0 plain stores or 1 + L2 policy kind of the vector store), e.g. a dist A_loc whose y the
  // nonlocal pass reads again
  int32_t y_store = -1;
  // no length class holds >= 90 % of the rows (set at upload): the auto tile order then runs the
  // row-only kernels in warp-granular original-row order (mode 3)
  bool mixed_classes = false;
};

struct ellr_mat {
  pjds::EllrHost h;
  uint32_t flags = 0;
  bool on_device = false;
  int device = -1;
  void* d_val = nullptr;
  int32_t* d_col = nullptr;
  int32_t* d_rowmax = nullptr;
};

namespace pjds {
int upload_pjds(pjds_mat* A, const int32_t* store_map /* optional: perm composed with this */);
int free_pjds_device(pjds_mat* A);
int build_tile_orders(pjds_mat* A, const int64_t* row_key = nullptr);

// ---- kernel launchers (kernels.cu) -----------------------------------------------------------
int launch_pjds_spmv(const pjds_mat* A, void* y, const void* x, cudaStream_t s, bool accumulate);
// y = A x (permuted basis) plus per-CTA partials of y.x into part[0 .. *nparts); part must hold
// n_pad / 256 + 1 doubles (the largest grid of any variant)
int launch_pjds_spmv_dot(const pjds_mat* A, void* y, const void* x, cudaStream_t s, double* part, int64_t* nparts);
// P2P transport kernels (p2p.cu)
int p2p_launch_wait(const uint64_t* flags, const int* peers, int np, uint64_t target, unsigned* err, cudaStream_t s);
int p2p_launch_signal(uint64_t* const* targets, int nt, uint64_t value, cudaStream_t s);
int p2p_launch_signal_wait(uint64_t* const* targets, int nt, uint64_t value, const uint64_t* flags, const int* peers,
                           int np, uint64_t target, unsigned* err, cudaStream_t s);
int p2p_launch_pack_put(const void* x, const int* idx, const int64_t* seg, void* const* dst, int npeers,
                        int64_t max_count, int dtype, cudaStream_t s);
int launch_ellr_spmv(const ellr_mat* A, void* y, const void* x, cudaStream_t s);
int launch_permute(const int32_t* perm, int64_t n, const void* src, void* dst, int dtype, int back, cudaStream_t s);
int launch_pack(const int32_t* idx, int64_t count, const void* x, void* buf, int dtype, cudaStream_t s);
int set_kernel_variant(int r, int u);
int set_cache_policy(int stream_kind, int x_kind);
int set_tile_order(int mode);
int set_schedule(int mode);
int set_launch_overlap(int mode, int prefetch_cols);
int bw_probe(int64_t bytes, int reps, double* copy_gbs, double* read_gbs);
int launch_copy16(const void* src, void* dst, size_t bytes, cudaStream_t s);  // bytes % 16 == 0
// devmem.cpp: column indices in generic compressible memory (pjds_set_compression)
int set_compression(int mode);
int dalloc_index(int32_t** dst, const int32_t* src, size_t bytes);
void dev_free(void* p);  // cudaFree, or the VMM release of a compressible allocation
bool is_compressible(const void* p);
void count_launch(int64_t k = 1);
}  // namespace pjds
