// Row-partitioned distributed spMVM (§3) over NCCL point-to-point.
//
//   plan    : split of this rank's rows into a local part (owned columns) and a nonlocal part
//             (columns owned by other ranks); recv lists per owner
//             (sorted unique global ids) and halo slots (position in the owner-ordered
//             concatenation).
//   create  : A_loc (all rows, local column ids) and A_nl (rows with >= 1 nonlocal entry,
//             halo-slot column ids) as pJDS; send schedule from the caller-exchanged lists.
//             A peer's list whose entries form at most kMaxRuns contiguous runs is sent straight
//             from x (one message per run, no pack); otherwise it is packed ("local gather",
//             Fig. 4 caption L401-402) into a contiguous buffer by a kernel.  Sender and receiver
//             apply the same rule to the same list, so message boundaries always match.
//   spmv    : task mode (L454-461) with a CUDA stream as the dedicated communication context:
//               comm stream (high priority): [pack] -> ncclGroupStart/Send/Recv/ncclGroupEnd
//               compute stream             : A_loc kernel (y = ...)      -- overlapped
//               compute stream             : wait(comm) -> A_nl kernel (y += ..., written twice, L445)
//             PJDS_NO_OVERLAP serialises everything on the compute stream (vector mode, L437-440).
//   DIRECT  : (PJDS_TRANSPORT_DIRECT) no exchange step at all: ONE pJDS matrix over the full local
//             rows whose nonlocal columns address the owners' x windows (CUDA-IPC mapped peer
//             memory; NVLink loads between GPUs).  One kernel runs every row's whole chain, the
//             remote gathers overlapping the local val/col stream tile by tile; flags order
//             "owner's x ready" -> kernel -> "reader done" (end barrier: x may be rewritten after).
#include <algorithm>
#include <cstring>
#include <dlfcn.h>
#include <mutex>
#include <new>
#include <omp.h>
#include "internal.h"
#include "nccl.h"

using namespace pjds;

struct pjds_plan {
  int32_t R = 1, rank = 0;
  int64_t n_global = 0, lo = 0, hi = 0, n_loc = 0, nnz_loc = 0;
  std::vector<int64_t> offsets;
  std::vector<int64_t> loc_rowptr, loc_src;  // local part: CRS with local column ids
  std::vector<int32_t> loc_col;
  std::vector<int64_t> nl_rowptr, nl_src;    // nonlocal part: CRS with halo-slot column ids
  std::vector<int32_t> nl_col, rows_nl;
  std::vector<int64_t> recv_counts;          // [R]
  std::vector<int32_t> recv_cols;            // [halo] global ids, owner-ordered
};

namespace {

constexpr int kMaxRuns = 64;
// sort scope of the nonlocal part A_nl (rows per window; 0 = the global sort), see dist create
int64_t g_nl_sigma = 1024;

// ---- NCCL (dlopen) ------------------------------------------------------------------------
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};
Nccl g_nccl;
std::mutex g_nccl_mu;

int nccl_load(const char* path) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return PJDS_OK;
  const char* names[] = {path, "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    if (!nm) continue;
    h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) return set_error(PJDS_ERR_NCCL, std::string("cannot dlopen NCCL: ") + dlerror());
  Nccl n;
  n.h = h;
#define SYM(field, name)                                                            \
  n.field = (decltype(n.field))dlsym(h, name);                                      \
  if (!n.field) return set_error(PJDS_ERR_NCCL, std::string("NCCL symbol missing: ") + name);
  SYM(getUniqueId, "ncclGetUniqueId");
  SYM(commInitRank, "ncclCommInitRank");
  SYM(commDestroy, "ncclCommDestroy");
  SYM(send, "ncclSend");
  SYM(recv, "ncclRecv");
  SYM(groupStart, "ncclGroupStart");
  SYM(groupEnd, "ncclGroupEnd");
  SYM(errStr, "ncclGetErrorString");
#undef SYM
  g_nccl = n;
  return PJDS_OK;
}

#define NCCL_TRY(expr)                                                                        \
  do {                                                                                        \
    ncclResult_t _r = (expr);                                                                 \
    if (_r != ncclSuccess) return set_error(PJDS_ERR_NCCL, std::string(#expr) + ": " + g_nccl.errStr(_r)); \
  } while (0)

ncclDataType_t nccl_type(int dt) { return dt == PJDS_F64 ? ncclFloat64 : ncclFloat32; }

// runs of consecutive values in ids[0..m)
std::vector<std::pair<int64_t, int64_t>> runs_of(const int32_t* ids, int64_t m) {
  std::vector<std::pair<int64_t, int64_t>> r;  // (first value, length)
  for (int64_t i = 0; i < m;) {
    int64_t j = i + 1;
    while (j < m && ids[j] == ids[j - 1] + 1) ++j;
    r.push_back({ids[i], j - i});
    i = j;
  }
  return r;
}

}  // namespace

struct pjds_dist {
  int32_t R = 1, rank = 0, transport = PJDS_TRANSPORT_NCCL, dtype = PJDS_F64, device = 0;
  int64_t n_loc = 0, halo = 0, send_total = 0, packed_total = 0;
  int64_t nnz_loc_part = 0, nnz_nl_part = 0, rows_nl = 0;
  pjds_mat* A_loc = nullptr;
  pjds_mat* A_nl = nullptr;
  // send side
  struct PeerSend {
    int32_t peer;
    bool packed;
    std::vector<std::pair<int64_t, int64_t>> runs;  // direct: (x_loc offset, count); packed: one (packbuf offset, count)
  };
  std::vector<PeerSend> sends;
  std::vector<int32_t> pack_idx_host;  // local ids for the pack kernel
  int32_t* d_pack_idx = nullptr;
  void* d_packbuf = nullptr;
  // recv side
  struct PeerRecv {
    int32_t peer;
    std::vector<std::pair<int64_t, int64_t>> runs;  // (halo offset, count), one per message
  };
  std::vector<PeerRecv> recvs;
  std::vector<int64_t> recv_counts;
  void* d_halo = nullptr;
  // streams / events
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_comm = nullptr;
  // phase timing (PJDS_TRACE): 0 start, 1 comm start, 2 pack end, 3 comm end, 4 local end,
  // 5 nonlocal start (after the wait), 6 end
  cudaEvent_t tev[7] = {};
  bool traced = false;
  ncclComm_t nccl = nullptr;
  int send_messages = 0, recv_messages = 0;
  bool permuted = false;
  // ---- P2P transport (p2p.cu): IPC-exported region [halo0 | halo1 | ready[R] | done[R] | err]
  char* p2p_region = nullptr;
  size_t p2p_halo_bytes = 0, p2p_region_bytes = 0;
  std::vector<int64_t> recv_off;               // my halo offset (entries) of each owner's segment
  std::vector<int32_t> send_peers, recv_peers;  // peers I send to / receive from (ascending rank)
  int32_t* d_p2p_idx = nullptr;                 // send ids of all send peers, concatenated
  int64_t* d_p2p_seg = nullptr;                 // [send_peers+1] segment starts
  int64_t p2p_max_count = 0;
  int32_t* d_send_peers = nullptr;              // for the done-wait
  int32_t* d_recv_peers = nullptr;              // for the ready-wait
  void** d_dst[2] = {nullptr, nullptr};         // per buffer parity: destination pointer per send peer
  uint64_t** d_ready_targets = nullptr;         // ready[rank] slot in each receiver's region
  uint64_t** d_done_targets = nullptr;          // done[rank] slot in each sender's region
  std::vector<void*> peer_regions;              // opened IPC mappings
  bool p2p_connected = false;
  uint64_t seq = 0;
  size_t p2p_flags_off = 0;                     // byte offset of ready[R] in the exported region
  // ---- DIRECT transport: region = [x window | ready[R] | done[R] | err]
  int32_t win_shift = 0;
  void** d_win = nullptr;                       // [kWinTable] x-window base per owner rank
  std::vector<int32_t> dir_send_pos;            // my window position of every send entry (send order)
  bool dir_cols_encoded = false;                // column codes rewritten (connect is not retryable after)
  std::vector<int64_t> offsets;                 // row offsets [R+1]
  uint64_t* ready_flags() const { return (uint64_t*)(p2p_region + p2p_flags_off); }
  uint64_t* done_flags() const { return ready_flags() + R; }
  // timeout word of the bounded peer waits: pinned, mapped host memory, so that every
  // pjds_dist_spmv call can see a timeout of an earlier call without a device synchronisation
  unsigned* h_err = nullptr;
  unsigned* d_h_err = nullptr;                  // device alias of h_err
  unsigned* err_flag() const { return d_h_err; }
};

namespace {

size_t vsz(const pjds_dist* D) { return dtype_size(D->dtype); }

// Enqueue this rank's sends and receives (NCCL transport) on `s`.
int post_nccl(pjds_dist* D, const void* x_loc, cudaStream_t s) {
  const size_t vs = vsz(D);
  NCCL_TRY(g_nccl.groupStart());
  ncclResult_t r = ncclSuccess;
  for (auto& ps : D->sends) {
    const char* base = ps.packed ? (const char*)D->d_packbuf : (const char*)x_loc;
    for (auto& run : ps.runs)
      if (r == ncclSuccess)
        r = g_nccl.send(base + run.first * vs, (size_t)run.second, nccl_type(D->dtype), ps.peer, D->nccl, s);
  }
  for (auto& pr : D->recvs)
    for (auto& run : pr.runs)
      if (r == ncclSuccess)
        r = g_nccl.recv((char*)D->d_halo + run.first * vs, (size_t)run.second, nccl_type(D->dtype), pr.peer, D->nccl, s);
  const ncclResult_t e = g_nccl.groupEnd();  // the group is closed even when a post failed
  if (r != ncclSuccess) return set_error(PJDS_ERR_NCCL, std::string("ncclSend/ncclRecv: ") + g_nccl.errStr(r));
  if (e != ncclSuccess) return set_error(PJDS_ERR_NCCL, std::string("ncclGroupEnd: ") + g_nccl.errStr(e));
  return PJDS_OK;
}

static int alloc_err_word(pjds_dist* D) {
  if (D->h_err) return PJDS_OK;
  PJDS_CUDA_TRY(cudaHostAlloc((void**)&D->h_err, 64, cudaHostAllocMapped));
  *(volatile unsigned*)D->h_err = 0;
  PJDS_CUDA_TRY(cudaHostGetDevicePointer((void**)&D->d_h_err, D->h_err, 0));
  return PJDS_OK;
}

// P2P transport: allocate the IPC-exported region and the per-call device tables.
int p2p_setup(pjds_dist* D, const std::vector<int32_t>& ids, const std::vector<int64_t>& seg) {
  const size_t vs = vsz(D);
  D->p2p_halo_bytes = (std::max<size_t>(D->halo * vs, 16) + 255) / 256 * 256;
  D->p2p_region_bytes = 2 * D->p2p_halo_bytes + 2 * (size_t)D->R * 8 + 256;
  D->p2p_flags_off = 2 * D->p2p_halo_bytes;
  PJDS_TRY(alloc_err_word(D));
  PJDS_CUDA_TRY(cudaMalloc(&D->p2p_region, D->p2p_region_bytes));
  PJDS_CUDA_TRY(cudaMemset(D->p2p_region, 0, D->p2p_region_bytes));
  const size_t ns = D->send_peers.size(), nr = D->recv_peers.size();
  PJDS_CUDA_TRY(cudaMalloc(&D->d_p2p_idx, std::max<size_t>(ids.size(), 1) * 4));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_p2p_seg, seg.size() * 8));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_send_peers, std::max<size_t>(ns, 1) * 4));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_recv_peers, std::max<size_t>(nr, 1) * 4));
  for (auto& d : D->d_dst) PJDS_CUDA_TRY(cudaMalloc(&d, std::max<size_t>(ns, 1) * sizeof(void*)));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_ready_targets, std::max<size_t>(ns, 1) * sizeof(void*)));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_done_targets, std::max<size_t>(nr, 1) * sizeof(void*)));
  if (!ids.empty()) PJDS_CUDA_TRY(cudaMemcpy(D->d_p2p_idx, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice));
  PJDS_CUDA_TRY(cudaMemcpy(D->d_p2p_seg, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice));
  if (ns) PJDS_CUDA_TRY(cudaMemcpy(D->d_send_peers, D->send_peers.data(), ns * 4, cudaMemcpyHostToDevice));
  if (nr) PJDS_CUDA_TRY(cudaMemcpy(D->d_recv_peers, D->recv_peers.data(), nr * 4, cudaMemcpyHostToDevice));
  D->peer_regions.assign(D->R, nullptr);
  return PJDS_OK;
}

constexpr int kWinTable = 64;  // = kMaxWin of the window kernel (kernels.cu)

// DIRECT transport: the IPC-exported x window + flags, the window-base table, the flag tables.
int direct_setup(pjds_dist* D) {
  const size_t vs = vsz(D);
  const size_t win = (std::max<size_t>(D->n_loc * vs, 16) + 255) / 256 * 256;
  D->p2p_flags_off = win;
  D->p2p_region_bytes = win + 2 * (size_t)D->R * 8 + 256;
  PJDS_TRY(alloc_err_word(D));
  PJDS_CUDA_TRY(cudaMalloc(&D->p2p_region, D->p2p_region_bytes));
  PJDS_CUDA_TRY(cudaMemset(D->p2p_region, 0, D->p2p_region_bytes));
  const size_t ns = D->send_peers.size(), nr = D->recv_peers.size();
  PJDS_CUDA_TRY(cudaMalloc(&D->d_send_peers, std::max<size_t>(ns, 1) * 4));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_recv_peers, std::max<size_t>(nr, 1) * 4));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_ready_targets, std::max<size_t>(ns, 1) * sizeof(void*)));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_done_targets, std::max<size_t>(nr, 1) * sizeof(void*)));
  PJDS_CUDA_TRY(cudaMalloc(&D->d_win, kWinTable * sizeof(void*)));
  PJDS_CUDA_TRY(cudaMemset(D->d_win, 0, kWinTable * sizeof(void*)));
  if (ns) PJDS_CUDA_TRY(cudaMemcpy(D->d_send_peers, D->send_peers.data(), ns * 4, cudaMemcpyHostToDevice));
  if (nr) PJDS_CUDA_TRY(cudaMemcpy(D->d_recv_peers, D->recv_peers.data(), nr * 4, cudaMemcpyHostToDevice));
  D->peer_regions.assign(D->R, nullptr);
  return PJDS_OK;
}

// Fixed-size blob each rank publishes: IPC handle of its region plus its halo layout.
constexpr int kP2PMaxRanks = 64;
struct P2PBlob {
  cudaIpcMemHandle_t handle;
  uint64_t halo_bytes;
  uint64_t flags_off;
  int32_t R, rank;
  int64_t recv_off[kP2PMaxRanks];
};

}  // namespace

extern "C" {

int pjds_nccl_load(const char* libpath) { return nccl_load(libpath); }

int pjds_set_dist_nl_sigma(int64_t sigma) {
  if (sigma < 0 || (sigma > 0 && sigma % 1024 != 0))
    return set_error(PJDS_ERR_INVALID_ARG, "pjds_set_dist_nl_sigma: 0 or a multiple of 1024");
  g_nl_sigma = sigma;
  return PJDS_OK;
}

int pjds_nccl_unique_id(void* out128) {
  if (!out128) return set_error(PJDS_ERR_INVALID_ARG, "pjds_nccl_unique_id: NULL");
  PJDS_TRY(nccl_load(nullptr));
  ncclUniqueId id;
  NCCL_TRY(g_nccl.getUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return PJDS_OK;
}

int pjds_dist_plan(pjds_plan_t* out, int32_t R, int32_t rank, int64_t n_global, const int64_t* offs,
                   const int64_t* rowptr, const int32_t* col) {
  if (!out || !offs || !rowptr) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_plan: NULL argument");
  *out = nullptr;
  if (R < 1 || rank < 0 || rank >= R) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_plan: bad nranks/rank");
  if (offs[0] != 0 || offs[R] != n_global) return set_error(PJDS_ERR_INVALID_ARG, "row_offsets must span [0, n_global]");
  for (int q = 0; q < R; ++q)
    if (offs[q + 1] < offs[q]) return set_error(PJDS_ERR_INVALID_ARG, "row_offsets must be non-decreasing");
  const int64_t lo = offs[rank], hi = offs[rank + 1], nl = hi - lo;
  PJDS_TRY(validate_crs(nl, n_global, rowptr, col));
  pjds_plan* P = new (std::nothrow) pjds_plan();
  if (!P) return set_error(PJDS_ERR_OOM, "plan allocation failed");
  try {
    P->R = R; P->rank = rank; P->n_global = n_global; P->lo = lo; P->hi = hi; P->n_loc = nl;
    P->offsets.assign(offs, offs + R + 1);
    const int64_t nnz = rowptr[nl];
    P->nnz_loc = nnz;
    // mark remote columns, then the owner-ordered sorted unique list == ascending global ids
    std::vector<uint8_t> mark(n_global, 0);
#pragma omp parallel for
    for (int64_t k = 0; k < nnz; ++k) {
      int64_t c = col[k];
      if (c < lo || c >= hi) mark[c] = 1;
    }
    for (int64_t c = 0; c < n_global; ++c)
      if (mark[c]) P->recv_cols.push_back((int32_t)c);
    P->recv_counts.assign(R, 0);
    for (int32_t c : P->recv_cols) {
      int q = (int)(std::upper_bound(offs, offs + R + 1, (int64_t)c) - offs) - 1;
      P->recv_counts[q]++;
    }
    // split rows
    std::vector<int32_t> loc_len(nl), nl_len(nl);
#pragma omp parallel for
    for (int64_t i = 0; i < nl; ++i) {
      int32_t a = 0, b = 0;
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
        if (col[k] >= lo && col[k] < hi) ++a;
        else ++b;
      }
      loc_len[i] = a;
      nl_len[i] = b;
    }
    P->loc_rowptr.assign(nl + 1, 0);
    for (int64_t i = 0; i < nl; ++i) {
      P->loc_rowptr[i + 1] = P->loc_rowptr[i] + loc_len[i];
      if (nl_len[i]) P->rows_nl.push_back((int32_t)i);
    }
    const int64_t m = (int64_t)P->rows_nl.size();
    P->nl_rowptr.assign(m + 1, 0);
    for (int64_t a = 0; a < m; ++a) P->nl_rowptr[a + 1] = P->nl_rowptr[a] + nl_len[P->rows_nl[a]];
    P->loc_col.resize(P->loc_rowptr[nl]);
    P->loc_src.resize(P->loc_rowptr[nl]);
    P->nl_col.resize(P->nl_rowptr[m]);
    P->nl_src.resize(P->nl_rowptr[m]);
    std::vector<int64_t> nl_pos(nl, -1);
    for (int64_t a = 0; a < m; ++a) nl_pos[P->rows_nl[a]] = P->nl_rowptr[a];
    const int32_t* rc = P->recv_cols.data();
    const int64_t h = (int64_t)P->recv_cols.size();
#pragma omp parallel for
    for (int64_t i = 0; i < nl; ++i) {
      int64_t pl = P->loc_rowptr[i], pn = nl_pos[i];
      for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
        const int32_t c = col[k];
        if (c >= lo && c < hi) {
          P->loc_col[pl] = (int32_t)(c - lo);
          P->loc_src[pl++] = k;
        } else {
          P->nl_col[pn] = (int32_t)(std::lower_bound(rc, rc + h, c) - rc);
          P->nl_src[pn++] = k;
        }
      }
    }
  } catch (const std::bad_alloc&) {
    delete P;
    return set_error(PJDS_ERR_OOM, "host allocation failed in pjds_dist_plan");
  }
  *out = P;
  return PJDS_OK;
}

int pjds_dist_plan_info(pjds_plan_t P, pjds_plan_info_t* o) {
  if (!P || !o) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_plan_info: NULL argument");
  std::memset(o, 0, sizeof(*o));
  o->n_loc = P->n_loc; o->nnz_loc = P->nnz_loc;
  o->nnz_local_part = (int64_t)P->loc_col.size();
  o->nnz_nonlocal_part = (int64_t)P->nl_col.size();
  o->rows_nonlocal = (int64_t)P->rows_nl.size();
  o->halo = (int64_t)P->recv_cols.size();
  o->nranks = P->R; o->rank = P->rank;
  return PJDS_OK;
}

int pjds_dist_plan_recv(pjds_plan_t P, int64_t* counts, int32_t* cols) {
  if (!P) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_plan_recv: NULL plan");
  if (counts) std::memcpy(counts, P->recv_counts.data(), P->recv_counts.size() * 8);
  if (cols) std::memcpy(cols, P->recv_cols.data(), P->recv_cols.size() * 4);
  return PJDS_OK;
}

int pjds_dist_plan_destroy(pjds_plan_t P) {
  delete P;
  return PJDS_OK;
}

int pjds_dist_destroy(pjds_dist_t D);

static int dist_create_impl(pjds_dist_t* out, pjds_plan_t P, const void* val, int dtype, int32_t block_rows,
                            const int64_t* send_counts, const int32_t* send_cols, int32_t transport,
                            const void* nccl_id, uint32_t flags, ncclComm_t comm_in);

int pjds_dist_create(pjds_dist_t* out, pjds_plan_t P, const void* val, int dtype, int32_t block_rows,
                     const int64_t* send_counts, const int32_t* send_cols, int32_t transport, const void* nccl_id,
                     uint32_t flags) {
  return dist_create_impl(out, P, val, dtype, block_rows, send_counts, send_cols, transport, nccl_id, flags, nullptr);
}

// One-call collective create (SURVEY §8(b) signature): NCCL communicator from the unique id, the
// plan, the recv-list -> send-list exchange over that communicator (counts, then ids, as grouped
// point-to-point messages), then the same create as the three-step path on the same communicator.
int pjds_dist_create_crs(pjds_dist_t* out, const void* nccl_id, int32_t nranks, int32_t rank, int64_t n_global,
                         const int64_t* row_offsets, const int64_t* rowptr_loc, const int32_t* col_global_loc,
                         const void* val_loc, int dtype, int32_t block_rows, uint32_t flags) {
  if (!out) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_create_crs: out is NULL");
  *out = nullptr;
  if (nranks > 1 && !nccl_id) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_create_crs: nccl_unique_id is NULL");
  pjds_plan_t P = nullptr;
  PJDS_TRY(pjds_dist_plan(&P, nranks, rank, n_global, row_offsets, rowptr_loc, col_global_loc));
  ncclComm_t comm = nullptr;
  cudaStream_t st = nullptr;
  int64_t* d_cnt = nullptr;  // [2R]: recv counts out, send counts in
  int32_t* d_ids = nullptr;  // [halo + send_total]
  std::vector<int64_t> sc(nranks, 0);
  std::vector<int32_t> scols;
  bool in_group = false;  // a failure between ncclGroupStart and ncclGroupEnd still closes the group
  auto cleanup = [&](int status) {
    if (in_group) g_nccl.groupEnd();
    if (st) cudaStreamDestroy(st);
    cudaFree(d_cnt);
    cudaFree(d_ids);
    if (status != PJDS_OK && comm) g_nccl.commDestroy(comm);
    pjds_dist_plan_destroy(P);
    return status;
  };
  if (nranks > 1) {
    int s = nccl_load(nullptr);
    if (s != PJDS_OK) return cleanup(s);
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = g_nccl.commInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
      comm = nullptr;
      return cleanup(set_error(PJDS_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.errStr(r)));
    }
    const int R = nranks;
    const int64_t halo = (int64_t)P->recv_cols.size();
    auto nccl_fail = [&](ncclResult_t rr, const char* what) {
      return cleanup(set_error(PJDS_ERR_NCCL, std::string(what) + ": " + g_nccl.errStr(rr)));
    };
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&d_cnt, 2 * R * 8) != cudaSuccess ||
        cudaMemcpy(d_cnt, P->recv_counts.data(), R * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return cleanup(set_error(PJDS_ERR_CUDA, "pjds_dist_create_crs: count buffers"));
    // 1. counts: my recv count from q goes to q, q's recv count from me comes back as my send count
    ncclResult_t rr;
    if ((rr = g_nccl.groupStart()) != ncclSuccess) return nccl_fail(rr, "ncclGroupStart");
    in_group = true;
    for (int q = 0; q < R; ++q) {
      if (q == rank) continue;
      if ((rr = g_nccl.send(d_cnt + q, 1, ncclInt64, q, comm, st)) != ncclSuccess) return nccl_fail(rr, "ncclSend");
      if ((rr = g_nccl.recv(d_cnt + R + q, 1, ncclInt64, q, comm, st)) != ncclSuccess) return nccl_fail(rr, "ncclRecv");
    }
    in_group = false;
    if ((rr = g_nccl.groupEnd()) != ncclSuccess) return nccl_fail(rr, "ncclGroupEnd");
    if (cudaStreamSynchronize(st) != cudaSuccess ||
        cudaMemcpy(sc.data(), d_cnt + R, R * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      return cleanup(set_error(PJDS_ERR_CUDA, "pjds_dist_create_crs: count exchange"));
    sc[rank] = 0;
    int64_t send_total = 0;
    for (int q = 0; q < R; ++q) {
      if (sc[q] < 0) return cleanup(set_error(PJDS_ERR_NCCL, "pjds_dist_create_crs: negative count received"));
      send_total += sc[q];
    }
    // 2. ids: my recv list from q goes to q and becomes q's send list to me
    if (cudaMalloc(&d_ids, std::max<int64_t>(halo + send_total, 1) * 4) != cudaSuccess ||
        (halo && cudaMemcpy(d_ids, P->recv_cols.data(), halo * 4, cudaMemcpyHostToDevice) != cudaSuccess))
      return cleanup(set_error(PJDS_ERR_OOM, "pjds_dist_create_crs: id buffers"));
    if ((rr = g_nccl.groupStart()) != ncclSuccess) return nccl_fail(rr, "ncclGroupStart");
    in_group = true;
    int64_t ro = 0, so = halo;
    for (int q = 0; q < R; ++q) {
      const int64_t rc = P->recv_counts[q];
      if (rc && (rr = g_nccl.send(d_ids + ro, (size_t)rc, ncclInt32, q, comm, st)) != ncclSuccess)
        return nccl_fail(rr, "ncclSend");
      if (sc[q] && (rr = g_nccl.recv(d_ids + so, (size_t)sc[q], ncclInt32, q, comm, st)) != ncclSuccess)
        return nccl_fail(rr, "ncclRecv");
      ro += rc;
      so += sc[q];
    }
    in_group = false;
    if ((rr = g_nccl.groupEnd()) != ncclSuccess) return nccl_fail(rr, "ncclGroupEnd");
    scols.resize(send_total);
    if (cudaStreamSynchronize(st) != cudaSuccess ||
        (send_total && cudaMemcpy(scols.data(), d_ids + halo, send_total * 4, cudaMemcpyDeviceToHost) != cudaSuccess))
      return cleanup(set_error(PJDS_ERR_CUDA, "pjds_dist_create_crs: id exchange"));
  }
  const int s = dist_create_impl(out, P, val_loc, dtype, block_rows, sc.data(), scols.data(), PJDS_TRANSPORT_NCCL,
                                 nullptr, flags, comm);
  comm = nullptr;  // dist_create_impl took ownership (and destroyed it on failure)
  return cleanup(s);
}

static int dist_create_impl(pjds_dist_t* out, pjds_plan_t P, const void* val, int dtype, int32_t block_rows,
                            const int64_t* send_counts, const int32_t* send_cols, int32_t transport,
                            const void* nccl_id, uint32_t flags, ncclComm_t comm_in) {
  // comm_in (optional): an NCCL communicator this call takes ownership of, also on failure
  auto drop_comm = [&](int st) {
    if (comm_in) g_nccl.commDestroy(comm_in);
    return st;
  };
  if (!out || !P) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_create: NULL argument"));
  *out = nullptr;
  if (flags & ~(uint32_t)PJDS_PERM_SYMMETRIC) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_create: unknown flags"));
  const bool sym = flags & PJDS_PERM_SYMMETRIC;
  if (dtype != PJDS_F32 && dtype != PJDS_F64) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "bad dtype"));
  if (transport != PJDS_TRANSPORT_NCCL && transport != PJDS_TRANSPORT_LOCAL && transport != PJDS_TRANSPORT_P2P &&
      transport != PJDS_TRANSPORT_DIRECT)
    return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "bad transport"));
  if (P->nnz_loc > 0 && !val) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "val is NULL"));
  if (P->R > 1 && !send_counts) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "send_counts is NULL"));
  if (block_rows == 0) block_rows = 32;
  const int R = P->R;
  int64_t send_total = 0;
  for (int q = 0; q < R && send_counts; ++q) {
    if (send_counts[q] < 0) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "negative send count"));
    if (q == P->rank && send_counts[q] != 0) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "send to self"));
    send_total += send_counts[q];
  }
  if (send_total > 0 && !send_cols) return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "send_cols is NULL"));
  for (int64_t i = 0; i < send_total; ++i)
    if (send_cols[i] < P->lo || send_cols[i] >= P->hi)
      return drop_comm(set_error(PJDS_ERR_INVALID_ARG, "send_cols entry not owned by this rank"));

  pjds_dist* D = new (std::nothrow) pjds_dist();
  if (!D) return drop_comm(set_error(PJDS_ERR_OOM, "dist allocation failed"));
  D->nccl = comm_in;  // owned by the handle from here on (pjds_dist_destroy releases it)
  comm_in = nullptr;
  D->R = R; D->rank = P->rank; D->transport = transport; D->dtype = dtype;
  D->n_loc = P->n_loc; D->halo = (int64_t)P->recv_cols.size(); D->send_total = send_total;
  D->nnz_loc_part = (int64_t)P->loc_col.size(); D->nnz_nl_part = (int64_t)P->nl_col.size();
  D->rows_nl = (int64_t)P->rows_nl.size();
  D->recv_counts = P->recv_counts;
  D->offsets = P->offsets;
  cudaGetDevice(&D->device);
  const size_t vs = dtype_size(dtype);
  int s = PJDS_OK;
  auto fail = [&](int st) { pjds_dist_destroy(D); return st; };
  std::vector<int32_t> p2p_ids;
  std::vector<int64_t> p2p_seg;
  try {
    std::vector<int32_t> inv;  // local inverse permutation (permuted basis: row i at position inv[i])
    if (transport == PJDS_TRANSPORT_DIRECT) {
      // ---- one pJDS matrix over the full local rows (CRS order kept within each row); columns
      // stay temporary codes until pjds_dist_direct_connect knows the owners' window positions:
      // local column c -> c, halo slot h -> n_loc + h
      int shift = 0;
      int64_t maxn = 1;
      for (int q = 0; q < R; ++q) maxn = std::max(maxn, P->offsets[q + 1] - P->offsets[q]);
      while ((int64_t(1) << shift) < maxn) ++shift;
      if (R > kWinTable || ((int64_t)R << shift) > (int64_t(1) << 31))
        return fail(set_error(PJDS_ERR_UNSUPPORTED, "DIRECT transport: needs nranks <= 64 and "
                                                    "nranks * 2^ceil(log2(max rows per rank)) <= 2^31"));
      D->win_shift = shift;
      const int64_t nl = P->n_loc;
      std::vector<int64_t> frp(nl + 1, 0);
      std::vector<int32_t> nl_len(nl, 0);
      for (int64_t a = 0; a < (int64_t)P->rows_nl.size(); ++a)
        nl_len[P->rows_nl[a]] = (int32_t)(P->nl_rowptr[a + 1] - P->nl_rowptr[a]);
      for (int64_t i = 0; i < nl; ++i) frp[i + 1] = frp[i] + (P->loc_rowptr[i + 1] - P->loc_rowptr[i]) + nl_len[i];
      std::vector<int32_t> fcol(P->nnz_loc);
      for (size_t k = 0; k < P->loc_src.size(); ++k) fcol[P->loc_src[k]] = P->loc_col[k];
      for (size_t k = 0; k < P->nl_src.size(); ++k) fcol[P->nl_src[k]] = (int32_t)(nl + P->nl_col[k]);
      D->A_loc = new pjds_mat();
      s = convert_pjds(D->A_loc->h, nl, nl + D->halo, frp.data(), fcol.data(), val, dtype, block_rows, false);
      if (s != PJDS_OK) return fail(s);
      if (sym) {
        inv.resize(nl);
        for (int64_t k = 0; k < nl; ++k) inv[D->A_loc->h.perm[k]] = (int32_t)k;
        D->A_loc->direct_store = true;
        D->A_loc->flags = PJDS_PERM_SYMMETRIC;
      }
      D->A_loc->ncols = nl + D->halo;
    } else {
      // ---- the two pJDS parts
      std::vector<uint8_t> v_loc(P->loc_src.size() * vs), v_nl(P->nl_src.size() * vs);
      const uint8_t* vin = (const uint8_t*)val;
      for (size_t k = 0; k < P->loc_src.size(); ++k) std::memcpy(&v_loc[k * vs], vin + P->loc_src[k] * vs, vs);
      for (size_t k = 0; k < P->nl_src.size(); ++k) std::memcpy(&v_nl[k * vs], vin + P->nl_src[k] * vs, vs);
      D->A_loc = new pjds_mat();
      s = convert_pjds(D->A_loc->h, P->n_loc, P->n_loc, P->loc_rowptr.data(), P->loc_col.data(), v_loc.data(), dtype,
                       block_rows, sym);
      if (s != PJDS_OK) return fail(s);  // (perm is not filled on failure)
      // local inverse permutation (permuted basis: local row i lives at position inv[i])
      if (sym) {
        inv.resize(P->n_loc);
        for (int64_t k = 0; k < P->n_loc; ++k) inv[D->A_loc->h.perm[k]] = (int32_t)k;
        D->A_loc->direct_store = true;
        D->A_loc->flags = PJDS_PERM_SYMMETRIC;
      }
      if ((s = upload_pjds(D->A_loc, nullptr)) != PJDS_OK) return fail(s);
      D->A_loc->ncols = P->n_loc;
      const int64_t m = (int64_t)P->rows_nl.size();
      if (m > 0) {
        D->A_nl = new pjds_mat();
        // store target of each nonlocal row: its local row (or its position in the local permuted
        // basis).  The nonlocal rows are taken in ascending TARGET order and sorted by length only
        // inside windows of g_nl_sigma rows (one CTA tile each), so the y += of one CTA touches one
        // compact range of y instead of scattered 8-byte read-modify-writes.  Each row's chain
        // (its nonlocal entries in CRS order) is unchanged, so y is bitwise the same.
        std::vector<int32_t> map(P->rows_nl);
        if (sym)
          for (auto& r : map) r = inv[r];
        const int64_t nlsig = (g_nl_sigma > 0 && g_nl_sigma % 1024 == 0 && g_nl_sigma % block_rows == 0) ? g_nl_sigma : 0;
        std::vector<int64_t> ord(m);
        for (int64_t a = 0; a < m; ++a) ord[a] = a;
        if (nlsig && sym)
          std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return map[x] < map[y]; });
        std::vector<int64_t> orp(m + 1, 0);
        for (int64_t a = 0; a < m; ++a) orp[a + 1] = orp[a] + (P->nl_rowptr[ord[a] + 1] - P->nl_rowptr[ord[a]]);
        std::vector<int32_t> ocol(orp[m]), omap(m);
        std::vector<uint8_t> oval(orp[m] * vs);
        for (int64_t a = 0; a < m; ++a) {
          const int64_t r = ord[a], b0 = P->nl_rowptr[r], cnt = P->nl_rowptr[r + 1] - b0;
          std::memcpy(&ocol[orp[a]], &P->nl_col[b0], cnt * 4);
          std::memcpy(&oval[orp[a] * vs], &v_nl[b0 * vs], cnt * vs);
          omap[a] = map[r];
        }
        s = convert_pjds(D->A_nl->h, m, std::max<int64_t>(D->halo, 1), orp.data(), ocol.data(), oval.data(), dtype,
                         block_rows, false, nlsig);
        if (s == PJDS_OK) s = upload_pjds(D->A_nl, omap.data());
        if (s != PJDS_OK) return fail(s);
        D->A_nl->ncols = D->halo;
      }
    }
    D->permuted = sym;
    // ---- send schedule
    int64_t pos = 0;
    p2p_seg.push_back(0);
    for (int q = 0; q < R && send_counts; ++q) {
      const int64_t cnt = send_counts[q];
      if (!cnt) continue;
      std::vector<int32_t> ids(cnt);
      for (int64_t i = 0; i < cnt; ++i) ids[i] = (int32_t)(send_cols[pos + i] - P->lo);
      if (sym)
        for (auto& v : ids) v = inv[v];  // gather from x in the local permuted basis
      pos += cnt;
      if (transport == PJDS_TRANSPORT_DIRECT) {  // q reads these window positions itself
        D->dir_send_pos.insert(D->dir_send_pos.end(), ids.begin(), ids.end());
        D->send_peers.push_back(q);
        pjds_dist::PeerSend ps;
        ps.peer = q;
        ps.packed = false;
        ps.runs = {{0, cnt}};
        D->sends.push_back(std::move(ps));
        continue;
      }
      if (transport == PJDS_TRANSPORT_P2P) {  // every entry is gathered by the fused pack+put kernel
        p2p_ids.insert(p2p_ids.end(), ids.begin(), ids.end());
        p2p_seg.push_back((int64_t)p2p_ids.size());
        D->send_peers.push_back(q);
        D->p2p_max_count = std::max(D->p2p_max_count, cnt);
      }
      auto runs = runs_of(ids.data(), cnt);
      pjds_dist::PeerSend ps;
      ps.peer = q;
      if (!sym && (int)runs.size() <= kMaxRuns) {
        ps.packed = false;
        ps.runs = runs;
      } else {
        ps.packed = true;
        ps.runs = {{D->packed_total, cnt}};
        D->pack_idx_host.insert(D->pack_idx_host.end(), ids.begin(), ids.end());
        D->packed_total += cnt;
      }
      D->send_messages += (int)ps.runs.size();
      D->sends.push_back(std::move(ps));
    }
    // ---- recv schedule (same run rule on the same lists)
    int64_t hoff = 0;
    D->recv_off.assign(R, 0);
    for (int q = 0; q < R; ++q) {
      D->recv_off[q] = hoff;
      const int64_t cnt = P->recv_counts[q];
      if (!cnt) continue;
      D->recv_peers.push_back(q);
      auto runs = runs_of(P->recv_cols.data() + hoff, cnt);
      pjds_dist::PeerRecv pr;
      pr.peer = q;
      if (transport == PJDS_TRANSPORT_DIRECT) {  // no messages: read in place from q's window
        pr.runs = {{hoff, cnt}};
        D->recvs.push_back(std::move(pr));
        hoff += cnt;
        continue;
      }
      if (!sym && (int)runs.size() <= kMaxRuns) {  // permuted basis: one packed message per peer
        int64_t o = hoff;
        for (auto& r : runs) {
          pr.runs.push_back({o, r.second});
          o += r.second;
        }
      } else {
        pr.runs = {{hoff, cnt}};
      }
      D->recv_messages += (int)pr.runs.size();
      D->recvs.push_back(std::move(pr));
      hoff += cnt;
    }
  } catch (const std::bad_alloc&) {
    return fail(set_error(PJDS_ERR_OOM, "host allocation failed in pjds_dist_create"));
  }
  // ---- device buffers, streams, transport
  if (transport == PJDS_TRANSPORT_P2P) {
    if ((s = p2p_setup(D, p2p_ids, p2p_seg)) != PJDS_OK) return fail(s);
  } else if (transport == PJDS_TRANSPORT_DIRECT) {
    if ((s = direct_setup(D)) != PJDS_OK) return fail(s);
  } else if (cudaMalloc(&D->d_halo, std::max<size_t>(D->halo * vs, 16)) != cudaSuccess) {
    return fail(set_error(PJDS_ERR_OOM, "halo allocation failed"));
  }
  if (D->packed_total && transport != PJDS_TRANSPORT_P2P) {
    if (cudaMalloc(&D->d_packbuf, D->packed_total * vs) != cudaSuccess ||
        cudaMalloc(&D->d_pack_idx, D->packed_total * 4) != cudaSuccess)
      return fail(set_error(PJDS_ERR_OOM, "pack buffer allocation failed"));
    if (cudaMemcpy(D->d_pack_idx, D->pack_idx_host.data(), D->packed_total * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_error(PJDS_ERR_CUDA, "pack index upload failed"));
  }
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  if (cudaStreamCreateWithPriority(&D->comm, cudaStreamNonBlocking, hi_prio) != cudaSuccess ||
      cudaEventCreateWithFlags(&D->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&D->ev_comm, cudaEventDisableTiming) != cudaSuccess)
    return fail(set_error(PJDS_ERR_CUDA, "stream/event creation failed"));
  if (transport == PJDS_TRANSPORT_NCCL && R > 1 && !D->nccl) {
    if (!nccl_id) return fail(set_error(PJDS_ERR_INVALID_ARG, "nccl_unique_id is NULL"));
    if ((s = nccl_load(nullptr)) != PJDS_OK) return fail(s);
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = g_nccl.commInitRank(&D->nccl, R, id, P->rank);
    if (r != ncclSuccess) return fail(set_error(PJDS_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.errStr(r)));
  }
  *out = D;
  return PJDS_OK;
}

int pjds_dist_destroy(pjds_dist_t D) {
  if (!D) return PJDS_OK;
  if (D->nccl && g_nccl.commDestroy) g_nccl.commDestroy(D->nccl);
  if (D->comm) cudaStreamDestroy(D->comm);
  if (D->ev_ready) cudaEventDestroy(D->ev_ready);
  if (D->ev_comm) cudaEventDestroy(D->ev_comm);
  for (auto e : D->tev)
    if (e) cudaEventDestroy(e);
  cudaFree(D->d_halo); cudaFree(D->d_packbuf); cudaFree(D->d_pack_idx);
  for (void* p : D->peer_regions)
    if (p) cudaIpcCloseMemHandle(p);
  cudaFree(D->p2p_region); cudaFree(D->d_p2p_idx); cudaFree(D->d_p2p_seg);
  cudaFree(D->d_send_peers); cudaFree(D->d_recv_peers);
  cudaFree(D->d_dst[0]); cudaFree(D->d_dst[1]); cudaFree(D->d_ready_targets); cudaFree(D->d_done_targets);
  cudaFree(D->d_win);
  if (D->h_err) cudaFreeHost(D->h_err);
  D->h_err = D->d_h_err = nullptr;
  pjds_destroy(D->A_loc);
  pjds_destroy(D->A_nl);
  delete D;
  return PJDS_OK;
}

int pjds_dist_p2p_export(pjds_dist_t D, void* blob, int64_t* bytes) {
  if (!D || !bytes) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_export: NULL argument");
  if (D->transport != PJDS_TRANSPORT_P2P && D->transport != PJDS_TRANSPORT_DIRECT)
    return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_export: not a P2P / DIRECT handle");
  if (D->R > kP2PMaxRanks) return set_error(PJDS_ERR_UNSUPPORTED, "P2P transport supports at most 64 ranks");
  *bytes = (int64_t)sizeof(P2PBlob);
  if (!blob) return PJDS_OK;
  P2PBlob b;
  std::memset(&b, 0, sizeof(b));
  PJDS_CUDA_TRY(cudaIpcGetMemHandle(&b.handle, D->p2p_region));
  b.halo_bytes = D->p2p_halo_bytes;
  b.flags_off = D->p2p_flags_off;
  b.R = D->R;
  b.rank = D->rank;
  for (int q = 0; q < D->R; ++q) b.recv_off[q] = D->recv_off[q];
  std::memcpy(blob, &b, sizeof(b));
  return PJDS_OK;
}

int pjds_dist_p2p_connect(pjds_dist_t D, const void* blobs, int64_t blob_bytes) {
  if (!D || !blobs) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_connect: NULL argument");
  if (D->transport != PJDS_TRANSPORT_P2P) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_connect: not a P2P handle");
  if (blob_bytes != (int64_t)sizeof(P2PBlob)) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_connect: blob size");
  const P2PBlob* b = (const P2PBlob*)blobs;
  for (int q = 0; q < D->R; ++q)
    if (b[q].R != D->R || b[q].rank != q) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_connect: blobs not rank-ordered");
  auto open = [&](int q) -> int {
    if (D->peer_regions[q]) return PJDS_OK;
    if (q == D->rank) {
      D->peer_regions[q] = nullptr;
      return PJDS_OK;
    }
    void* p = nullptr;
    PJDS_CUDA_TRY(cudaIpcOpenMemHandle(&p, b[q].handle, cudaIpcMemLazyEnablePeerAccess));
    D->peer_regions[q] = p;
    return PJDS_OK;
  };
  const size_t vs = vsz(D);
  std::vector<void*> dst0, dst1;
  std::vector<uint64_t*> ready_t, done_t;
  for (int q : D->send_peers) {  // my data goes to q's halo at q's offset for owner = me
    PJDS_TRY(open(q));
    char* base = (char*)D->peer_regions[q];
    const size_t off = (size_t)b[q].recv_off[D->rank] * vs;
    dst0.push_back(base + off);
    dst1.push_back(base + b[q].halo_bytes + off);
    ready_t.push_back((uint64_t*)(base + b[q].flags_off) + D->rank);
  }
  for (int p : D->recv_peers) {  // tell p when I am done reading its data
    PJDS_TRY(open(p));
    char* base = (char*)D->peer_regions[p];
    done_t.push_back((uint64_t*)(base + b[p].flags_off) + D->R + D->rank);
  }
  if (!dst0.empty()) {
    PJDS_CUDA_TRY(cudaMemcpy(D->d_dst[0], dst0.data(), dst0.size() * sizeof(void*), cudaMemcpyHostToDevice));
    PJDS_CUDA_TRY(cudaMemcpy(D->d_dst[1], dst1.data(), dst1.size() * sizeof(void*), cudaMemcpyHostToDevice));
    PJDS_CUDA_TRY(cudaMemcpy(D->d_ready_targets, ready_t.data(), ready_t.size() * sizeof(void*), cudaMemcpyHostToDevice));
  }
  if (!done_t.empty())
    PJDS_CUDA_TRY(cudaMemcpy(D->d_done_targets, done_t.data(), done_t.size() * sizeof(void*), cudaMemcpyHostToDevice));
  D->p2p_connected = true;
  return PJDS_OK;
}

int pjds_dist_x_window(pjds_dist_t D, void** x_window) {
  if (!D || !x_window) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_x_window: NULL argument");
  if (D->transport != PJDS_TRANSPORT_DIRECT) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_x_window: not a DIRECT handle");
  *x_window = D->p2p_region;
  return PJDS_OK;
}

int pjds_dist_direct_positions(pjds_dist_t D, int32_t* pos) {
  if (!D) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_positions: NULL handle");
  if (D->transport != PJDS_TRANSPORT_DIRECT) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_positions: not a DIRECT handle");
  if (!D->dir_send_pos.empty()) {
    if (!pos) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_positions: NULL pos");
    std::memcpy(pos, D->dir_send_pos.data(), D->dir_send_pos.size() * 4);
  }
  return PJDS_OK;
}

int pjds_dist_direct_connect(pjds_dist_t D, const int32_t* halo_pos, const void* blobs, int64_t blob_bytes) {
  if (!D || !blobs) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: NULL argument");
  if (D->transport != PJDS_TRANSPORT_DIRECT) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: not a DIRECT handle");
  if (D->p2p_connected) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: already connected");
  if (D->dir_cols_encoded) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: an earlier connect failed after "
                                                                 "rewriting the columns; destroy the handle");
  if (D->halo > 0 && !halo_pos) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: NULL halo_pos");
  if (blob_bytes != (int64_t)sizeof(P2PBlob)) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: blob size");
  const P2PBlob* b = (const P2PBlob*)blobs;
  for (int q = 0; q < D->R; ++q)
    if (b[q].R != D->R || b[q].rank != q) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: blobs not rank-ordered");
  // halo slot -> owner; every position must lie inside the owner's window
  std::vector<int32_t> owner(D->halo);
  for (int q = 0, h = 0; q < D->R; ++q)
    for (int64_t i = 0; i < D->recv_counts[q]; ++i, ++h) {
      owner[h] = q;
      if (halo_pos[h] < 0 || halo_pos[h] >= D->offsets[q + 1] - D->offsets[q])
        return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_direct_connect: halo position outside the owner's rows");
    }
  auto open = [&](int q) -> int {
    if (q == D->rank || D->peer_regions[q]) return PJDS_OK;
    void* p = nullptr;
    PJDS_CUDA_TRY(cudaIpcOpenMemHandle(&p, b[q].handle, cudaIpcMemLazyEnablePeerAccess));
    D->peer_regions[q] = p;
    return PJDS_OK;
  };
  std::vector<void*> bases(kWinTable, nullptr);
  std::vector<uint64_t*> ready_t, done_t;
  bases[D->rank] = D->p2p_region;
  for (int q : D->send_peers) {  // q reads my window: tell q when it holds this call's x
    PJDS_TRY(open(q));
    ready_t.push_back((uint64_t*)((char*)D->peer_regions[q] + b[q].flags_off) + D->rank);
  }
  for (int p : D->recv_peers) {  // I read p's window: tell p when I am done with it
    PJDS_TRY(open(p));
    bases[p] = D->peer_regions[p];
    done_t.push_back((uint64_t*)((char*)D->peer_regions[p] + b[p].flags_off) + D->R + D->rank);
  }
  PJDS_CUDA_TRY(cudaMemcpy(D->d_win, bases.data(), kWinTable * sizeof(void*), cudaMemcpyHostToDevice));
  if (!ready_t.empty())
    PJDS_CUDA_TRY(cudaMemcpy(D->d_ready_targets, ready_t.data(), ready_t.size() * sizeof(void*), cudaMemcpyHostToDevice));
  if (!done_t.empty())
    PJDS_CUDA_TRY(cudaMemcpy(D->d_done_targets, done_t.data(), done_t.size() * sizeof(void*), cudaMemcpyHostToDevice));
  // final column codes (owner << shift) | window position, then upload
  pjds_mat* A = D->A_loc;
  auto& h = A->h;
  const int64_t nl = D->n_loc;
  const int sh = D->win_shift;
  std::vector<int32_t> inv(nl);
  for (int64_t k = 0; k < nl; ++k) inv[h.perm[k]] = D->permuted ? (int32_t)k : h.perm[k];
  const int32_t me = D->rank << sh;
  D->dir_cols_encoded = true;
#pragma omp parallel for
  for (int64_t k = 0; k < (int64_t)h.col.size(); ++k) {
    const int32_t c = h.col[k];
    if (c < nl) {
      h.col[k] = me | inv[c];
    } else {
      const int64_t hs = c - nl;
      h.col[k] = (owner[hs] << sh) | halo_pos[hs];
    }
  }
  int s = upload_pjds(A, nullptr);
  if (s != PJDS_OK) return s;
  A->d_win = D->d_win;
  A->win_shift = sh;
  D->p2p_connected = true;
  return PJDS_OK;
}

int pjds_dist_p2p_check(pjds_dist_t D, int32_t* timed_out) {
  if (!D || !timed_out) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_p2p_check: NULL argument");
  if (D->transport != PJDS_TRANSPORT_P2P && D->transport != PJDS_TRANSPORT_DIRECT) {
    *timed_out = 0;
    return PJDS_OK;
  }
  // every wait enqueued so far has finished (or given up) before the word is read; reading it
  // clears it, so a caller that has handled a timeout can continue
  PJDS_CUDA_TRY(cudaDeviceSynchronize());
  volatile unsigned* w = D->h_err;
  *timed_out = w ? (int32_t)*w : 0;
  if (w) *w = 0;
  return PJDS_OK;
}

int pjds_dist_info(pjds_dist_t D, pjds_dist_info_t* o) {
  if (!D || !o) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_info: NULL argument");
  std::memset(o, 0, sizeof(*o));
  o->n_loc = D->n_loc; o->halo = D->halo; o->send_total = D->send_total; o->packed_send = D->packed_total;
  o->rows_nonlocal = D->rows_nl; o->nnz_local_part = D->nnz_loc_part; o->nnz_nonlocal_part = D->nnz_nl_part;
  o->nranks = D->R; o->rank = D->rank;
  o->peers_send = (int32_t)D->sends.size(); o->peers_recv = (int32_t)D->recvs.size();
  o->send_messages = D->send_messages; o->recv_messages = D->recv_messages;
  o->permuted = D->permuted;
  return PJDS_OK;
}

int pjds_dist_stats(pjds_dist_t D, pjds_dist_info_t* o, int64_t* recv_per_peer, int64_t* send_per_peer) {
  if (!D) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_stats: NULL handle");
  if (o) PJDS_TRY(pjds_dist_info(D, o));
  if (recv_per_peer) {
    for (int q = 0; q < D->R; ++q) recv_per_peer[q] = 0;
    for (const auto& r : D->recvs)
      for (const auto& run : r.runs) recv_per_peer[r.peer] += run.second;
  }
  if (send_per_peer) {
    for (int q = 0; q < D->R; ++q) send_per_peer[q] = 0;
    for (const auto& sd : D->sends)
      for (const auto& run : sd.runs) send_per_peer[sd.peer] += run.second;
  }
  return PJDS_OK;
}

int pjds_dist_permute(pjds_dist_t D, void* dst, const void* src, int32_t direction, void* stream) {
  if (!D) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_permute: NULL handle");
  return pjds_permute(D->A_loc, dst, src, direction, stream);
}

int pjds_dist_parts(pjds_dist_t D, pjds_t* a, pjds_t* b) {
  if (!D) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_parts: NULL");
  if (a) *a = D->A_loc;
  if (b) *b = D->A_nl;
  return PJDS_OK;
}

int pjds_dist_spmv(pjds_dist_t D, void* y, const void* x, void* stream, uint32_t flags) {
  if (!D || (D->n_loc > 0 && (!y || !x))) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_spmv: NULL argument");
  if (y == x && D->n_loc > 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_spmv: y aliases x");
  if (D->transport == PJDS_TRANSPORT_LOCAL) return set_error(PJDS_ERR_INVALID_ARG, "use pjds_dist_group_spmv for LOCAL transport");
  cudaStream_t s = (cudaStream_t)stream;
  if (D->h_err && *(volatile unsigned*)D->h_err)
    return set_error(PJDS_ERR_CUDA, "pjds_dist_spmv: a bounded peer wait of an earlier call timed out (its y is "
                                    "invalid); pjds_dist_p2p_check reports and clears it");
  const bool comm_needed = D->R > 1 && (!D->sends.empty() || !D->recvs.empty());
  const bool tr = flags & PJDS_TRACE;
  if (tr && !D->tev[0])
    for (auto& e : D->tev) PJDS_CUDA_TRY(cudaEventCreate(&e));
  auto mark = [&](int i, cudaStream_t st) -> int {
    if (tr) PJDS_CUDA_TRY(cudaEventRecord(D->tev[i], st));
    return PJDS_OK;
  };
  if (D->transport == PJDS_TRANSPORT_DIRECT) {
    // x into this rank's window (skipped when the caller computed it there), "ready" to the
    // ranks that read it, wait for the owners I read, ONE kernel over all local rows, then
    // "done" to the owners and wait until every reader of my window is done (x reusable after)
    if (!D->p2p_connected) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_spmv: call pjds_dist_direct_connect first");
    if (y == (void*)D->p2p_region && D->n_loc > 0) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_spmv: y aliases the x window");
    const uint64_t sq = ++D->seq;
    const int ns = (int)D->send_peers.size(), nr = (int)D->recv_peers.size();
    PJDS_TRY(mark(0, s));
    PJDS_TRY(mark(1, s));
    if (x != (const void*)D->p2p_region && D->n_loc > 0)
      PJDS_CUDA_TRY(cudaMemcpyAsync(D->p2p_region, x, D->n_loc * vsz(D), cudaMemcpyDeviceToDevice, s));
    PJDS_TRY(mark(2, s));
    PJDS_TRY(p2p_launch_signal_wait(D->d_ready_targets, ns, sq, D->ready_flags(), D->d_recv_peers, nr, sq,
                                    D->err_flag(), s));
    PJDS_TRY(mark(3, s));
    PJDS_TRY(launch_pjds_spmv(D->A_loc, y, D->p2p_region, s, false));
    PJDS_TRY(mark(4, s));
    PJDS_TRY(mark(5, s));
    PJDS_TRY(p2p_launch_signal_wait(D->d_done_targets, nr, sq, D->done_flags(), D->d_send_peers, ns, sq,
                                    D->err_flag(), s));
    PJDS_TRY(mark(6, s));
    D->traced = D->traced || tr;
    return PJDS_OK;
  }
  if (!comm_needed) {  // R = 1 or no halo: local part only (+ empty nonlocal)
    for (int i = 0; i < 4; ++i) PJDS_TRY(mark(i, s));
    PJDS_TRY(launch_pjds_spmv(D->A_loc, y, x, s, false));
    for (int i = 4; i < 7; ++i) PJDS_TRY(mark(i, s));
    D->traced = D->traced || tr;
    return PJDS_OK;
  }
  if (D->transport == PJDS_TRANSPORT_P2P) {
    // fused local gather + put into the receivers' halo buffers, flag signalling (p2p.cu)
    if (!D->p2p_connected) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_spmv: call pjds_dist_p2p_connect first");
    const uint64_t sq = ++D->seq;
    const int b = (int)(sq & 1);
    const bool vec = flags & PJDS_NO_OVERLAP;
    cudaStream_t cs = vec ? s : D->comm;
    const int ns = (int)D->send_peers.size(), nr = (int)D->recv_peers.size();
    PJDS_TRY(mark(0, s));
    if (!vec) {
      PJDS_CUDA_TRY(cudaEventRecord(D->ev_ready, s));
      PJDS_CUDA_TRY(cudaStreamWaitEvent(cs, D->ev_ready, 0));
    }
    PJDS_TRY(mark(1, cs));
    if (sq >= 3) PJDS_TRY(p2p_launch_wait(D->done_flags(), D->d_send_peers, ns, sq - 2, D->err_flag(), cs));
    PJDS_TRY(p2p_launch_pack_put(x, D->d_p2p_idx, D->d_p2p_seg, D->d_dst[b], ns, D->p2p_max_count, D->dtype, cs));
    PJDS_TRY(mark(2, cs));
    PJDS_TRY(p2p_launch_signal(D->d_ready_targets, ns, sq, cs));
    if (vec) PJDS_TRY(p2p_launch_wait(D->ready_flags(), D->d_recv_peers, nr, sq, D->err_flag(), s));
    PJDS_TRY(mark(3, cs));
    if (!vec) PJDS_CUDA_TRY(cudaEventRecord(D->ev_comm, cs));
    PJDS_TRY(launch_pjds_spmv(D->A_loc, y, x, s, false));
    PJDS_TRY(mark(4, s));
    if (!vec) {
      PJDS_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_comm, 0));  // own gather done: x may be reused
      PJDS_TRY(p2p_launch_wait(D->ready_flags(), D->d_recv_peers, nr, sq, D->err_flag(), s));
    }
    PJDS_TRY(mark(5, s));
    if (D->A_nl) PJDS_TRY(launch_pjds_spmv(D->A_nl, y, D->p2p_region + b * D->p2p_halo_bytes, s, true));
    PJDS_TRY(p2p_launch_signal(D->d_done_targets, nr, sq, s));
    PJDS_TRY(mark(6, s));
    D->traced = D->traced || tr;
    return PJDS_OK;
  }
  if (flags & PJDS_NO_OVERLAP) {  // vector mode: exchange, then both parts, one stream
    PJDS_TRY(mark(0, s));
    PJDS_TRY(mark(1, s));
    if (D->packed_total) PJDS_TRY(launch_pack(D->d_pack_idx, D->packed_total, x, D->d_packbuf, D->dtype, s));
    PJDS_TRY(mark(2, s));
    PJDS_TRY(post_nccl(D, x, s));
    PJDS_TRY(mark(3, s));
    PJDS_TRY(launch_pjds_spmv(D->A_loc, y, x, s, false));
    PJDS_TRY(mark(4, s));
    PJDS_TRY(mark(5, s));
    if (D->A_nl) PJDS_TRY(launch_pjds_spmv(D->A_nl, y, D->d_halo, s, true));
    PJDS_TRY(mark(6, s));
    D->traced = D->traced || tr;
    return PJDS_OK;
  }
  // task mode: comm stream starts after x is ready on the compute stream
  PJDS_TRY(mark(0, s));
  PJDS_CUDA_TRY(cudaEventRecord(D->ev_ready, s));
  PJDS_CUDA_TRY(cudaStreamWaitEvent(D->comm, D->ev_ready, 0));
  PJDS_TRY(mark(1, D->comm));
  if (D->packed_total) PJDS_TRY(launch_pack(D->d_pack_idx, D->packed_total, x, D->d_packbuf, D->dtype, D->comm));
  PJDS_TRY(mark(2, D->comm));
  PJDS_TRY(post_nccl(D, x, D->comm));
  PJDS_TRY(mark(3, D->comm));
  PJDS_CUDA_TRY(cudaEventRecord(D->ev_comm, D->comm));
  PJDS_TRY(launch_pjds_spmv(D->A_loc, y, x, s, false));
  PJDS_TRY(mark(4, s));
  PJDS_CUDA_TRY(cudaStreamWaitEvent(s, D->ev_comm, 0));
  PJDS_TRY(mark(5, s));
  if (D->A_nl) PJDS_TRY(launch_pjds_spmv(D->A_nl, y, D->d_halo, s, true));
  PJDS_TRY(mark(6, s));
  D->traced = D->traced || tr;
  return PJDS_OK;
}

int pjds_dist_trace(pjds_dist_t D, double* ms) {
  if (!D || !ms) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_trace: NULL argument");
  if (!D->traced) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_trace: no traced pjds_dist_spmv call yet");
  PJDS_CUDA_TRY(cudaEventSynchronize(D->tev[6]));
  PJDS_CUDA_TRY(cudaEventSynchronize(D->tev[3]));
  float t[7];
  for (int i = 1; i < 7; ++i) PJDS_CUDA_TRY(cudaEventElapsedTime(&t[i], D->tev[0], D->tev[i]));
  ms[0] = t[6];          // total
  ms[1] = t[4];          // start -> local part done
  ms[2] = t[2] - t[1];   // pack
  ms[3] = t[3] - t[2];   // NCCL exchange
  ms[4] = t[5] - t[4];   // compute stream waiting for the exchange after the local part
  ms[5] = t[6] - t[5];   // nonlocal part
  return PJDS_OK;
}

int pjds_dist_group_spmv(pjds_dist_t* Ds, int32_t R, void* const* y, const void* const* x, void* stream,
                         uint32_t flags) {
  (void)flags;
  if (!Ds || R < 1 || !y || !x) return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_group_spmv: bad argument");
  for (int r = 0; r < R; ++r)
    if (!Ds[r] || Ds[r]->R != R || Ds[r]->rank != r || Ds[r]->transport != PJDS_TRANSPORT_LOCAL)
      return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_group_spmv: handles must be LOCAL, rank-ordered, same R");
  cudaStream_t s = (cudaStream_t)stream;
  // 1. pack (local gather) on every rank
  for (int r = 0; r < R; ++r) {
    pjds_dist* D = Ds[r];
    if (D->packed_total) PJDS_TRY(launch_pack(D->d_pack_idx, D->packed_total, x[r], D->d_packbuf, D->dtype, s));
  }
  // 2. exchange: receiver r's message list from peer q matches sender q's list to r one-to-one
  for (int r = 0; r < R; ++r) {
    pjds_dist* D = Ds[r];
    const size_t vs = vsz(D);
    for (auto& pr : D->recvs) {
      pjds_dist* S = Ds[pr.peer];
      const pjds_dist::PeerSend* ps = nullptr;
      for (auto& c : S->sends)
        if (c.peer == r) ps = &c;
      if (!ps || ps->runs.size() != pr.runs.size())
        return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_group_spmv: send/recv schedules do not match");
      const char* base = ps->packed ? (const char*)S->d_packbuf : (const char*)x[pr.peer];
      for (size_t i = 0; i < pr.runs.size(); ++i) {
        if (ps->runs[i].second != pr.runs[i].second)
          return set_error(PJDS_ERR_INVALID_ARG, "pjds_dist_group_spmv: message sizes do not match");
        PJDS_CUDA_TRY(cudaMemcpyAsync((char*)D->d_halo + pr.runs[i].first * vs, base + ps->runs[i].first * vs,
                                      pr.runs[i].second * vs, cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  // 3. local then nonlocal part on every rank
  for (int r = 0; r < R; ++r) {
    pjds_dist* D = Ds[r];
    PJDS_TRY(launch_pjds_spmv(D->A_loc, y[r], x[r], s, false));
    if (D->A_nl) PJDS_TRY(launch_pjds_spmv(D->A_nl, y[r], D->d_halo, s, true));
  }
  return PJDS_OK;
}

}  // extern "C"
