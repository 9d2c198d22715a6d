/*
 * pjds.h — C ABI of libpjds: sparse matrix-vector multiplication y = A x in the padded jagged
 * diagonals storage (pJDS) format of Kreutzer, Hager, Wellein, Fehske, Basermann, Bishop,
 * "Sparse matrix-vector multiplication on GPGPU clusters: A new storage format and a scalable
 * implementation" (arXiv 1112.5588; cited as PAPER.md L<line>), with ELLPACK-R as the in-library
 * comparison format, on NVIDIA B200 (sm_100a).
 *
 * Conventions for every entry point
 *   - Return value: pjds_status (0 = PJDS_OK, < 0 = error).  Nothing aborts; on error a
 *     thread-local message is available from pjds_last_error().
 *   - Host arrays passed to *_create* are only read during the call (the caller keeps ownership).
 *   - Handles own all device memory they allocate until *_destroy.
 *   - x / y in *_spmv are caller-owned DEVICE pointers on the handle's device with the handle's
 *     dtype (float for PJDS_F32, double for PJDS_F64); y must not alias x (PJDS_ERR_INVALID_ARG).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is enqueued
 *     and the call returns; launch errors are returned immediately, asynchronous faults surface
 *     at the caller's next synchronisation.
 *   - Preconditions on values: x must be finite (padding slots compute +0.0 * x[0], reading 7).
 *   - Index types: rowptr int64, column indices int32 (n < 2^31), offsets int64.
 */
#ifndef PJDS_H
#define PJDS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pjds_mat* pjds_t;
typedef struct ellr_mat* ellr_t;
typedef struct pjds_plan* pjds_plan_t;
typedef struct pjds_dist* pjds_dist_t;

typedef enum { PJDS_F32 = 0, PJDS_F64 = 1 } pjds_dtype;

typedef enum {
  PJDS_OK = 0,
  PJDS_ERR_INVALID_ARG = -1, /* null pointer, bad size, bad block_rows, aliasing, wrong mode */
  PJDS_ERR_BAD_CSR = -2,     /* rowptr[0] != 0, decreasing rowptr, column out of range */
  PJDS_ERR_OOM = -3,         /* host or device allocation failed */
  PJDS_ERR_CUDA = -4,        /* CUDA runtime error (message has cudaGetErrorString) */
  PJDS_ERR_NCCL = -5,        /* NCCL missing or failed (message has ncclGetErrorString) */
  PJDS_ERR_UNSUPPORTED = -6  /* feature not available in this build / on this device */
} pjds_status;

/* create flags */
enum {
  PJDS_PERM_ROWS = 0u,      /* default: rows permuted only; x and y in the ORIGINAL basis,
                               y stored through perm (reading 9) */
  PJDS_PERM_SYMMETRIC = 1u, /* permuted basis: columns mapped through
                               invperm, x and y both in the permuted basis (P A P^T) */
  PJDS_HOST_ONLY = 2u       /* convert on the host only, no device allocation (export/info
                               work, spmv returns PJDS_ERR_INVALID_ARG); used by CPU tests */
};

/* ------------------------------------------------------------------ single-GPU formats */

/*
 * pjds_create_from_crs — CRS -> pJDS, §2.1 L213-229 and Listing 2:
 *   a1 row lengths (stored CRS entries, explicit zeros and duplicates count);
 *   a2 "sort": rows by descending length, ties by ascending original row (stable), perm[new]=old;
 *   a3 "pad": n_pad = ceil(n/block_rows)*block_rows with zero-length virtual rows, every block of
 *      block_rows consecutive sorted rows padded to its longest row: block_len[b] (non-increasing);
 *   a4 col_start[j] (j = 0..width, width = block_len[0]): offset of jagged column j,
 *      col_start[j+1] = col_start[j] + block_rows * #{b : block_len[b] > j};
 *   a5 fill: val[col_start[j] + k] = j-th stored entry of sorted row k (CRS order kept),
 *      padding (+0.0, column 0); then one upload to the current CUDA device.
 *  n          rows = columns (square), 0 <= n < 2^31
 *  rowptr     host int64[n+1], rowptr[0] = 0, non-decreasing
 *  col        host int32[rowptr[n]], 0 <= col < n
 *  val        host float[] / double[] per dtype, rowptr[n] entries
 *  block_rows b_r: a positive multiple of 32 (warp size); 0 means 32
 *  flags      PJDS_PERM_* | PJDS_HOST_ONLY
 */
int pjds_create_from_crs(pjds_t* out, int64_t n, const int64_t* rowptr, const int32_t* col,
                         const void* val, int dtype, int32_t block_rows, uint32_t flags);
/*
 * pjds_create_from_crs_ex — as pjds_create_from_crs with a sort scope `sigma` (SURVEY §8(f)
 * NEXT-2, the sliced-ELLPACK / SELL-C-sigma idea the paper names as future comparison, PAPER.md
 * L527-531): rows are sorted by descending length only within consecutive windows of sigma rows,
 * each window is padded and stored jagged column-major on its own (per-window col_start), so the
 * permutation never moves a row out of its window (RHS locality).
 * sigma = 0: one global window (the paper's pJDS).  Otherwise a multiple of 1024 and of block_rows.
 */
int pjds_create_from_crs_ex(pjds_t* out, int64_t n, const int64_t* rowptr, const int32_t* col,
                            const void* val, int dtype, int32_t block_rows, int64_t sigma,
                            uint32_t flags);
int pjds_destroy(pjds_t A);

/*
 * pjds_spmv — y = A x (overwrite; reading 11) with the pJDS kernel (Listing 2,
 * PAPER.md L231-237; one thread per row, rows of a warp in one block).
 * Per row: one fused multiply-add chain over the row's stored entries in CRS order, starting
 * from +0.0, in the matrix precision; padded slots add exact +0.  Rows of length 0 give y = +0.
 * PJDS_PERM_ROWS: x, y original basis.  PJDS_PERM_SYMMETRIC: x, y permuted basis.
 */
int pjds_spmv(pjds_t A, void* y, const void* x, void* stream);
/* y[perm[k]] += (A x)_k for a row-permuted handle: y = y + A x, each row's chain from +0.0 added to
   y_i with ONE rounding add (the dist nonlocal pass, "written twice"; reading 25).
   Same arguments as pjds_spmv.  PJDS_ERR_UNSUPPORTED for PJDS_PERM_SYMMETRIC handles. */
int pjds_spmv_accum(pjds_t A, void* y, const void* x, void* stream);

/*
 * pjds_permute — basis change for the permuted-basis mode ("permutation of
 * the indices needs to be done only before the start and after the end of the algorithm"):
 * direction 0: dst[k] = src[perm[k]] (original -> permuted), 1: dst[perm[k]] = src[k] (back).
 * Device pointers of n entries, handle dtype; dst must not alias src.  Any handle may be used.
 */
int pjds_permute(pjds_t A, void* dst, const void* src, int32_t direction, void* stream);

/*
 * pjds_spmv_host — end-to-end variant with HOST x / y in the ORIGINAL basis (any host memory;
 * pinned is faster): copies x host->device, (PJDS_PERM_SYMMETRIC: permutes x to the permuted
 * basis), runs the pJDS kernel, (permutes y back), copies y device->host, synchronises `stream`.
 * The transfer cost is the paper's T_PCI (Eq. 2).  Staging buffers are
 * allocated on first use and owned by the handle, so calls on one handle must not run
 * concurrently from several host threads (pjds_spmv itself has no such restriction).
 */
int pjds_spmv_host(pjds_t A, void* y_host, const void* x_host, void* stream);

/*
 * pjds_spmv_host_batch — `count` independent products y_host[i] = A x_host[i] with host vectors
 * (original basis), pipelined: the host->device copy of x_{i+1} and the device->host copy of y_{i-1}
 * run on two copy streams while product i runs on `stream` (double-buffered staging owned by the
 * handle), so PCIe traffic in both directions overlaps the kernels.  Host vectors should be
 * pinned for the copies to be asynchronous.  Synchronises `stream` before returning.  Same
 * one-caller-at-a-time rule per handle as pjds_spmv_host.
 */
int pjds_spmv_host_batch(pjds_t A, void* const* y_host, const void* const* x_host, int32_t count,
                         void* stream);

typedef struct {
  int64_t n, nnz, n_pad, n_blocks, stored;
  int32_t block_rows, width, dtype, flags;
  int32_t len_min, len_max;
  double len_mean;
  /* Fig. 2 counters, lane-slots: useful = nnz, padded = stored - nnz
     (executed as +0 FMAs), idle = 0 (every lane of a block runs block_len steps) */
  int64_t useful_fma, padded_fma, idle_lane_slots;
  /* footprint (Table 1): values, int32 column indices,
     aux = col_start (int64, width+1) + block_len (int32, n_blocks) + perm (int32, n) */
  int64_t bytes_values, bytes_indices, bytes_aux, bytes_total;
  double data_reduction_vs_ellpack; /* 1 - stored / (ceil(n/32)*32 * width), entries basis */
  int32_t on_device;
  int32_t device;
  int64_t sigma;          /* sort scope in rows (n_pad for the paper's global sort) */
  int64_t n_windows;      /* number of sort windows (1 for the global sort) */
  int64_t col_start_len;  /* entries of the concatenated per-window col_start (width+1 if global) */
  int32_t col_compressible; /* 1: col lives in generic compressible memory (pjds_set_compression) */
} pjds_info_t;

int pjds_info(pjds_t A, pjds_info_t* out);

/*
 * Footprint and statistics under the names of SURVEY §8(b) (views of pjds_info / ellr_info):
 * pjds_footprint — bytes per component (Table 1 L291 and L284-286): values (stored x s_v),
 *   int32 column indices, col_start (int64, width+1 per window, + window tables), block_len
 *   (int32, n_blocks), perm (int32, n); bytes_rowmax = 0.  ellr_footprint — values, indices,
 *   rowmax (int32, N_pad); the pJDS aux fields are 0.  Both: stored / nnz / n_pad entries.
 * pjds_stats — shape and Fig. 2 counters: n, nnz, n_pad, n_blocks,
 *   padding = stored - nnz, width, block_rows, row-length min/max/mean, entries-based reduction
 *   vs ELLPACK (1 - stored / (ceil(n/32)*32 * width)), useful / padded / idle lane-slots.
 * Host-side only (no device access); INVALID_ARG on NULL.
 */
typedef struct {
  int64_t bytes_values, bytes_indices;
  int64_t bytes_col_start, bytes_block_len, bytes_perm; /* pJDS aux; 0 for ELLPACK-R */
  int64_t bytes_rowmax;                                 /* ELLPACK-R aux; 0 for pJDS */
  int64_t bytes_total, stored, nnz, n_pad;
} pjds_footprint_t;
int pjds_footprint(pjds_t A, pjds_footprint_t* out);
typedef struct {
  int64_t n, nnz, n_pad, n_blocks, padding;
  int32_t width, block_rows, len_min, len_max;
  double len_mean, reduction_vs_ellpack;
  int64_t useful_fma, padded_fma, idle_lane_slots;
} pjds_stats_t;
int pjds_stats(pjds_t A, pjds_stats_t* out);

/* Window layout (host buffers of n_windows+1 entries): wstart[w] = first stored slot of window w
   (wstart[n_windows] = stored); wcs_off[w] = start of window w's col_start in the export array. */
int pjds_export_windows(pjds_t A, int64_t* wstart, int64_t* wcs_off);

/* Row-length histogram (Fig. 3, bin size 1): counts[L] = #rows of length L
   for L < nbins (rows longer than nbins-1 are not counted). */
int pjds_histogram(pjds_t A, int64_t* counts, int32_t nbins);

/* Copy the format arrays into caller HOST buffers sized from pjds_info: perm[n],
   block_len[n_blocks], col_start[col_start_len] (per window, relative to the window's first
   stored slot, concatenated), col[stored], val[stored] (any may be NULL). */
int pjds_export(pjds_t A, int32_t* perm, int32_t* block_len, int64_t* col_start, int32_t* col,
                void* val);

/*
 * ellr_create_from_crs — CRS -> ELLPACK-R: entries shifted
 * left, N_pad = ceil(n/32)*32 rows x width = N^max_nzr columns stored column by column
 * (val[j*N_pad + i]), padding (+0.0, col 0), rowmax[i] = row length (0 for pad rows).
 * Same argument rules as pjds_create_from_crs (flags: 0 or PJDS_HOST_ONLY).
 */
int ellr_create_from_crs(ellr_t* out, int64_t n, const int64_t* rowptr, const int32_t* col,
                         const void* val, int dtype, uint32_t flags);
int ellr_destroy(ellr_t A);
/* y = A x with the ELLPACK-R kernel (Listing 1), same chain semantics. */
int ellr_spmv(ellr_t A, void* y, const void* x, void* stream);

typedef struct {
  int64_t n, nnz, n_pad, stored;
  int32_t width, dtype;
  int64_t useful_fma, padded_fma, idle_lane_slots; /* idle = sum_warps sum_lanes (max - len) */
  int64_t bytes_values, bytes_indices, bytes_aux, bytes_total; /* aux = rowmax int32[n_pad] */
  int32_t on_device, device;
  int32_t col_compressible; /* 1: col lives in generic compressible memory (pjds_set_compression) */
} ellr_info_t;
int ellr_info(ellr_t A, ellr_info_t* out);
int ellr_footprint(ellr_t A, pjds_footprint_t* out); /* see pjds_footprint */
int ellr_export(ellr_t A, int32_t* rowmax, int32_t* col, void* val);

/* ------------------------------------------------------------------ distributed (§3) */

/*
 * Row-partitioned spMVM.  Rank r owns rows and x entries
 * [row_offsets[r], row_offsets[r+1]).  Its rows are split into a local part (columns it owns)
 * and a nonlocal part (columns owned by other ranks); the nonlocal x entries
 * (halo) are exchanged with NCCL send/recv on a high-priority side stream while the local part
 * runs (task mode), then the nonlocal part accumulates y += (the result is
 * written twice, L445).
 *
 * Setup is three steps so that the only cross-rank setup traffic (index lists) is plumbing done
 * by the caller (e.g. torch.distributed all_to_all):
 *   1. pjds_dist_plan      (local, host): split + recv lists.  Halo schedule conventions:
 *                          recv list from owner q = sorted unique global columns owned by q;
 *                          halo slot = position in the concatenation ordered by owner rank.
 *   2. caller exchanges recv lists -> send lists (what each peer needs from this rank).
 *   3. pjds_dist_create    builds A_loc (all local rows, local column ids) and A_nl (rows with
 *                          >= 1 nonlocal entry, halo-slot column ids), both pJDS, uploads, and
 *                          sets up the transport.
 */
int pjds_dist_plan(pjds_plan_t* out, int32_t nranks, int32_t rank, int64_t n_global,
                   const int64_t* row_offsets /* [nranks+1] */,
                   const int64_t* rowptr_loc /* [n_loc+1], rowptr_loc[0] = 0 */,
                   const int32_t* col_global_loc /* global column ids of this rank's rows */);
typedef struct {
  int64_t n_loc, nnz_loc, nnz_local_part, nnz_nonlocal_part, rows_nonlocal, halo;
  int32_t nranks, rank;
} pjds_plan_info_t;
int pjds_dist_plan_info(pjds_plan_t P, pjds_plan_info_t* out);
/* recv_counts[nranks]; recv_cols[halo] (global ids, owner-ordered); either may be NULL */
int pjds_dist_plan_recv(pjds_plan_t P, int64_t* recv_counts, int32_t* recv_cols);
int pjds_dist_plan_destroy(pjds_plan_t P);

enum {
  PJDS_TRANSPORT_NCCL = 0,  /* one process per GPU; nccl_unique_id = 128-byte ncclUniqueId */
  PJDS_TRANSPORT_LOCAL = 1, /* all ranks' handles in this process (pjds_dist_group_spmv);
                               halo moved with device-to-device copies; test harness */
  PJDS_TRANSPORT_P2P = 2,   /* one process per GPU (or several per GPU), no NCCL per call: a fused
                               gather+put kernel stores the send entries straight into the
                               receivers' halo buffers through CUDA-IPC mappings (NVLink P2P),
                               release/acquire flags order put -> nonlocal part -> buffer reuse.
                               Connect with pjds_dist_p2p_export / _connect after create. */
  PJDS_TRANSPORT_DIRECT = 3 /* one process per GPU (or several per GPU): NO exchange step.  ONE pJDS
                               matrix over the full local rows (CRS order kept within each row, so
                               y is bitwise the unsplit FMA chain); its nonlocal columns address the
                               owners' x windows directly (CUDA-IPC mapped peer memory: NVLink loads
                               between GPUs), so the transfer happens inside the spMVM kernel, tile
                               by tile, overlapped with the local val/col stream -- the B200 form of
                               the paper's communication/computation overlap.
                               Per call: x -> window (skipped if x IS the window), release "ready"
                               to the readers, acquire the owners' "ready", kernel, release "done"
                               to the owners, acquire the readers' "done" (when the call completes
                               on the stream nobody reads this rank's window any more).  Setup:
                               create -> pjds_dist_direct_positions -> caller all_to_all ->
                               pjds_dist_p2p_export / all_gather -> pjds_dist_direct_connect.
                               Needs nranks <= 64 and nranks * 2^ceil(log2(max rows per rank)) <=
                               2^31 (column code (owner << shift) | position in 32 bits);
                               PJDS_NO_OVERLAP has no meaning here (there is nothing to overlap). */
};
enum {
  PJDS_NO_OVERLAP = 1u, /* serialise exchange and compute (vector mode) */
  PJDS_TRACE = 2u       /* record phase events for pjds_dist_trace (Fig. 4 timeline analogue) */
};

/*
 * pjds_dist_create
 *  plan          from pjds_dist_plan (not consumed; may be destroyed afterwards)
 *  val_loc       host values of this rank's rows, in the CRS order given to pjds_dist_plan
 *  send_counts   [nranks] entries this rank sends to each peer
 *  send_cols     concatenation over peers (ascending rank) of GLOBAL column ids owned by this rank,
 *                each peer's list in that peer's recv order (ascending)
 *  transport     PJDS_TRANSPORT_*; nccl_unique_id used for NCCL when nranks > 1 (collective call)
 *  block_rows    as pjds_create_from_crs
 *  flags         0: x_loc / y_loc in the original local order (rows of A_loc permuted only);
 *                PJDS_PERM_SYMMETRIC: x_loc / y_loc in the local permuted basis of A_loc
 *                (convert with pjds_dist_permute); every peer list is then
 *                packed into one message.  All ranks must pass the same flags.
 */
int pjds_dist_create(pjds_dist_t* out, pjds_plan_t plan, const void* val_loc, int dtype,
                     int32_t block_rows, const int64_t* send_counts, const int32_t* send_cols,
                     int32_t transport, const void* nccl_unique_id, uint32_t flags);
/*
 * pjds_dist_create_crs: the one-call collective create of SURVEY §8(b) (NCCL transport; every rank
 * calls it with the same nranks, n_global, row_offsets, block_rows and flags).
 *  nccl_unique_id  128-byte ncclUniqueId, identical on every rank (rank 0 makes it with
 *                  pjds_nccl_unique_id and the caller broadcasts it); unused when nranks == 1
 *  row_offsets     [nranks+1], rank r owns rows and x entries [row_offsets[r], row_offsets[r+1])
 *  rowptr_loc      [n_loc+1] CRS row pointers of this rank's rows (rowptr_loc[0] = 0)
 *  col_global_loc  GLOBAL column ids of this rank's rows;  val_loc: their values (dtype)
 * Inside: pjds_dist_plan, ncclCommInitRank on the caller's current device, the recv-list ->
 * send-list exchange as grouped ncclSend/ncclRecv (counts, then ids), and pjds_dist_create on the
 * same communicator.  Host arrays are copied; the caller keeps ownership.  Errors as
 * pjds_dist_create (+ PJDS_ERR_NCCL for a failed communicator or exchange); nothing is left
 * allocated on failure.  Blocks until every rank has joined (a collective).
 */
int pjds_dist_create_crs(pjds_dist_t* out, const void* nccl_unique_id, int32_t nranks, int32_t rank,
                         int64_t n_global, const int64_t* row_offsets, const int64_t* rowptr_loc,
                         const int32_t* col_global_loc, const void* val_loc, int dtype, int32_t block_rows,
                         uint32_t flags);
/* PJDS_TRANSPORT_P2P setup (collective; the caller all-gathers the blobs, e.g. with
   torch.distributed.all_gather_object):
   pjds_dist_p2p_export: writes this rank's fixed-size blob (CUDA IPC handle of its halo/flag region
     and its halo layout) to `blob` (may be NULL to query) and its size to *bytes.
   pjds_dist_p2p_connect: `blobs` = nranks blobs in rank order; opens the peers' regions.
   pjds_dist_p2p_check: synchronises the device, then *timed_out = 1 if a bounded flag wait gave up
     (~10 s) since create or the previous check, and clears the word.  While it is set, every
     pjds_dist_spmv call of a P2P / DIRECT handle returns PJDS_ERR_CUDA without enqueuing work (the
     y of the call that timed out is invalid: it ran on a stale halo / window). */
int pjds_dist_p2p_export(pjds_dist_t D, void* blob, int64_t* bytes);
int pjds_dist_p2p_connect(pjds_dist_t D, const void* blobs, int64_t blob_bytes);
int pjds_dist_p2p_check(pjds_dist_t D, int32_t* timed_out);
/* PJDS_TRANSPORT_DIRECT setup and use.
   pjds_dist_direct_positions: pos[send_total] = the position in this rank's x window of every
     entry of send_cols (same order): local row id, or its index in the local permuted basis
     (PJDS_PERM_SYMMETRIC).  The caller returns each peer's slice to that peer (all_to_all).
   pjds_dist_direct_connect (collective in effect): halo_pos[halo] = for every halo slot (owner-
     ordered, as pjds_dist_plan_recv), its position in the owner's window, i.e. the owner's
     pjds_dist_direct_positions entries for this rank; blobs = nranks pjds_dist_p2p_export blobs in
     rank order.  Opens the peers' windows, rewrites the matrix's column codes and uploads it.
     INVALID_ARG if a position lies outside the owner's rows.
   pjds_dist_x_window: *x_window = this rank's exported x window (device, n_loc entries of the
     handle dtype, in the basis of the handle).  Compute x there to skip the per-call copy; rewrite
     it only between calls (stream order). */
int pjds_dist_direct_positions(pjds_dist_t D, int32_t* pos);
int pjds_dist_direct_connect(pjds_dist_t D, const int32_t* halo_pos, const void* blobs, int64_t blob_bytes);
int pjds_dist_x_window(pjds_dist_t D, void** x_window);
/* Basis change of a local vector for PJDS_PERM_SYMMETRIC dist handles (see pjds_permute). */
int pjds_dist_permute(pjds_dist_t D, void* dst, const void* src, int32_t direction, void* stream);
/* y_loc = A[rows of this rank, :] x ; x_loc / y_loc device pointers of length n_loc. */
int pjds_dist_spmv(pjds_dist_t D, void* y_loc, const void* x_loc, void* stream, uint32_t flags);
/* PJDS_TRANSPORT_LOCAL: one call runs all R ranks' spMVMs (same device allowed), D/y/x indexed by rank. */
int pjds_dist_group_spmv(pjds_dist_t* D, int32_t nranks, void* const* y_loc, const void* const* x_loc,
                         void* stream, uint32_t flags);
typedef struct {
  int64_t n_loc, halo, send_total, packed_send, rows_nonlocal;
  int64_t nnz_local_part, nnz_nonlocal_part;
  int32_t nranks, rank, peers_send, peers_recv, send_messages, recv_messages;
  int32_t permuted;
} pjds_dist_info_t;
int pjds_dist_info(pjds_dist_t D, pjds_dist_info_t* out);
/* pjds_dist_stats (SURVEY §8(b) name): pjds_dist_info plus the halo size per peer (PAPER.md
   L442-447): recv_per_peer[q] = entries received from rank q (halo slots owned by q),
   send_per_peer[q] = entries sent to rank q; caller host arrays of nranks entries, either may be
   NULL (out may be NULL too).  Sum over q equals halo / send_total. */
int pjds_dist_stats(pjds_dist_t D, pjds_dist_info_t* out, int64_t* recv_per_peer, int64_t* send_per_peer);
/* Phase timeline of the last pjds_dist_spmv call made with PJDS_TRACE (CUDA events on the compute
   and comm streams; synchronises them): ms[0] total, [1] start -> local part done, [2] pack,
   [3] NCCL exchange, [4] compute stream waiting for the exchange, [5] nonlocal part.
   INVALID_ARG if no traced call was made. */
int pjds_dist_trace(pjds_dist_t D, double* ms /* [6] */);
/* The two pJDS parts (owned by D; do not destroy): A_loc, A_nl (A_nl may be NULL if empty).
   DIRECT handles: A_loc = the one matrix over the full local rows (its spmv gathers from the x
   windows, whatever x pointer is passed), A_nl = NULL. */
int pjds_dist_parts(pjds_dist_t D, pjds_t* A_loc, pjds_t* A_nl);
/* Frees the handle (and, for NCCL, the communicator; for P2P, the IPC mappings and the exported
   region).  Collective in effect: synchronise all ranks' streams and barrier before destroying, so
   no peer still writes into (P2P) or exchanges with (NCCL) this rank. */
int pjds_dist_destroy(pjds_dist_t D);
/* Tuning knob (process-wide, read by later pjds_dist_create calls): sort scope of the nonlocal part
   A_nl in rows.  Default 1024: the nonlocal rows are taken in ascending order of their y target
   and sorted by length only within windows of 1024 rows (one CTA tile), so the y += of a CTA
   touches one compact range of y; 0 = the global sort over all nonlocal rows.  Every row's chain
   is the same either way (bitwise-identical y).  INVALID_ARG unless 0 or a multiple of 1024. */
int pjds_set_dist_nl_sigma(int64_t sigma);

/* NCCL helpers (NCCL is dlopen-ed; `libpath` NULL tries "libnccl.so.2"). */
int pjds_nccl_load(const char* libpath);
int pjds_nccl_unique_id(void* out128);

/* ------------------------------------------------------------------ eigensolver driver */

/*
 * pjds_lanczos — m steps of the symmetric Lanczos recurrence, the eigensolver usage the paper's
 * HMEp matrix comes from, on a PJDS_PERM_SYMMETRIC handle, entirely
 * in the permuted basis:
 *   v_0 = v0/||v0||; w = A v_j; alpha_j = w.v_j; w -= alpha_j v_j + beta_{j-1} v_{j-1};
 *   beta_j = ||w||; v_{j+1} = w / beta_j.
 * Precondition: A symmetric (not checked).  v0: device vector (permuted basis, handle dtype, n
 * entries, not modified; INVALID_ARG if its norm is 0).  alpha[m], beta[m]: host outputs (double).
 * *steps_done = m, or j+1 if beta_j = 0 exactly (invariant subspace; entries past steps_done are
 * unspecified).  Dot products accumulate in double.  The m iterations (pJDS kernel with the
 * alpha partials fused into its epilogue, a two-level deterministic alpha reduce, and the vector
 * update whose last CTA computes beta: 3 launches each) are captured into one CUDA graph and
 * launched on `stream`; the call synchronises `stream`.  Work buffers (3 vectors) are allocated
 * and freed inside.
 */
int pjds_lanczos(pjds_t A, const void* v0, int32_t m, double* alpha, double* beta,
                 int32_t* steps_done, void* stream);

/* Eigenvalues (ascending) of the m x m symmetric tridiagonal matrix with diagonal alpha[m] and
   off-diagonal beta[m-1] (the Ritz values of pjds_lanczos), by Sturm bisection; host only. */
int pjds_tridiag_eigenvalues(int32_t m, const double* alpha, const double* beta, double* evals);

/* ------------------------------------------------------------------ misc */

/* Stream-bandwidth probe (roofline denominator, measured in the same run): copies / reads
   `bytes` of device memory `reps` times; returns best GB/s of a copy (read+write bytes) and of a
   read-only reduction.  Allocates and frees its own buffers. */
int pjds_bw_probe(int64_t bytes, int32_t reps, double* copy_gbs, double* read_gbs);

/* Tuning knob (process-wide): pJDS kernel variant with `rows_per_thread` R in {1,2,4} consecutive
   sorted rows per thread (vector loads, R independent FMA chains) and j-unroll `unroll` in {2,4,8}.
   (0, 0) restores the automatic choice.  R is reduced until it divides block_rows.  Every
   variant computes bit-identical y (one FMA chain per row, stored order).  unroll + 16 selects
   the software-pipelined main loop (next chunk's loads issued before the current FMAs);
   rows_per_thread + 8 forces the 64-bit jagged-offset kernels (used when stored + n_pad >= 2^31)
   on any matrix, so tests can cover them.  rows_per_thread = 16 + S selects the long-row split-j
   kernel (S in {2,4} with unroll 4 or 8, or S = 8 with unroll 4): S warps share 32 rows, each
   runs the chain over slots j = s mod S, partials added in the tree ((p0+p1)+(p2+p3))+... — a
   different (fixed, deterministic) summation order from the single chain, within the same O2
   bound.  unroll + 32 selects lane-interleaved rows (a thread's R rows are
   32 apart, so one gather instruction covers 32 consecutive sorted rows; needs block_rows % 32R
   == 0).  The automatic choice (0, 0): R = 4, U = 2 for n_pad / 4 >= 2^19, else R = 2, U = 4
   (software-pipelined in SP), else R = 1, U = 8; lane-interleaved at R = 4 with block_rows a
   multiple of 128 for DP products (the permuted basis, the Lanczos fused-dot product, the DIRECT
   window kernel; the row-only basis and y += A x when x is at most 64 MB, inside the warp tiles of
   the warp-granular order) and for SP products when one length class holds >= 90 % of the rows. */
int pjds_set_kernel_variant(int32_t rows_per_thread, int32_t unroll);

/* Execution order of the CTA tiles of one handle (used whenever the tile order is on: mode 1, or
   mode 2's automatic choice — pjds_set_tile_order): tiles run sorted (stably) by key[orig] of their
   first row's ORIGINAL index, e.g. a 2-D (phonon window, electronic block) key for HMEp-type
   Kronecker matrices so that RHS entries shared across blocks are reused while in L2 (PAPER.md
   L246-249).  key: host int64[n] (copied) or NULL to restore the default key (the original index
   itself).  Only the order of independent tiles changes: results are bit-identical.  Not safe
   while a product on this handle is running. */
int pjds_set_tile_keys(pjds_t A, const int64_t* key, int64_t n);

/* Tuning knob (process-wide): L2 eviction priority of the pJDS kernel's streamed val/col loads
   and of its x gathers; kinds 0 evict_normal, 1 evict_first, 2 evict_last, 3 evict_unchanged.
   Bits 8-15 of stream_kind select the y store of the permuted-basis kernel: 0 = plain scalar
   stores, 1 + kind = one R-wide vector store per thread with that L2 kind.  Bits 16-23 select the
   scattered stores through perm (row-only basis y[perm[k]], dist nonlocal y +=): 0 = plain
   (default), 1 + kind = L1::no_allocate store (and load, for +=) with that L2 kind.  Default:
   stream 1, x 2, y 2 (vector, evict_first; the Lanczos product keeps evict_normal for its y),
   perm stores plain.  Results are unaffected. */
int pjds_set_cache_policy(int32_t stream_kind, int32_t x_kind);
/* Per-handle override of the permuted-basis y store (the policy part of stream_kind bits 8-15
   above): -1 = follow pjds_set_cache_policy (default); 0 = plain scalar stores; 1 + kind = one
   R-wide vector store with L2 policy `kind`.  Used for a dist A_loc, whose y the nonlocal pass
   reads again (an evict-first store would send it to DRAM first).  Results are unchanged. */
int pjds_set_y_store(pjds_t A, int32_t kind);

/* Tuning knob (process-wide): execution order of the pJDS kernel's CTA tiles.  0 = storage
   order (longest blocks first); 1 = tiles ordered by the original index of their first row, so
   rows of all length classes from one region of the matrix run together (RHS reuse in L2,
   local y stores); 3 = the key of mode 1 at warp-tile granularity (32 R sorted rows): each warp of
   a CTA takes the warp tile a table assigns, so one CTA mixes length classes of one region (sort
   scope 0 only); 2 = auto (default): 3 for the row-only basis when no length class holds 90 % of
   the rows, else 1 in the row-only basis or when x exceeds 64 MB, else 0.
   The per-row arithmetic, and therefore y, is identical. */
int pjds_set_tile_order(int32_t mode);
/* pjds_set_schedule (process-wide knob; results are identical): 0 = static grid of CTA tiles
   (default); 1 = dynamic warp tiles (a persistent grid of SMs x resident CTAs whose warps take
   tiles of 32R sorted rows from a per-handle counter).  Measured slower on every config (the
   scattered warp tiles lose the L1 reuse of x between adjacent rows); kept as an experiment.  A
   handle must not run on two streams at once under the dynamic schedule.  Not used by the
   Lanczos-fused product, sigma-windowed handles or the lane-interleaved variant. */
int pjds_set_schedule(int32_t mode);
/* pjds_set_launch_overlap (process-wide knob; results are identical): programmatic dependent launch
   of the pJDS y = A x / y += A x kernel and the ELLPACK-R kernel.  mode 1: launched with
   cudaLaunchAttributeProgrammaticStreamSerialization, a product's CTAs may start while the previous
   kernel on the stream drains its last wave; they run the matrix-only prologue and wait
   (griddepcontrol.wait) for that kernel to complete before reading x or writing y, so the stream
   order of an iterative scheme is kept.  prefetch_cols > 0: first-wave warps
   also prefetch the first prefetch_cols jagged columns of their val/col rows into L2 (global sort
   only) before waiting.  mode 3: dependent launch whose trigger is issued after a CTA's row chains
   (the next grid is scheduled once every CTA has finished its chains; no prefetch).  mode 0: plain
   launches; mode 2 (default, prefetch_cols 2): mode 1 for grids of more than one wave (SMs x
   resident CTAs), mode 3 otherwise -- a one-wave grid launched as an early-triggered dependent
   lands unevenly on the SMs the previous grid frees first (measured slower on the one-wave DLR1
   matrix, faster on multi-wave ones).  The Lanczos-fused product always launches plainly.
   Errors: INVALID_ARG for mode outside {0, 1, 2, 3} or prefetch_cols outside [0, 64]. */
int pjds_set_launch_overlap(int32_t mode, int32_t prefetch_cols);
/* pjds_set_compression (process-wide knob, applied when a handle uploads; results are identical):
   mode 1 (default): the int32 index arrays of every pJDS / ELLPACK-R handle (>= 1 MiB: col, the
   pJDS row-store targets perm, the ELLPACK-R rowmax) are placed in generic compressible device memory (driver VMM, CU_MEM_ALLOCATION_COMP_GENERIC), where
   B200 compresses data between L2 and HBM transparently to the kernels -- the format, layout and
   values are those of PAPER.md L213-237 bit for bit, only the bytes crossing the HBM interface
   shrink (column indices of a jagged column are runs of nearby integers).  Falls back to plain
   cudaMalloc when the driver does not grant compression; pjds_info / ellr_info report
   col_compressible.  mode 0: plain cudaMalloc.  Errors: INVALID_ARG for mode outside {0, 1}. */
int pjds_set_compression(int32_t mode);

/* Number of kernel launches this library has enqueued (process-wide counter). */
int64_t pjds_launch_count(void);

const char* pjds_last_error(void);
const char* pjds_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PJDS_H */
