"""B200-native pJDS sparse matrix-vector multiplication (arXiv 1112.5588, Kreutzer et al.).

Thin Python layer over the C ABI in ``include/pjds.h`` (``libpjds.so``): argument marshalling
only.  Conversion, kernels, halo exchange and everything else on the path run in the library.
PyTorch is used for device memory, streams and process groups.

    A = PjdsMatrix.from_crs(n, rowptr, col, val, block_rows=32)      # CRS -> pJDS on the GPU
    A.spmv(y, x)                                                      # y = A x   (torch CUDA tensors)
    E = EllrMatrix.from_crs(n, rowptr, col, val)                      # ELLPACK-R comparison format
    D = DistPjds.create(n, offsets, rowptr_loc, col_loc, val_loc)     # row-partitioned, NCCL halo
    D.spmv(y_loc, x_loc)
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import (PJDS_F32, PJDS_F64, PJDS_HOST_ONLY, PJDS_NO_OVERLAP, PJDS_PERM_ROWS,  # noqa: F401
                   PJDS_PERM_SYMMETRIC, PJDS_TRANSPORT_LOCAL, PJDS_TRANSPORT_NCCL, PjdsError, call, launch_count,
                   lib, struct_dict)

__all__ = ["PjdsMatrix", "EllrMatrix", "DistPjds", "bw_probe", "launch_count", "lib", "PjdsError"]


def _dt(val) -> int:
    d = np.asarray(val).dtype
    if d == np.float64:
        return PJDS_F64
    if d == np.float32:
        return PJDS_F32
    raise TypeError(f"values must be float32 or float64, got {d}")


def _np_dtype(dt: int):
    return np.float64 if dt == PJDS_F64 else np.float32


def _crs(rowptr, col, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val)
    _dt(val)
    return rowptr, col, val


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _check_vec(t, n, dt, name):
    import torch
    want = torch.float64 if dt == PJDS_F64 else torch.float32
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != want or not t.is_contiguous() or t.numel() < n:
        raise ValueError(f"{name}: need contiguous {want} with >= {n} elements, got {t.dtype} {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


class PjdsMatrix:
    """pJDS matrix (§2.1) owned by libpjds."""

    def __init__(self, handle, keep=None):
        self._h = handle
        self._keep = keep
        inf = _lib.PjdsInfo()
        call("pjds_info", self._h, ctypes.byref(inf))
        self.info = struct_dict(inf)
        self.n = self.info["n"]
        self.dtype = self.info["dtype"]

    @property
    def symmetric(self) -> bool:
        """True for a permuted-basis handle (PJDS_PERM_SYMMETRIC): spmv takes and returns permuted vectors."""
        return bool(self.info["flags"] & PJDS_PERM_SYMMETRIC)

    @classmethod
    def from_crs(cls, n, rowptr, col, val, block_rows: int = 32, symmetric: bool = False, host_only: bool = False,
                 sigma: int = 0):
        """sigma: sort scope in rows (0 = the paper's global sort; else a multiple of 1024)."""
        rowptr, col, val = _crs(rowptr, col, val)
        flags = (PJDS_PERM_SYMMETRIC if symmetric else 0) | (PJDS_HOST_ONLY if host_only else 0)
        h = ctypes.c_void_p()
        call("pjds_create_from_crs_ex", ctypes.byref(h), int(n), rowptr.ctypes.data, col.ctypes.data,
             val.ctypes.data, _dt(val), int(block_rows), int(sigma), flags)
        return cls(h)

    def close(self):
        if getattr(self, "_h", None) and self._keep is None:
            lib().pjds_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def spmv(self, y, x, stream=None):
        """y = A x on the GPU (torch CUDA tensors of the matrix dtype).

        The basis depends on how the handle was built: a row-permuted handle (symmetric=False)
        takes x and returns y in the ORIGINAL basis; a symmetric=True handle (the paper's permuted
        basis) takes x and returns y in the PERMUTED basis -- convert once with
        to_permuted / from_permuted before and after an iterative scheme."""
        call("pjds_spmv", self._h, _check_vec(y, self.n, self.dtype, "y"), _check_vec(x, self.n, self.dtype, "x"),
             _stream_ptr(stream))
        return y

    def spmv_accum(self, y, x, stream=None):
        """y += A x (row-permuted handles; one rounding add per row, the dist nonlocal pass)."""
        call("pjds_spmv_accum", self._h, _check_vec(y, self.n, self.dtype, "y"), _check_vec(x, self.n, self.dtype, "x"),
             _stream_ptr(stream))
        return y

    def to_permuted(self, dst, src, stream=None):
        """dst[k] = src[perm[k]] on the GPU (basis change before an iterative scheme)."""
        call("pjds_permute", self._h, _check_vec(dst, self.n, self.dtype, "dst"), _check_vec(src, self.n, self.dtype, "src"),
             0, _stream_ptr(stream))
        return dst

    def from_permuted(self, dst, src, stream=None):
        """dst[perm[k]] = src[k] on the GPU (basis change after the iterative scheme)."""
        call("pjds_permute", self._h, _check_vec(dst, self.n, self.dtype, "dst"), _check_vec(src, self.n, self.dtype, "src"),
             1, _stream_ptr(stream))
        return dst

    def spmv_host(self, y, x, stream=None):
        """End-to-end y = A x with host numpy arrays in the ORIGINAL basis (H2D x, [permute], kernel,
        [permute back], D2H y, synchronised)."""
        nd = _np_dtype(self.dtype)
        assert x.dtype == nd and y.dtype == nd and x.flags.c_contiguous and y.flags.c_contiguous
        assert len(x) >= self.n and len(y) >= self.n
        call("pjds_spmv_host", self._h, y.ctypes.data, x.ctypes.data, _stream_ptr(stream))
        return y

    def spmv_host_batch(self, ys, xs, stream=None):
        """Pipelined end-to-end products ys[i] = A xs[i] with (pinned) host numpy arrays in the original
        basis: H2D of the next x and D2H of the previous y overlap the current product."""
        nd = _np_dtype(self.dtype)
        assert len(ys) == len(xs)
        for v in list(xs) + list(ys):
            assert v.dtype == nd and v.flags.c_contiguous and len(v) >= self.n
        Y = (ctypes.c_void_p * len(ys))(*[v.ctypes.data for v in ys])
        X = (ctypes.c_void_p * len(xs))(*[v.ctypes.data for v in xs])
        call("pjds_spmv_host_batch", self._h, Y, X, len(xs), _stream_ptr(stream))
        return ys

    def lanczos(self, v0, m: int, stream=None):
        """m Lanczos steps in the permuted basis (needs symmetric=True and a symmetric matrix).
        v0: CUDA tensor in the permuted basis.  Returns (alpha, beta, steps_done) as numpy."""
        alpha = np.zeros(m)
        beta = np.zeros(m)
        steps = ctypes.c_int32()
        call("pjds_lanczos", self._h, _check_vec(v0, self.n, self.dtype, "v0"), int(m), alpha.ctypes.data,
             beta.ctypes.data, ctypes.byref(steps), _stream_ptr(stream))
        return alpha, beta, steps.value

    def set_tile_keys(self, keys=None):
        """Tile execution order by a key per ORIGINAL row (pjds_set_tile_keys); None restores the
        default (original index).  Results are unchanged; only L2 reuse can differ."""
        if keys is None:
            call("pjds_set_tile_keys", self._h, None, 0)
        else:
            k = np.ascontiguousarray(keys, dtype=np.int64)
            call("pjds_set_tile_keys", self._h, k.ctypes.data, len(k))
        return self

    def footprint(self) -> dict:
        """Bytes per component (pjds_footprint: values, indices, col_start, block_len, perm)."""
        f = _lib.Footprint()
        call("pjds_footprint", self._h, ctypes.byref(f))
        return struct_dict(f)

    def stats(self) -> dict:
        """Shape, padding, row lengths, reduction vs ELLPACK and Fig. 2 counters (pjds_stats)."""
        st = _lib.Stats()
        call("pjds_stats", self._h, ctypes.byref(st))
        return struct_dict(st)

    def histogram(self):
        counts = np.zeros(self.info["len_max"] + 1, dtype=np.int64)
        call("pjds_histogram", self._h, counts.ctypes.data, len(counts))
        return counts

    def export(self):
        i = self.info
        out = dict(perm=np.empty(i["n"], np.int32), block_len=np.empty(i["n_blocks"], np.int32),
                   col_start=np.empty(i["col_start_len"], np.int64), col=np.empty(i["stored"], np.int32),
                   val=np.empty(i["stored"], _np_dtype(i["dtype"])),
                   wstart=np.empty(i["n_windows"] + 1, np.int64), wcs_off=np.empty(i["n_windows"] + 1, np.int64))
        call("pjds_export", self._h, out["perm"].ctypes.data, out["block_len"].ctypes.data,
             out["col_start"].ctypes.data, out["col"].ctypes.data, out["val"].ctypes.data)
        call("pjds_export_windows", self._h, out["wstart"].ctypes.data, out["wcs_off"].ctypes.data)
        return out


class EllrMatrix:
    """ELLPACK-R matrix owned by libpjds."""

    def __init__(self, handle):
        self._h = handle
        inf = _lib.EllrInfo()
        call("ellr_info", self._h, ctypes.byref(inf))
        self.info = struct_dict(inf)
        self.n = self.info["n"]
        self.dtype = self.info["dtype"]

    @classmethod
    def from_crs(cls, n, rowptr, col, val, host_only: bool = False):
        rowptr, col, val = _crs(rowptr, col, val)
        h = ctypes.c_void_p()
        call("ellr_create_from_crs", ctypes.byref(h), int(n), rowptr.ctypes.data, col.ctypes.data, val.ctypes.data,
             _dt(val), PJDS_HOST_ONLY if host_only else 0)
        return cls(h)

    def close(self):
        if getattr(self, "_h", None):
            lib().ellr_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def spmv(self, y, x, stream=None):
        call("ellr_spmv", self._h, _check_vec(y, self.n, self.dtype, "y"), _check_vec(x, self.n, self.dtype, "x"),
             _stream_ptr(stream))
        return y

    def footprint(self) -> dict:
        """Bytes per component (ellr_footprint: values, indices, rowmax)."""
        f = _lib.Footprint()
        call("ellr_footprint", self._h, ctypes.byref(f))
        return struct_dict(f)

    def export(self):
        i = self.info
        out = dict(rowmax=np.empty(i["n_pad"], np.int32), col=np.empty(i["stored"], np.int32),
                   val=np.empty(i["stored"], _np_dtype(i["dtype"])))
        call("ellr_export", self._h, out["rowmax"].ctypes.data, out["col"].ctypes.data, out["val"].ctypes.data)
        return out


class DistPlan:
    """Host-side split + halo schedule of one rank (pjds_dist_plan)."""

    def __init__(self, nranks, rank, n_global, offsets, rowptr_loc, col_loc):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        rowptr_loc = np.ascontiguousarray(rowptr_loc, dtype=np.int64)
        col_loc = np.ascontiguousarray(col_loc, dtype=np.int32)
        self._h = ctypes.c_void_p()
        call("pjds_dist_plan", ctypes.byref(self._h), int(nranks), int(rank), int(n_global),
             self.offsets.ctypes.data, rowptr_loc.ctypes.data, col_loc.ctypes.data)
        inf = _lib.PlanInfo()
        call("pjds_dist_plan_info", self._h, ctypes.byref(inf))
        self.info = struct_dict(inf)
        self.nranks, self.rank = nranks, rank

    def recv(self):
        counts = np.zeros(self.nranks, np.int64)
        cols = np.zeros(self.info["halo"], np.int32)
        call("pjds_dist_plan_recv", self._h, counts.ctypes.data, cols.ctypes.data)
        return counts, cols

    def close(self):
        if getattr(self, "_h", None):
            lib().pjds_dist_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _nccl_path():
    """The libnccl.so.2 torch uses (the pip nvidia-nccl package), so libpjds and torch share one
    NCCL; None lets the library fall back to the loader's search path."""
    import glob
    import os
    import site
    if os.environ.get("PJDS_NCCL_LIB"):  # explicit choice (tests substitute a one-GPU stand-in)
        return os.environ["PJDS_NCCL_LIB"].encode()
    for d in site.getsitepackages():
        hits = glob.glob(os.path.join(d, "nvidia", "nccl", "lib", "libnccl.so*"))
        if hits:
            return sorted(hits)[0].encode()
    return None


def exchange_lists(recv_counts, recv_cols, group=None):
    """Turn every rank's recv lists into its send lists with torch.distributed all_to_all_single
    (setup-time plumbing; works on gloo (CPU) and NCCL (CUDA tensors))."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    rc = torch.as_tensor(np.asarray(recv_counts, np.int64), device=dev)
    sc = torch.empty_like(rc)
    dist.all_to_all_single(sc, rc, group=group)
    send_counts = sc.cpu().numpy().astype(np.int64)
    inp = torch.as_tensor(np.asarray(recv_cols, np.int32), device=dev)
    out = torch.empty(int(send_counts.sum()), dtype=torch.int32, device=dev)
    dist.all_to_all_single(out, inp, output_split_sizes=send_counts.tolist(),
                           input_split_sizes=[int(v) for v in recv_counts], group=group)
    return send_counts, out.cpu().numpy().astype(np.int32)


def _alltoallv_i32(arr, in_splits, out_splits, group=None):
    """all_to_all_single of an int32 array with the given splits (setup-time plumbing)."""
    import torch
    import torch.distributed as dist
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl"
           else torch.device("cpu"))
    inp = torch.as_tensor(np.ascontiguousarray(arr, np.int32), device=dev)
    out = torch.empty(int(np.sum(out_splits)), dtype=torch.int32, device=dev)
    dist.all_to_all_single(out, inp, output_split_sizes=[int(v) for v in out_splits],
                           input_split_sizes=[int(v) for v in in_splits], group=group)
    return out.cpu().numpy().astype(np.int32)


class _DeviceArray:
    """__cuda_array_interface__ view of library-owned device memory (no ownership)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


class DistPjds:
    """Row-partitioned distributed pJDS spMVM (§3): local part overlapped with the
    NCCL halo exchange on a high-priority side stream, then the nonlocal part (y +=)."""

    def __init__(self, handle, plan_info, nranks, rank, dtype):
        self._h = handle
        self.nranks, self.rank, self.dtype = nranks, rank, dtype
        self.plan_info = plan_info
        inf = _lib.DistInfo()
        call("pjds_dist_info", self._h, ctypes.byref(inf))
        self.info = struct_dict(inf)
        self.n_loc = self.info["n_loc"]

    @classmethod
    def create(cls, n_global, offsets, rowptr_loc, col_loc, val_loc, block_rows: int = 32, group=None,
               permuted: bool = False, transport: str = "nccl"):
        """Collective over the torch.distributed default (or given) group: one rank per GPU.
        permuted: x_loc / y_loc live in the local permuted basis (to_permuted / from_permuted).
        transport: "nccl" (grouped send/recv on a side stream), "p2p" (fused gather+put kernel
        into the peers' halo buffers through CUDA-IPC mappings, no NCCL per call) or "direct" (no
        exchange step: ONE kernel per call whose nonlocal gathers read the owners' x windows
        through CUDA-IPC mappings; place x in `x_window()` to skip the per-call copy)."""
        import torch.distributed as dist
        R, rank = dist.get_world_size(group), dist.get_rank(group)
        val_loc = np.ascontiguousarray(val_loc)
        if transport == "nccl":
            # the one-call collective create: the library plans, builds its NCCL
            # communicator and exchanges the index lists over it; Python only broadcasts the id
            uid = (ctypes.c_char * 128)()
            if R > 1:
                call("pjds_nccl_load", _nccl_path())
                if rank == 0:
                    call("pjds_nccl_unique_id", uid)
                obj = [bytes(uid) if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0, group=group)
                ctypes.memmove(uid, obj[0], 128)
            offs = np.ascontiguousarray(offsets, np.int64)
            rp = np.ascontiguousarray(rowptr_loc, np.int64)
            cl = np.ascontiguousarray(col_loc, np.int32)
            h = ctypes.c_void_p()
            call("pjds_dist_create_crs", ctypes.byref(h), uid, R, rank, int(n_global), offs.ctypes.data,
                 rp.ctypes.data, cl.ctypes.data, val_loc.ctypes.data, _dt(val_loc), int(block_rows),
                 PJDS_PERM_SYMMETRIC if permuted else 0)
            return cls(h, None, R, rank, _dt(val_loc))
        plan = DistPlan(R, rank, n_global, offsets, rowptr_loc, col_loc)
        rc, rcols = plan.recv()
        sc, scols = exchange_lists(rc, rcols, group)
        uid = (ctypes.c_char * 128)()
        tr = {"p2p": _lib.PJDS_TRANSPORT_P2P, "direct": _lib.PJDS_TRANSPORT_DIRECT}[transport]
        h = ctypes.c_void_p()
        call("pjds_dist_create", ctypes.byref(h), plan._h, val_loc.ctypes.data, _dt(val_loc), int(block_rows),
             sc.ctypes.data, scols.ctypes.data, tr, uid, PJDS_PERM_SYMMETRIC if permuted else 0)
        obj = cls(h, plan.info, R, rank, _dt(val_loc))  # owns h from here on (freed on any later error)
        plan.close()
        if transport == "p2p":
            nb = ctypes.c_int64()
            call("pjds_dist_p2p_export", h, None, ctypes.byref(nb))
            blob = (ctypes.c_char * nb.value)()
            call("pjds_dist_p2p_export", h, blob, ctypes.byref(nb))
            blobs = [None] * R
            dist.all_gather_object(blobs, bytes(blob), group=group)
            allb = b"".join(blobs)
            call("pjds_dist_p2p_connect", h, ctypes.c_char_p(allb), nb.value)
            dist.barrier(group=group)
        if transport == "direct":
            # my window positions of what each peer reads from me -> that peer's halo positions
            pos = np.zeros(max(int(sc.sum()), 1), np.int32)
            call("pjds_dist_direct_positions", h, pos.ctypes.data)
            halo_pos = _alltoallv_i32(pos[:int(sc.sum())], sc, rc, group)
            nb = ctypes.c_int64()
            call("pjds_dist_p2p_export", h, None, ctypes.byref(nb))
            blob = (ctypes.c_char * nb.value)()
            call("pjds_dist_p2p_export", h, blob, ctypes.byref(nb))
            blobs = [None] * R
            dist.all_gather_object(blobs, bytes(blob), group=group)
            hp = np.ascontiguousarray(halo_pos if len(halo_pos) else np.zeros(1, np.int32))
            call("pjds_dist_direct_connect", h, hp.ctypes.data, ctypes.c_char_p(b"".join(blobs)), nb.value)
            dist.barrier(group=group)
        return obj

    def x_window(self):
        """DIRECT transport: this rank's exported x window as a torch tensor view (n_loc entries;
        valid while the handle lives).  Compute x there (e.g. to_permuted(D.x_window(), x)) and
        pass it to spmv to skip the per-call copy; rewrite it only between calls."""
        import torch
        p = ctypes.c_void_p()
        call("pjds_dist_x_window", self._h, ctypes.byref(p))
        ts = "<f8" if self.dtype == PJDS_F64 else "<f4"
        return torch.as_tensor(_DeviceArray(p.value or 0, self.n_loc, ts), device="cuda")

    def p2p_timed_out(self) -> bool:
        v = ctypes.c_int32()
        call("pjds_dist_p2p_check", self._h, ctypes.byref(v))
        return bool(v.value)

    @classmethod
    def create_group(cls, n, rowptr, col, val, offsets, block_rows: int = 32, permuted: bool = False):
        """All ranks in THIS process (PJDS_TRANSPORT_LOCAL; halo by device copies) — test harness
        for the split data path on a single GPU.  Returns a list of per-rank handles."""
        rowptr, col, val = _crs(rowptr, col, val)
        offsets = np.asarray(offsets, np.int64)
        R = len(offsets) - 1
        plans = []
        for r in range(R):
            lo, hi = offsets[r], offsets[r + 1]
            rp = rowptr[lo:hi + 1] - rowptr[lo]
            plans.append(DistPlan(R, r, n, offsets, rp, col[rowptr[lo]:rowptr[hi]]))
        recv = [p.recv() for p in plans]
        out = []
        for r in range(R):
            lo, hi = offsets[r], offsets[r + 1]
            # send list r -> q = q's recv list from r
            sc = np.array([recv[q][0][r] for q in range(R)], np.int64)
            parts = []
            for q in range(R):
                c, cols = recv[q]
                start = int(c[:r].sum())
                parts.append(cols[start:start + int(c[r])])
            scols = np.ascontiguousarray(np.concatenate(parts) if parts else np.zeros(0, np.int32), dtype=np.int32)
            v = np.ascontiguousarray(val[rowptr[lo]:rowptr[hi]])
            h = ctypes.c_void_p()
            call("pjds_dist_create", ctypes.byref(h), plans[r]._h, v.ctypes.data, _dt(val), int(block_rows),
                 sc.ctypes.data, scols.ctypes.data, PJDS_TRANSPORT_LOCAL, None,
                 PJDS_PERM_SYMMETRIC if permuted else 0)
            out.append(cls(h, plans[r].info, R, r, _dt(val)))
        for p in plans:
            p.close()
        return out

    @staticmethod
    def group_spmv(handles, ys, xs, stream=None, no_overlap=False):
        R = len(handles)
        H = (ctypes.c_void_p * R)(*[h._h.value for h in handles])
        Y = (ctypes.c_void_p * R)(*[_check_vec(y, h.n_loc, h.dtype, "y").value for y, h in zip(ys, handles)])
        X = (ctypes.c_void_p * R)(*[_check_vec(x, h.n_loc, h.dtype, "x").value for x, h in zip(xs, handles)])
        call("pjds_dist_group_spmv", H, R, Y, X, _stream_ptr(stream), PJDS_NO_OVERLAP if no_overlap else 0)

    def spmv(self, y_loc, x_loc, stream=None, no_overlap: bool = False, trace: bool = False):
        call("pjds_dist_spmv", self._h, _check_vec(y_loc, self.n_loc, self.dtype, "y"),
             _check_vec(x_loc, self.n_loc, self.dtype, "x"), _stream_ptr(stream),
             (PJDS_NO_OVERLAP if no_overlap else 0) | (_lib.PJDS_TRACE if trace else 0))
        return y_loc

    def trace(self):
        """Phase times (ms) of the last traced spmv: total, local, pack, exchange, wait, nonlocal."""
        ms = np.zeros(6)
        call("pjds_dist_trace", self._h, ms.ctypes.data)
        return dict(zip(("total", "local", "pack", "exchange", "wait", "nonlocal"), ms.tolist()))

    def to_permuted(self, dst, src, stream=None):
        call("pjds_dist_permute", self._h, _check_vec(dst, self.n_loc, self.dtype, "dst"),
             _check_vec(src, self.n_loc, self.dtype, "src"), 0, _stream_ptr(stream))
        return dst

    def from_permuted(self, dst, src, stream=None):
        call("pjds_dist_permute", self._h, _check_vec(dst, self.n_loc, self.dtype, "dst"),
             _check_vec(src, self.n_loc, self.dtype, "src"), 1, _stream_ptr(stream))
        return dst

    def stats(self) -> dict:
        """pjds_dist_stats: the dist info plus entries received from / sent to each peer."""
        inf = _lib.DistInfo()
        recv = np.zeros(self.nranks, np.int64)
        send = np.zeros(self.nranks, np.int64)
        call("pjds_dist_stats", self._h, ctypes.byref(inf), recv.ctypes.data, send.ctypes.data)
        d = struct_dict(inf)
        d["recv_per_peer"], d["send_per_peer"] = recv.tolist(), send.tolist()
        return d

    def parts(self):
        a, b = ctypes.c_void_p(), ctypes.c_void_p()
        call("pjds_dist_parts", self._h, ctypes.byref(a), ctypes.byref(b))
        return (PjdsMatrix(a, keep=self), PjdsMatrix(b, keep=self) if b.value else None)

    def close(self):
        if getattr(self, "_h", None):
            lib().pjds_dist_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bw_probe(nbytes: int = 4 << 30, reps: int = 5):
    """Device stream bandwidth (copy: read+write bytes; read-only), GB/s, best of `reps`."""
    c, r = ctypes.c_double(), ctypes.c_double()
    call("pjds_bw_probe", int(nbytes), int(reps), ctypes.byref(c), ctypes.byref(r))
    return c.value, r.value


def tridiag_eigenvalues(alpha, beta):
    """Ritz values: ascending eigenvalues of tridiag(beta, alpha, beta) (library bisection)."""
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    ev = np.zeros(len(a))
    call("pjds_tridiag_eigenvalues", len(a), a.ctypes.data, b.ctypes.data, ev.ctypes.data)
    return ev
