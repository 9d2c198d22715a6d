"""ctypes binding of libpjds.so (include/pjds.h).  Argument marshalling only: every step of the
path runs in the library's C++/CUDA code.  There is no fallback: if the library is missing, every
call raises."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PJDS_LIB_PATH") or os.path.join(_HERE, "libpjds.so")  # override: dev A/B builds only

PJDS_F32, PJDS_F64 = 0, 1
PJDS_PERM_ROWS, PJDS_PERM_SYMMETRIC, PJDS_HOST_ONLY = 0, 1, 2
PJDS_TRANSPORT_NCCL, PJDS_TRANSPORT_LOCAL, PJDS_TRANSPORT_P2P, PJDS_TRANSPORT_DIRECT = 0, 1, 2, 3
PJDS_NO_OVERLAP, PJDS_TRACE = 1, 2
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "BAD_CSR", -3: "OOM", -4: "CUDA", -5: "NCCL", -6: "UNSUPPORTED"}

c_i64, c_i32, c_u32, c_p, c_dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_double


class PjdsInfo(ctypes.Structure):
    _fields_ = [("n", c_i64), ("nnz", c_i64), ("n_pad", c_i64), ("n_blocks", c_i64), ("stored", c_i64),
                ("block_rows", c_i32), ("width", c_i32), ("dtype", c_i32), ("flags", c_i32),
                ("len_min", c_i32), ("len_max", c_i32), ("len_mean", c_dbl),
                ("useful_fma", c_i64), ("padded_fma", c_i64), ("idle_lane_slots", c_i64),
                ("bytes_values", c_i64), ("bytes_indices", c_i64), ("bytes_aux", c_i64), ("bytes_total", c_i64),
                ("data_reduction_vs_ellpack", c_dbl), ("on_device", c_i32), ("device", c_i32),
                ("sigma", c_i64), ("n_windows", c_i64), ("col_start_len", c_i64), ("col_compressible", c_i32)]


class EllrInfo(ctypes.Structure):
    _fields_ = [("n", c_i64), ("nnz", c_i64), ("n_pad", c_i64), ("stored", c_i64), ("width", c_i32), ("dtype", c_i32),
                ("useful_fma", c_i64), ("padded_fma", c_i64), ("idle_lane_slots", c_i64),
                ("bytes_values", c_i64), ("bytes_indices", c_i64), ("bytes_aux", c_i64), ("bytes_total", c_i64),
                ("on_device", c_i32), ("device", c_i32), ("col_compressible", c_i32)]


class Footprint(ctypes.Structure):
    _fields_ = [("bytes_values", c_i64), ("bytes_indices", c_i64), ("bytes_col_start", c_i64),
                ("bytes_block_len", c_i64), ("bytes_perm", c_i64), ("bytes_rowmax", c_i64),
                ("bytes_total", c_i64), ("stored", c_i64), ("nnz", c_i64), ("n_pad", c_i64)]


class Stats(ctypes.Structure):
    _fields_ = [("n", c_i64), ("nnz", c_i64), ("n_pad", c_i64), ("n_blocks", c_i64), ("padding", c_i64),
                ("width", c_i32), ("block_rows", c_i32), ("len_min", c_i32), ("len_max", c_i32),
                ("len_mean", c_dbl), ("reduction_vs_ellpack", c_dbl),
                ("useful_fma", c_i64), ("padded_fma", c_i64), ("idle_lane_slots", c_i64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_loc", c_i64), ("nnz_loc", c_i64), ("nnz_local_part", c_i64), ("nnz_nonlocal_part", c_i64),
                ("rows_nonlocal", c_i64), ("halo", c_i64), ("nranks", c_i32), ("rank", c_i32)]


class DistInfo(ctypes.Structure):
    _fields_ = [("n_loc", c_i64), ("halo", c_i64), ("send_total", c_i64), ("packed_send", c_i64),
                ("rows_nonlocal", c_i64), ("nnz_local_part", c_i64), ("nnz_nonlocal_part", c_i64),
                ("nranks", c_i32), ("rank", c_i32), ("peers_send", c_i32), ("peers_recv", c_i32),
                ("send_messages", c_i32), ("recv_messages", c_i32), ("permuted", c_i32)]


def struct_dict(s) -> dict:
    return {name: getattr(s, name) for name, _ in s._fields_}


_SIGS = {
    "pjds_create_from_crs": [c_p, c_i64, c_p, c_p, c_p, ctypes.c_int, c_i32, c_u32],
    "pjds_create_from_crs_ex": [c_p, c_i64, c_p, c_p, c_p, ctypes.c_int, c_i32, c_i64, c_u32],
    "pjds_export_windows": [c_p, c_p, c_p],
    "pjds_destroy": [c_p],
    "pjds_spmv": [c_p, c_p, c_p, c_p],
    "pjds_spmv_accum": [c_p, c_p, c_p, c_p],
    "pjds_spmv_host": [c_p, c_p, c_p, c_p],
    "pjds_spmv_host_batch": [c_p, c_p, c_p, c_i32, c_p],
    "pjds_permute": [c_p, c_p, c_p, c_i32, c_p],
    "pjds_info": [c_p, c_p],
    "pjds_histogram": [c_p, c_p, c_i32],
    "pjds_footprint": [c_p, c_p],
    "pjds_stats": [c_p, c_p],
    "ellr_footprint": [c_p, c_p],
    "pjds_export": [c_p, c_p, c_p, c_p, c_p, c_p],
    "ellr_create_from_crs": [c_p, c_i64, c_p, c_p, c_p, ctypes.c_int, c_u32],
    "ellr_destroy": [c_p],
    "ellr_spmv": [c_p, c_p, c_p, c_p],
    "ellr_info": [c_p, c_p],
    "ellr_export": [c_p, c_p, c_p, c_p],
    "pjds_dist_plan": [c_p, c_i32, c_i32, c_i64, c_p, c_p, c_p],
    "pjds_dist_plan_info": [c_p, c_p],
    "pjds_dist_plan_recv": [c_p, c_p, c_p],
    "pjds_dist_plan_destroy": [c_p],
    "pjds_dist_create": [c_p, c_p, c_p, ctypes.c_int, c_i32, c_p, c_p, c_i32, c_p, c_u32],
    "pjds_dist_create_crs": [c_p, c_p, c_i32, c_i32, c_i64, c_p, c_p, c_p, c_p, ctypes.c_int, c_i32, c_u32],
    "pjds_dist_permute": [c_p, c_p, c_p, c_i32, c_p],
    "pjds_dist_spmv": [c_p, c_p, c_p, c_p, c_u32],
    "pjds_dist_group_spmv": [c_p, c_i32, c_p, c_p, c_p, c_u32],
    "pjds_dist_info": [c_p, c_p],
    "pjds_dist_stats": [c_p, c_p, c_p, c_p],
    "pjds_dist_trace": [c_p, c_p],
    "pjds_dist_p2p_export": [c_p, c_p, c_p],
    "pjds_dist_p2p_connect": [c_p, c_p, c_i64],
    "pjds_dist_p2p_check": [c_p, c_p],
    "pjds_dist_direct_positions": [c_p, c_p],
    "pjds_dist_direct_connect": [c_p, c_p, c_p, c_i64],
    "pjds_dist_x_window": [c_p, c_p],
    "pjds_dist_parts": [c_p, c_p, c_p],
    "pjds_dist_destroy": [c_p],
    "pjds_nccl_load": [ctypes.c_char_p],
    "pjds_set_dist_nl_sigma": [c_i64],
    "pjds_nccl_unique_id": [c_p],
    "pjds_bw_probe": [c_i64, c_i32, c_p, c_p],
    "pjds_set_kernel_variant": [c_i32, c_i32],
    "pjds_set_cache_policy": [c_i32, c_i32],
    "pjds_set_y_store": [c_p, c_i32],
    "pjds_set_tile_order": [c_i32],
    "pjds_set_schedule": [c_i32],
    "pjds_set_launch_overlap": [c_i32, c_i32],
    "pjds_set_compression": [c_i32],
    "pjds_set_tile_keys": [c_p, c_p, c_i64],
    "pjds_lanczos": [c_p, c_p, c_i32, c_p, c_p, c_p, c_p],
    "pjds_tridiag_eigenvalues": [c_i32, c_p, c_p, c_p],
}
EXPORTED = sorted(list(_SIGS) + ["pjds_launch_count", "pjds_last_error", "pjds_version"])

_lib = None


class PjdsError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libpjds.so (raises if it has not been built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing; build it with `python build_native.py` "
                               "(or __graft_entry__.build()). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.pjds_launch_count.restype = c_i64
        L.pjds_launch_count.argtypes = []
        L.pjds_last_error.restype = ctypes.c_char_p
        L.pjds_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def call(name: str, *args) -> None:
    L = lib()
    st = getattr(L, name)(*args)
    if st != 0:
        raise PjdsError(name, st, L.pjds_last_error().decode(errors="replace"))


def launch_count() -> int:
    return int(lib().pjds_launch_count())
