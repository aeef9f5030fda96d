"""ctypes binding of libhbp.so (include/hbp.h) -- the only path to the kernels.

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  Pointers are torch CUDA tensors'
data_ptr(); the stream is torch's current stream.
"""
from __future__ import annotations

import ctypes
import os

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
# HBP_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("HBP_LIB_PATH") or os.path.join(PKG, "libhbp.so")

HBP_OK = 0
HBP_E_ARG = 1001
HBP_E_PERM = 1002
HBP_E_DUP = 1003
HBP_E_UNSUPPORTED = 1004
HBP_E_FORMAT = 1005
HBP_F32 = 0
HBP_F64 = 1
LLONG_MAX = (1 << 63) - 1

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_size_p = ctypes.POINTER(ctypes.c_size_t)


class FormatT(ctypes.Structure):
    """Mirror of hbp_format_t."""
    _fields_ = [
        ("rows", c_i64), ("cols", c_i64), ("col_width", c_i64), ("row_height", c_i64),
        ("warp_size", c_i64), ("nrb", c_i64), ("ncb", c_i64), ("nzb", c_i64), ("nnz", c_i64),
        ("dtype", ctypes.c_int32), ("exact", ctypes.c_int32),
        ("blk_br", c_vp), ("blk_bc", c_vp), ("slot_len", c_vp), ("perm", c_vp),
        ("group_start", c_vp), ("col", c_vp), ("data", c_vp), ("rb_ptr", c_vp), ("rb_blk", c_vp),
        ("phase_ptr", c_vp), ("phases", c_vp),
        ("scol", c_vp), ("hot_cols", c_vp), ("n_hot", c_i64), ("n_warm", c_i64),
        ("cold_last", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("refresh_cols", c_vp), ("refresh_slots", c_vp),
    ]


class ScheduleT(ctypes.Structure):
    """Mirror of hbp_schedule_t."""
    _fields_ = [
        ("workers", c_i64), ("fixed_count", c_i64), ("ticket", c_vp),
        ("log_worker", c_vp), ("log_kind", c_vp), ("log_start_ns", c_vp), ("log_end_ns", c_vp),
    ]


class SegT(ctypes.Structure):
    """Mirror of hbp_seg_t."""
    _fields_ = [("ctas", c_i64), ("fixed_count", c_i64), ("ticket", c_vp), ("win_lo", c_vp),
                ("win_hi", c_vp), ("win_cap", c_i64)]


MAX_PEERS = 7  # HBP_MAX_PEERS
IPC_HANDLE_BYTES = 64  # HBP_IPC_HANDLE_BYTES


class BalancedT(ctypes.Structure):
    """Mirror of hbp_balanced_t."""
    _fields_ = [("workers", c_i64), ("part_head", c_vp), ("part_tail", c_vp),
                ("cut_end", c_vp), ("counters", c_vp), ("x_hot", c_vp),
                ("slice_lo", c_vp), ("slice_g", c_vp), ("rb_done", c_vp), ("y_sumsq", c_vp),
                ("hub_min", c_i64), ("pieces", c_i64), ("fixed_elems", c_i64),
                ("ticket", c_vp), ("warp_ns", c_vp), ("cost_prefix", c_vp),
                ("warp_map", c_i64), ("tail", c_i64), ("piece_base", c_i64),
                ("n_peers", c_i64), ("y_peer", c_vp * MAX_PEERS)]


# name -> argtypes (all return int status)
_SIGS = {
    "hbp_abi_version": [],
    "hbp_struct_sizes": [c_vp],
    "hbp_last_error": [],
    "hbp_device_sm_count": [ctypes.POINTER(c_int)],
    "hbp_spmv_default_workers": [c_int, c_i64, ctypes.POINTER(c_i64)],
    "hbp_exclusive_sum_i64": [c_vp, c_vp, c_i64, c_vp, c_size_p, c_vp],
    "hbp_inclusive_sum_i64": [c_vp, c_vp, c_i64, c_vp, c_size_p, c_vp],
    "hbp_sort_pairs_u32": [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_size_p, c_vp],
    "hbp_sort_pairs_u64": [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_size_p, c_vp],
    "hbp_coo_finish_csr": [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp,
                           c_vp],
    "hbp_coo_run_heads": [c_vp, c_i64, c_vp, c_vp],
    "hbp_coo_reduce_runs": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp],
    "hbp_grid_count_runs": [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp],
    "hbp_grid_emit_runs": [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                           c_vp],
    "hbp_grid_block_heads": [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp],
    "hbp_grid_fill_slots": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                            c_vp, c_vp],
    "hbp_block_nnz": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "hbp_sample_counts": [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp],
    "hbp_hash_perm": [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp,
                      c_vp, c_vp],
    "hbp_hash_perm_empty": [c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "hbp_sort_perm": [c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp],
    "hbp_merge_comparisons": [c_vp, c_i64, c_vp, c_vp],
    "hbp_group_costs": [c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp],
    "hbp_rowstage_plan": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "hbp_hot_remap_packed": [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp],
    "hbp_spmv_rowstage": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp],
    "hbp_gather_dense_perm": [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp],
    "hbp_slot_lengths": [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                         c_vp],
    "hbp_emit": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_int,
                 c_vp, c_vp, c_vp, c_vp],
    "hbp_row_block_counts": [c_vp, c_i64, c_vp, c_vp],
    "hbp_csr_spmv": [c_vp, c_vp, c_vp, c_int, c_i64, c_vp, c_vp, c_vp],
    "hbp_block2d_spmv": [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_int, c_vp, c_vp,
                         c_vp],
    "hbp_group_stats": [c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp,
                        c_vp, c_vp, c_vp, c_vp],
    "hbp_phase_counts": [c_vp, c_i64, c_vp, c_vp],
    "hbp_phase_emit": [c_vp, c_i64, c_vp, c_vp, c_vp],
    "hbp_expand_reference": [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp,
                             c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "hbp_walk_chains": [c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                        c_vp, c_vp, c_vp, c_vp],
    "hbp_chain_lengths": [c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp],
    "hbp_combine_dense": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "hbp_spmv_blocks": [ctypes.POINTER(FormatT), ctypes.POINTER(ScheduleT), c_vp, c_vp, c_vp,
                        c_vp],
    "hbp_balanced_workers": [ctypes.POINTER(FormatT), ctypes.POINTER(c_i64)],
    "hbp_spmv_balanced": [ctypes.POINTER(FormatT), ctypes.POINTER(BalancedT), c_vp, c_vp, c_vp,
                          c_vp],
    "hbp_stream_workers": [ctypes.POINTER(FormatT), ctypes.POINTER(c_i64)],
    "hbp_stream_slices": [ctypes.POINTER(FormatT), ctypes.POINTER(BalancedT), c_vp],
    "hbp_stream_set_variant": [c_int],
    "hbp_spmv_stream": [ctypes.POINTER(FormatT), ctypes.POINTER(BalancedT), c_vp, c_vp, c_vp,
                        c_vp],
    "hbp_col_degree": [c_vp, c_i64, c_i64, c_vp, c_vp],
    "hbp_hot_capacity": [c_int, c_int, ctypes.POINTER(c_i64)],
    "hbp_hot_slots": [c_vp, c_i64, c_vp, c_vp],
    "hbp_hot_remap": [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp],
    "hbp_hot_gather": [c_vp, c_int, c_vp, c_i64, c_vp, c_vp],
    "hbp_sumsq": [c_vp, c_int, c_i64, c_vp, c_vp, c_vp],
    "hbp_sumsq_scratch": [ctypes.POINTER(c_i64)],
    "hbp_add": [c_vp, c_vp, c_int, c_i64, c_vp],
    "hbp_ipc_export": [c_vp, c_vp, ctypes.POINTER(c_i64)],
    "hbp_ipc_open": [c_vp, c_i64, ctypes.POINTER(c_vp)],
    "hbp_ipc_close": [c_vp],
    "hbp_scale": [c_vp, c_int, c_i64, c_vp, c_vp, c_vp],
    "hbp_l2_persist": [c_vp, ctypes.c_size_t, ctypes.c_float, c_vp],
    "hbp_l2_persist_reset": [c_vp],
    "hbp_l2_info": [ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
    "hbp_seg_windows": [ctypes.POINTER(FormatT), c_vp, c_vp, c_vp, c_vp],
    "hbp_seg_workers": [ctypes.POINTER(FormatT), c_i64, ctypes.POINTER(c_i64)],
    "hbp_seg_set_variant": [c_int],
    "hbp_spmv_seg": [ctypes.POINTER(FormatT), ctypes.POINTER(SegT), c_vp, c_vp, c_vp, c_vp],
    "hbp_combine": [ctypes.POINTER(FormatT), c_vp, c_vp, c_vp],
    "hbp_spmv_rowblock": [ctypes.POINTER(FormatT), c_vp, c_vp, c_vp],
    "hbp_zero_empty_rows": [ctypes.POINTER(FormatT), c_vp, c_vp],
    "hbp_expand_partial": [ctypes.POINTER(FormatT), c_vp, c_vp, c_vp],
    "hbp_to_triplets": [ctypes.POINTER(FormatT), c_vp, c_vp, c_vp, c_vp],
}

EXPORTED = tuple(_SIGS) + ("hbp_status_string",)

_lib = None


class HbpError(RuntimeError):
    """A CUDA or ABI failure inside libhbp.so."""


def load_library(path: str = LIB_PATH):
    """Load libhbp.so and declare every signature (no CUDA call is made)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2504_08860_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = c_int
    lib.hbp_status_string.argtypes = [c_int]
    lib.hbp_status_string.restype = ctypes.c_char_p
    _lib = lib
    return lib


def lib():
    if _lib is None:
        load_library()
    return _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_08860_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> c_vp:
    return c_vp(torch.cuda.current_stream().cuda_stream)


def P(t) -> c_vp:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return c_vp(0)
    return c_vp(t.data_ptr())


def call(name: str, *args) -> None:
    st = getattr(lib(), name)(*args)
    if st != HBP_OK:
        msg = lib().hbp_status_string(st).decode()
        if st == HBP_E_DUP:
            raise ValueError("duplicate (row, col) entries; canonicalize first")
        if st in (HBP_E_ARG, HBP_E_UNSUPPORTED):
            raise ValueError(f"{name}: {msg}")
        raise HbpError(f"{name} failed: {msg} (status {st})")


def temp_call(name: str, *args_before_temp, stream_arg=True, device=None):
    """Two-phase CUB call: size query with NULL temp, then the real call."""
    sz = ctypes.c_size_t(0)
    call(name, *args_before_temp, c_vp(0), ctypes.byref(sz), stream())
    tmp = torch.empty(max(1, sz.value), dtype=torch.uint8, device=device or require_cuda())
    call(name, *args_before_temp, P(tmp), ctypes.byref(sz), stream())
    return tmp


def exclusive_sum(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(x)
    if x.numel():
        temp_call("hbp_exclusive_sum_i64", P(x), P(out), c_i64(x.numel()), device=x.device)
    return out


def inclusive_sum(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(x)
    if x.numel():
        temp_call("hbp_inclusive_sum_i64", P(x), P(out), c_i64(x.numel()), device=x.device)
    return out


def sort_pairs_u32(keys: torch.Tensor, vals: torch.Tensor, end_bit: int):
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    if keys.numel():
        temp_call("hbp_sort_pairs_u32", P(keys), P(ko), P(vals), P(vo), c_i64(keys.numel()),
                  c_int(end_bit), device=keys.device)
    return ko, vo


def sort_pairs_u64(keys: torch.Tensor, vals: torch.Tensor, end_bit: int):
    ko, vo = torch.empty_like(keys), torch.empty_like(vals)
    if keys.numel():
        temp_call("hbp_sort_pairs_u64", P(keys), P(ko), P(vals), P(vo), c_i64(keys.numel()),
                  c_int(end_bit), device=keys.device)
    return ko, vo


def dtype_code(t: torch.dtype) -> int:
    if t == torch.float64:
        return HBP_F64
    if t == torch.float32:
        return HBP_F32
    raise ValueError(f"unsupported value dtype {t} (float32 or float64)")


def sm_count() -> int:
    v = c_int(0)
    call("hbp_device_sm_count", ctypes.byref(v))
    return v.value


def default_workers(dtype: torch.dtype, warp_size: int) -> int:
    v = c_i64(0)
    call("hbp_spmv_default_workers", c_int(dtype_code(dtype)), c_i64(warp_size), ctypes.byref(v))
    return int(v.value)


def l2_bytes() -> int:
    """Device L2 capacity (hbp_l2_info)."""
    l2, mp, mw = c_int(0), c_int(0), c_int(0)
    call("hbp_l2_info", ctypes.byref(l2), ctypes.byref(mp), ctypes.byref(mw))
    return int(l2.value)
