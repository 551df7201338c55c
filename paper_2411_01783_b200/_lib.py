"""ctypes binding of the in-tree C-ABI library ``_ringcp_b200.so``.

The product path has no CPU fallback: if the library is missing, or CUDA is
not available, every call raises.  Argument errors reported by the C side
(RCP_ERR_INVALID) surface as ValueError with the C message; CUDA failures as
RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# RCP_LIB_PATH selects an alternative build of the same ABI (A/B experiments, trace builds).
LIB_PATH = os.environ.get("RCP_LIB_PATH") or os.path.join(_PKG, "_ringcp_b200.so")

RCP_OK = 0
RCP_ERR_INVALID = -1
RCP_ERR_CUDA = -2
MODE_OVERWRITE = 0
MODE_MERGE = 1
SEQ_PAD_Q = -(2 ** 31)
SEQ_PAD_K = -(2 ** 31) + 1
POS_PAD_K = 2 ** 31 - 1

_c_void_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_size_t = ctypes.c_size_t
_f32 = ctypes.c_float

# name -> (restype, argtypes); mirrors include/ringcp_b200.h
SIGNATURES = {
    "rcp_ipc_alloc": (ctypes.c_int, [_size_t, ctypes.POINTER(_c_void_p), _c_void_p]),
    "rcp_ipc_free": (ctypes.c_int, [_c_void_p]),
    "rcp_ipc_open": (ctypes.c_int, [_c_void_p, ctypes.POINTER(_c_void_p)]),
    "rcp_ipc_close": (ctypes.c_int, [_c_void_p]),
    "rcp_last_error": (ctypes.c_char_p, []),
    "rcp_version": (ctypes.c_char_p, []),
    "rcp_attn_workspace_bytes": (_size_t, [_i64, _i64]),
    "rcp_attn_fwd": (ctypes.c_int, [
        _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64,
        _c_void_p, _c_void_p, _c_void_p, _c_void_p,
        _i64, _i64, _i32, _i32, _i32, _f32,
        _c_void_p, _c_void_p, _i32, _c_void_p, _size_t, _c_void_p]),
    "rcp_merge_attn": (ctypes.c_int, [
        ctypes.POINTER(_c_void_p), ctypes.POINTER(_c_void_p), _i32, _i64, _i32,
        _c_void_p, _c_void_p, _c_void_p]),
    "rcp_fill_empty": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _i32, _c_void_p]),
    "rcp_shard_gather": (ctypes.c_int, [
        _c_void_p, ctypes.POINTER(_c_void_p), ctypes.POINTER(_i64), ctypes.POINTER(_i64),
        ctypes.POINTER(_i64), _i32, _i32, _i32, _i64, _c_void_p, _c_void_p, _i32, _c_void_p]),
    "rcp_gather_rows": (ctypes.c_int, [_c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p]),
    "rcp_fold_meta": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i32, _c_void_p, _c_void_p, _c_void_p]),
    "rcp_decode_workspace_bytes": (_size_t, [_i64, _i32, _i64]),
    "rcp_decode_attn": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _i64, _i64,
        _i32, _i32, _i32, _f32, _c_void_p, _c_void_p, _c_void_p, _size_t, _c_void_p]),
}

_lib = None

# Kernel launches issued through this binding (per C-ABI call: rcp_attn_fwd 4 =
# two tile summaries + active lists + attention; rcp_decode_attn 2; others 1).
LAUNCHES_PER_CALL = {"rcp_attn_fwd": 4, "rcp_decode_attn": 2}
launch_count = 0


def count(name: str) -> None:
    global launch_count
    launch_count += LAUNCHES_PER_CALL.get(name, 1)


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"ringcp_b200 CUDA extension not built ({LIB_PATH} missing); run "
            "`python -m paper_2411_01783_b200._build` — there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == RCP_OK:
        return
    msg = load().rcp_last_error().decode()
    if rc == RCP_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"ringcp_b200 error {rc}: {msg}")


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def ptr_array(ptrs):
    arr = (_c_void_p * len(ptrs))(*ptrs)
    return arr


def i64_array(vals):
    return (_i64 * len(vals))(*[int(v) for v in vals])


def h2d(arr, device):
    """Host array -> device tensor without a host/device sync: staged through
    pinned memory (torch's caching host allocator keeps the staging block alive
    until the copy has run) and copied with non_blocking=True.  A pageable
    source would make the copy wait for all earlier work on the stream."""
    import numpy as np
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr))
    if device is None or torch.device(device).type != "cuda":
        return t
    staged = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    staged.copy_(t)
    return staged.to(device, non_blocking=True)

