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
    "rcp_vmm_granularity": (ctypes.c_int, [_i32, ctypes.POINTER(_size_t)]),
    "rcp_vmm_reserve": (ctypes.c_int, [_size_t, ctypes.POINTER(_c_void_p)]),
    "rcp_vmm_map": (ctypes.c_int, [_c_void_p, _size_t, _size_t, _i32, ctypes.POINTER(ctypes.c_uint64)]),
    "rcp_vmm_unmap": (ctypes.c_int, [_c_void_p, _size_t, _size_t, ctypes.c_uint64]),
    "rcp_vmm_free": (ctypes.c_int, [_c_void_p, _size_t]),
    "rcp_cast_f32_bf16": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _c_void_p]),
    "rcp_debug_stamp": (ctypes.c_int, [_c_void_p, _c_void_p, _i32, _c_void_p]),
    "rcp_step_select": (ctypes.c_int, [_c_void_p, _c_void_p, _i64, _c_void_p, _i64, _c_void_p]),
    "rcp_shard_scatter": (ctypes.c_int, [
        ctypes.POINTER(_c_void_p), _c_void_p, ctypes.POINTER(_i64), _i32, _i32, _i32, _i64, _c_void_p]),
    "rcp_fold_meta": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i32, _c_void_p, _c_void_p, _c_void_p]),
    "rcp_attn_version": (_i32, []),
    "rcp_attn_fwd_qk8": (ctypes.c_int, [
        _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p,
        _i64, _i64, _i32, _i32, _i32, _f32, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _c_void_p, _size_t,
        _c_void_p]),
    "rcp_decode_workspace_bytes": (_size_t, [_i64, _i32, _i64]),
    "rcp_decode_attn": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _i64, _i64,
        _i32, _i32, _i32, _f32, _c_void_p, _c_void_p, _c_void_p, _size_t, _c_void_p]),
    "rcp_decode_attn_fp8": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _i64, _i64,
        _i32, _i32, _i32, _f32, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _size_t, _c_void_p]),
    "rcp_decode_attn_routed": (ctypes.c_int, [
        _c_void_p, _c_void_p, _c_void_p, _i64, _i64, _c_void_p, _c_void_p, _i64, _i64,
        _i32, _i32, _i32, _f32, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _i32, _i64, _c_void_p, _c_void_p,
        _c_void_p, _c_void_p, _size_t, _c_void_p]),
    "rcp_p2p_epoch_advance": (ctypes.c_int, [_c_void_p, _c_void_p]),
    "rcp_p2p_put": (ctypes.c_int, [_c_void_p, _i32, _c_void_p, _size_t, _c_void_p, _c_void_p, _c_void_p,
                                    _c_void_p]),
    "rcp_p2p_signal": (ctypes.c_int, [_c_void_p, _i32, _c_void_p, _c_void_p]),
    "rcp_p2p_wait": (ctypes.c_int, [_c_void_p, _i32, _c_void_p, _c_void_p, _c_void_p]),
    "rcp_kv_quantize_e4m3": (ctypes.c_int, [
        _c_void_p, _i64, _c_void_p, _c_void_p, _i64, _i64, _i32, _i32, _c_void_p, _c_void_p]),
    "rcp_kv_dequantize_e4m3": (ctypes.c_int, [
        _c_void_p, _i64, _c_void_p, _i64, _i64, _i32, _i32, _c_void_p, _c_void_p]),
    "rcp_decode_append": (ctypes.c_int, [
        _c_void_p, _i32, _i64, _i64, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _i64, _i32, _i32, _c_void_p,
        _c_void_p, _c_void_p, _c_void_p, _c_void_p]),
    "rcp_kv_calibrate_e4m3": (ctypes.c_int, [
        _c_void_p, _i64, _i64, _i32, _i32, _c_void_p, _c_void_p, _c_void_p]),
}

_lib = None

# Kernel launches issued through this binding (per C-ABI call: rcp_attn_fwd 4 =
# two tile summaries + active lists + attention; rcp_decode_attn(_fp8) 2 =
# split-KV + combine; rcp_kv_calibrate_e4m3 2 = absmax + scale; others 1).
LAUNCHES_PER_CALL = {"rcp_attn_fwd": 4, "rcp_decode_attn": 2, "rcp_decode_attn_fp8": 2, "rcp_decode_attn_routed": 2,
                     "rcp_kv_calibrate_e4m3": 2}
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


class _PinnedRing:
    """One persistent page-locked staging arena for the small host->device
    uploads of the hot path (metadata, index maps).  Allocating page-locked
    memory (or device memory) between stream commands implicitly synchronises
    the device, so a per-call pinned block — which torch's caching host
    allocator cannot recycle while the host runs ahead of the GPU — stalls
    the copy/compute overlap.  Regions are handed out circularly; each is
    reused only after the event recorded behind its copy has completed (a host
    wait only if the host is a whole arena ahead of the device)."""

    def __init__(self, nbytes: int):
        import collections

        import torch

        self.buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self.cap = nbytes
        self.head = 0
        self.live = collections.deque()  # (start, end, event), allocation order
        self.free_events = []            # retired events, re-recorded instead of created

    def _retire(self, ev) -> None:
        self.free_events.append(ev)

    def take(self, n: int):
        n = (n + 255) // 256 * 256
        if self.head + n > self.cap:
            self.head = 0
        a, b = self.head, self.head + n
        if len(self.live) > 32:  # retire completed copies (lazily: query costs host time)
            while self.live and self.live[0][2].query():
                self._retire(self.live.popleft()[2])
        if self.live and any(s < b and a < e for s, e, _ in self.live):
            keep = type(self.live)()
            for s, e, ev in self.live:
                if s < b and a < e:
                    ev.synchronize()  # host a whole arena ahead: wait for that copy
                    self._retire(ev)
                else:
                    keep.append((s, e, ev))
            self.live = keep
        self.head = b
        return a, b

    def commit(self, a: int, b: int) -> None:
        import torch

        ev = self.free_events.pop() if self.free_events else torch.cuda.Event()
        ev.record()
        self.live.append((a, b, ev))


def _torch_dtype(arr):
    import numpy as np
    import torch

    return torch.from_numpy(np.zeros(0, dtype=np.asarray(arr).dtype)).dtype


_RING = None
_RING_BYTES = 64 << 20
_RING_MAX = 8 << 20


_META_STREAMS = {}


def _meta_stream(device):
    import torch

    key = torch.device(device).index
    s = _META_STREAMS.get(key)
    if s is None:
        s = _META_STREAMS[key] = torch.cuda.Stream(device=device)
    return s


def h2d(arr, device, out=None, side=False):
    """Host array -> device tensor (or into ``out``) without a host/device
    sync: staged through the persistent pinned ring (_PinnedRing) and copied
    with non_blocking=True.  Arrays above 8 MB get a dedicated pinned block
    instead.  A pageable source would make the copy wait for all earlier work
    on the stream.

    ``side=True`` (without ``out``) runs the copy on a dedicated metadata
    stream that depends on nothing and makes the current stream wait for it:
    copy engines serve host->device copies in submission order, so a small
    copy ordered behind the compute stream's earlier work would otherwise
    queue behind any large transfer submitted meanwhile (e.g. the next
    request's staged inputs).  It costs a few tens of microseconds of host
    time, so latency-bound paths (decode) keep the default."""
    global _RING
    import numpy as np
    import torch

    if side and out is None and torch.device(device).type == "cuda" and not torch.cuda.is_current_stream_capturing():
        cur = torch.cuda.current_stream(device)
        ms = _meta_stream(device)
        with torch.cuda.stream(ms):
            d = h2d(arr, device, out=torch.empty(np.shape(arr), dtype=_torch_dtype(arr), device=device))
            ev = torch.cuda.Event()
            ev.record(ms)
        cur.wait_event(ev)
        d.record_stream(cur)
        return d

    t = torch.from_numpy(np.ascontiguousarray(arr))
    if device is None or torch.device(device).type != "cuda":
        return t if out is None else out.copy_(t)
    nbytes = t.numel() * t.element_size()
    if nbytes == 0:
        return torch.empty(t.shape, dtype=t.dtype, device=device) if out is None else out
    if nbytes > _RING_MAX:
        staged = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        staged.copy_(t)
        return staged.to(device, non_blocking=True) if out is None else out.copy_(staged, non_blocking=True)
    if _RING is None:
        _RING = _PinnedRing(_RING_BYTES)
    a, b = _RING.take(nbytes)
    pv = _RING.buf[a:a + nbytes].view(t.dtype).view(t.shape)
    pv.copy_(t)
    d = pv.to(device, non_blocking=True) if out is None else out.copy_(pv, non_blocking=True)
    _RING.commit(a, b)
    return d
