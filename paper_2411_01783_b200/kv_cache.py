"""Per-rank persistent KV store on the GPU — the SPEC's ``RankKvCache``.

Reference: SPEC.md:167-219 (module ``kv_cache``; not shipped in pkg/).  One
cache per rank holds, for every sequence, only VALID key/value rows in
ascending position order.  Storage is one HBM arena per rank
(K, V as [capacity, n_kv_heads, head_dim] bf16 plus folded int32 key
metadata), each sequence owning a contiguous segment that grows by doubling,
so decode appends are O(1) and a sequence's history is a single contiguous
row range — exactly what the decode kernel (rcp_decode_attn) and the ring
message builder need.

FP8 KV (``kv_dtype="e4m3"``; beyond the SPEC's bf16
contract): K/V rows are stored as OCP e4m3 bytes with one fp32 scale per KV
head (value = scale * e4m3; scales given, or calibrated from the first append
as absmax / 448 rounded up to a power of two, which makes e4m3 * scale exact
in bf16).  Rows are quantised on the device as they are appended
(rcp_kv_quantize_e4m3), decode reads them directly (rcp_decode_attn_fp8, half
the bytes per key), and snapshots / prefill messages dequantise them to bf16
(rcp_kv_dequantize_e4m3).  ``dtype`` stays the dtype rows are handed out in.

Position bookkeeping lives on the host (every append comes from a plan whose
positions the host knows, or is checked once), so snapshots and ring messages
are built without device synchronisation.

Growth.  On a CUDA device the arenas are CUDA-VMM reservations (``_VmmArena``:
one virtual range per array, physical memory mapped in as the cache grows), so
growing the cache never copies the cached rows, never holds an old and a new
arena at once, and never moves the base pointer that CUDA graphs and tensor
maps hold.  A sequence whose segment is full moves to a larger segment (a copy
of that sequence only, amortised by doubling); ``evict`` frees a sequence's
segment for reuse (first fit).  ``capacity_balance`` checks the SPEC's
decode capacity invariant over the ranks' caches.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .attention import EmbeddingBlock, _device

__all__ = ["RankKvCache", "capacity_balance"]


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (no ownership)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class _VmmArena:
    """A growable device array [rows, *row_shape] backed by one CUDA VMM
    virtual reservation (rcp_vmm_*): ``grow`` maps more physical memory after
    the existing rows; the base address and the existing data never move."""

    _TYPESTR = {torch.bfloat16: ("<i2", 2), torch.int32: ("<i4", 4), torch.float32: ("<f4", 4),
                torch.int64: ("<i8", 8), torch.uint8: ("|u1", 1)}

    def __init__(self, max_rows: int, row_shape, dtype, device: torch.device):
        import ctypes

        lib = _lib.load()
        self.device = device
        self.row_shape = tuple(row_shape)
        self.dtype = dtype
        self.typestr, self.elem = self._TYPESTR[dtype]
        self.row_bytes = int(np.prod(self.row_shape, dtype=np.int64)) * self.elem if self.row_shape else self.elem
        g = ctypes.c_size_t()
        _lib.check(lib.rcp_vmm_granularity(device.index, ctypes.byref(g)))
        self.gran = max(int(g.value), 2 << 20)
        # K / V map in >= 64 MB steps; the 4-byte metadata arrays in granules
        self.chunk = max(self.gran, 64 << 20) if self.row_bytes >= 64 else self.gran
        self.reserved = -(-max(max_rows, 1) * self.row_bytes // self.gran) * self.gran
        base = ctypes.c_void_p()
        _lib.check(lib.rcp_vmm_reserve(self.reserved, ctypes.byref(base)))
        self.base = int(base.value)
        self.mapped = 0
        self._maps = []  # (offset, bytes, handle)
        self.rows = 0

    def capacity_rows(self) -> int:
        return self.mapped // self.row_bytes

    def grow(self, rows: int) -> bool:
        """Map memory for at least ``rows`` rows; True if memory was added."""
        import ctypes

        need = rows * self.row_bytes
        if need <= self.mapped:
            return False
        if need > self.reserved:
            raise RuntimeError(f"KV arena reservation exhausted ({self.reserved} bytes)")
        add = max(-(-(need - self.mapped) // self.chunk) * self.chunk, self.mapped)  # at least double
        add = min(add, self.reserved - self.mapped)
        h = ctypes.c_uint64()
        _lib.check(_lib.load().rcp_vmm_map(self.base, self.mapped, add, self.device.index, ctypes.byref(h)))
        self._maps.append((self.mapped, add, int(h.value)))
        self.mapped += add
        return True

    def tensor(self) -> torch.Tensor:
        """The mapped rows as a tensor view (same base pointer every time)."""
        rows = self.capacity_rows()
        shape = (rows,) + self.row_shape
        if self.dtype == torch.bfloat16:
            t = torch.as_tensor(_CudaArray(self.base, shape, self.typestr), device=self.device)
            return t.view(torch.bfloat16)
        return torch.as_tensor(_CudaArray(self.base, shape, self.typestr), device=self.device)

    def close(self) -> None:
        lib = _lib.load()
        torch.cuda.synchronize(self.device)
        for off, nbytes, h in reversed(self._maps):
            lib.rcp_vmm_unmap(self.base, off, nbytes, h)
        self._maps = []
        if self.base:
            lib.rcp_vmm_free(self.base, self.reserved)
        self.base = 0


def capacity_balance(caches, seq_ids=None) -> dict:
    """SPEC.md:200-203 invariants over the ranks' caches: per sequence the
    cached rows summed over ranks (the Σ-invariant: every prefilled / decoded
    token is cached exactly once), and the decode capacity balance — max over
    ranks minus min over ranks of the rows a rank holds for the batch (after
    k·N decode iterations of a B-sequence batch it is at most B)."""
    ids = sorted(set(seq_ids) if seq_ids is not None else {s for c in caches for s in c.seq_ids()})
    per_rank = [sum(c.cached_len(s) for s in ids) for c in caches]
    return {"per_seq_total": {s: sum(c.cached_len(s) for c in caches) for s in ids},
            "per_rank": per_rank, "spread": max(per_rank) - min(per_rank) if per_rank else 0}


@dataclass
class _Segment:
    start: int      # first arena row
    cap: int        # rows reserved
    length: int     # rows used
    max_pos: int    # largest cached position (-1 when empty)


class RankKvCache:
    """``append(seq_id, k_block, v_block) -> cached_len`` and
    ``snapshot_padded(seq_id, max_len) -> (k_block, v_block)`` as in SPEC.md:180-198."""

    KV_DTYPES = ("bf16", "e4m3")

    def __init__(self, n_kv_heads: int, head_dim: int, capacity_tokens: int = 1 << 16,
                 dtype=torch.bfloat16, device=None, growth: str | None = None, max_tokens: int | None = None,
                 kv_dtype: str = "bf16", k_scale=None, v_scale=None):
        """``growth``: "vmm" (default on CUDA: growable virtual arenas, no copy on
        growth) or "copy" (reallocate by doubling; CPU tensors / tests).
        ``max_tokens`` bounds the VMM reservation (default: what fits in the
        device's memory).  ``kv_dtype``: "bf16" or "e4m3" (FP8 storage with
        per-KV-head ``k_scale`` / ``v_scale``: a float or one per head; None
        calibrates from the first append)."""
        if kv_dtype not in self.KV_DTYPES:
            raise ValueError(f"kv_dtype must be one of {self.KV_DTYPES}, got {kv_dtype!r}")
        self.n_kv_heads = int(n_kv_heads)
        self.head_dim = int(head_dim)
        self.dtype = dtype
        self.kv_dtype = kv_dtype
        self.fp8 = kv_dtype == "e4m3"
        self.storage_dtype = torch.uint8 if self.fp8 else dtype
        self.device = torch.device(device) if device is not None else _device()
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._cap = max(int(capacity_tokens), 1)
        if growth is None:
            growth = "vmm" if self.device.type == "cuda" else "copy"
        self.growth = growth
        self.k_scale = self.v_scale = None
        if self.fp8:
            if self.device.type != "cuda" or dtype != torch.bfloat16:
                raise ValueError("kv_dtype='e4m3' needs a CUDA device and bf16 rows")
            self.k_scale = self._scale_tensor(k_scale)
            self.v_scale = self._scale_tensor(v_scale)
        self._free: list[tuple[int, int]] = []  # (start, cap) of evicted segments
        self._used = 0
        self._segs: dict[int, _Segment] = {}
        if growth == "vmm":
            row = self.n_kv_heads * self.head_dim * torch.tensor([], dtype=self.storage_dtype).element_size()
            if max_tokens is None:
                total = torch.cuda.get_device_properties(self.device).total_memory
                max_tokens = total // (2 * row)
            max_tokens = max(int(max_tokens), self._cap)
            self._arenas = {
                "k": _VmmArena(max_tokens, (n_kv_heads, head_dim), self.storage_dtype, self.device),
                "v": _VmmArena(max_tokens, (n_kv_heads, head_dim), self.storage_dtype, self.device),
                "pos": _VmmArena(max_tokens, (), torch.int32, self.device),
                "seq": _VmmArena(max_tokens, (), torch.int32, self.device),
            }
            self._cap = 0
            self._grow_arena(max(int(capacity_tokens), 1))
        else:
            self._arenas = None
            self.k = torch.zeros((self._cap, n_kv_heads, head_dim), dtype=self.storage_dtype, device=self.device)
            self.v = torch.zeros_like(self.k)
            self.pos = torch.full((self._cap,), _lib.POS_PAD_K, dtype=torch.int32, device=self.device)
            self.seq = torch.full((self._cap,), _lib.SEQ_PAD_K, dtype=torch.int32, device=self.device)

    # ---------------------------------------------------------------- storage
    def _grow_arena(self, need_rows: int):
        if self._arenas is not None:
            if need_rows <= self._cap:
                return
            old = self._cap
            for a in self._arenas.values():
                a.grow(need_rows)
            self._cap = min(a.capacity_rows() for a in self._arenas.values())
            self.k, self.v = self._arenas["k"].tensor(), self._arenas["v"].tensor()
            self.pos, self.seq = self._arenas["pos"].tensor(), self._arenas["seq"].tensor()
            # only the new rows are initialised; cached rows are neither copied nor moved
            self.k[old:].zero_()
            self.v[old:].zero_()
            self.pos[old:].fill_(_lib.POS_PAD_K)
            self.seq[old:].fill_(_lib.SEQ_PAD_K)
            return
        new_cap = self._cap
        while new_cap < need_rows:
            new_cap *= 2
        if new_cap == self._cap:
            return
        for name, fill in (("k", 0), ("v", 0)):
            old = getattr(self, name)
            t = torch.zeros((new_cap,) + tuple(old.shape[1:]), dtype=old.dtype, device=self.device)
            t[: self._used].copy_(old[: self._used])
            setattr(self, name, t)
        for name, fill in (("pos", _lib.POS_PAD_K), ("seq", _lib.SEQ_PAD_K)):
            old = getattr(self, name)
            t = torch.full((new_cap,), fill, dtype=torch.int32, device=self.device)
            t[: self._used].copy_(old[: self._used])
            setattr(self, name, t)
        self._cap = new_cap

    def _scale_tensor(self, s):
        if s is None:
            return None
        a = np.broadcast_to(np.asarray(s, np.float32).reshape(-1), (self.n_kv_heads,)).copy()
        if not np.all(np.isfinite(a)) or np.any(a <= 0):
            raise ValueError("fp8 kv scales must be finite and positive")
        return torch.from_numpy(a).to(self.device)

    def _calibrate(self, k_rows: torch.Tensor, v_rows: torch.Tensor) -> None:
        """Per-KV-head scales (absmax / 448, rounded up to a power of two) from
        the first rows appended."""
        lib = _lib.load()
        ws = torch.empty(self.n_kv_heads, dtype=torch.int32, device=self.device)
        for name, rows in (("k_scale", k_rows), ("v_scale", v_rows)):
            if getattr(self, name) is not None:
                continue
            out = torch.empty(self.n_kv_heads, dtype=torch.float32, device=self.device)
            r = rows.reshape(rows.shape[0], -1).contiguous()
            _lib.count("rcp_kv_calibrate_e4m3")
            _lib.check(lib.rcp_kv_calibrate_e4m3(_lib.ptr(r), r.stride(0), r.shape[0], self.n_kv_heads,
                                                 self.head_dim, _lib.ptr(out), _lib.ptr(ws), _lib.stream_handle()))
            setattr(self, name, out)

    def _store(self, a: int, n: int, k_rows: torch.Tensor, v_rows: torch.Tensor, rows_d=None) -> None:
        """Write n K/V rows at arena rows a.. (or at rows_d, device int64)."""
        if not self.fp8:
            if rows_d is None:
                self.k[a:a + n].copy_(k_rows.to(self.dtype))
                self.v[a:a + n].copy_(v_rows.to(self.dtype))
            else:
                self.k.index_copy_(0, rows_d, k_rows.to(self.dtype))
                self.v.index_copy_(0, rows_d, v_rows.to(self.dtype))
            return
        if self.k_scale is None or self.v_scale is None:
            self._calibrate(k_rows, v_rows)
        lib = _lib.load()
        row = self.n_kv_heads * self.head_dim
        for arena, rows, scale in ((self.k, k_rows, self.k_scale), (self.v, v_rows, self.v_scale)):
            src = rows.to(torch.bfloat16).reshape(n, row).contiguous()
            dst = arena.data_ptr() + (0 if rows_d is not None else a * row)
            _lib.count("rcp_kv_quantize_e4m3")
            _lib.check(lib.rcp_kv_quantize_e4m3(dst, row, _lib.ptr(rows_d), _lib.ptr(src), row, n,
                                                self.n_kv_heads, self.head_dim, _lib.ptr(scale),
                                                _lib.stream_handle()))

    def store_rows(self, rows_d: torch.Tensor, k_rows: torch.Tensor, v_rows: torch.Tensor) -> None:
        """Scatter K/V rows to arena rows ``rows_d`` (device int64) in the
        cache's storage format (graph-capturable: no host work)."""
        self._store(0, int(rows_d.shape[0]), k_rows, v_rows, rows_d)

    def load_rows(self, start: int, n: int, k_out: torch.Tensor, v_out: torch.Tensor) -> None:
        """Copy arena rows [start, start+n) as ``dtype`` rows into k_out / v_out
        ([n, H, D] views; e4m3 rows are dequantised)."""
        if n == 0:
            return
        if not self.fp8:
            k_out.copy_(self.k[start:start + n])
            v_out.copy_(self.v[start:start + n])
            return
        lib = _lib.load()
        row = self.n_kv_heads * self.head_dim
        for arena, out, scale in ((self.k, k_out, self.k_scale), (self.v, v_out, self.v_scale)):
            if out.dtype != torch.bfloat16 or out.stride(0) != row or out.stride(-1) != 1:
                raise ValueError("fp8 rows dequantise into contiguous bf16 [n, H, D] rows")
            _lib.count("rcp_kv_dequantize_e4m3")
            _lib.check(lib.rcp_kv_dequantize_e4m3(_lib.ptr(out), row, arena.data_ptr() + start * row, row, n,
                                                  self.n_kv_heads, self.head_dim, _lib.ptr(scale),
                                                  _lib.stream_handle()))

    def decode_kwargs(self) -> dict:
        """Extra arguments of the decode kernel call for this cache's format."""
        return {"scales": (self.k_scale, self.v_scale)} if self.fp8 else {}

    def _reserve(self, seq_id: int, extra: int) -> _Segment:
        seg = self._segs.get(seq_id)
        if seg is None:
            seg = _Segment(start=self._used, cap=0, length=0, max_pos=-1)
            self._segs[seq_id] = seg
        if seg.length + extra <= seg.cap:
            return seg
        new_cap = max(2 * seg.cap, seg.length + extra, 64)
        if seg.cap and seg.start + seg.cap == self._used:  # last segment: grow in place
            self._grow_arena(seg.start + new_cap)
            self._used = seg.start + new_cap
            seg.cap = new_cap
            return seg
        start = self._take_free(new_cap)
        if start is None:
            start = self._used
            self._grow_arena(start + new_cap)
            self._used = start + new_cap
        if seg.length:
            for t in (self.k, self.v, self.pos, self.seq):
                t[start:start + seg.length].copy_(t[seg.start:seg.start + seg.length])
        if seg.cap:
            self._release(seg.start, seg.cap)
        seg.start, seg.cap = start, new_cap
        return seg

    def _take_free(self, rows: int):
        """First fit among evicted / vacated segments (the remainder stays free)."""
        for i, (st, cap) in enumerate(self._free):
            if cap >= rows:
                if cap > rows:
                    self._free[i] = (st + rows, cap - rows)
                else:
                    self._free.pop(i)
                return st
        return None

    def _release(self, start: int, cap: int) -> None:
        self._free.append((start, cap))
        self._free.sort()
        merged = []
        for st, cp in self._free:  # coalesce neighbours
            if merged and merged[-1][0] + merged[-1][1] == st:
                merged[-1] = (merged[-1][0], merged[-1][1] + cp)
            else:
                merged.append((st, cp))
        if merged and merged[-1][0] + merged[-1][1] == self._used:  # trailing space: shrink the used region
            self._used = merged.pop()[0]
        self._free = merged

    def evict(self, seq_id: int) -> int:
        """Drop a sequence from this rank's cache; its rows become reusable.
        Returns the number of rows freed."""
        seg = self._segs.pop(seq_id, None)
        if seg is None:
            return 0
        if seg.cap:
            self._release(seg.start, seg.cap)
        return seg.length

    def close(self) -> None:
        """Release the device memory (VMM arenas: unmap and free the reservations
        after the device has finished with them)."""
        if getattr(self, "_arenas", None) is not None:
            self.k = self.v = self.pos = self.seq = None
            for a in self._arenas.values():
                a.close()
            self._arenas = None

    def __del__(self):
        try:
            if torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
                return  # never synchronise inside a graph capture; the reservation is leaked
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown / CUDA already torn down
            pass

    def reset(self) -> None:
        """Forget every sequence (keeps the arena allocation)."""
        self._used = 0
        self._segs.clear()
        self._free = []

    def truncate(self, seq_id: int, length: int) -> None:
        """Drop every row of a sequence beyond the first `length` (restores the
        cache to an earlier turn; rows are position-sorted, so this drops the
        most recent tokens)."""
        seg = self._segs.get(seq_id)
        if seg is None or length >= seg.length:
            return
        seg.length = max(0, int(length))
        seg.max_pos = int(self.pos[seg.start + seg.length - 1].item()) if seg.length else -1

    # ---------------------------------------------------------------- SPEC API
    def cached_len(self, seq_id: int) -> int:
        seg = self._segs.get(seq_id)
        return 0 if seg is None else seg.length

    def seq_ids(self):
        return list(self._segs.keys())

    def segment(self, seq_id: int) -> tuple[int, int]:
        """(first arena row, length) of a sequence's contiguous history."""
        seg = self._segs.get(seq_id)
        return (0, 0) if seg is None else (seg.start, seg.length)

    def append(self, seq_id: int, k_block: EmbeddingBlock, v_block: EmbeddingBlock) -> int:
        """Store the VALID rows of k/v; keeps position order."""
        if tuple(k_block.data.shape) != tuple(v_block.data.shape):
            raise ValueError("k/v shape mismatch")
        if k_block.n_heads != self.n_kv_heads or k_block.head_dim != self.head_dim:
            raise ValueError(f"kv blocks are [{k_block.n_heads} x {k_block.head_dim}] but cache "
                             f"wants [{self.n_kv_heads} x {self.head_dim}]")
        keep = k_block.valid & (k_block.seq_ids == seq_id)
        idx = torch.nonzero(keep).flatten()
        pos = k_block.positions[idx]
        n = int(idx.numel())
        if n == 0:
            return self.cached_len(seq_id)
        pos_host = pos.cpu().numpy()
        return self._append_rows(seq_id, k_block.data[idx], v_block.data[idx], pos_host)

    def append_rows(self, seq_id: int, k_rows: torch.Tensor, v_rows: torch.Tensor,
                    positions: np.ndarray, positions_dev: torch.Tensor | None = None) -> int:
        """Fast path with host-known positions (no device sync): rows are valid,
        belong to seq_id and are in the given position order.  ``positions_dev``
        (int32, on the device, equal to ``positions``) saves the upload."""
        return self._append_rows(seq_id, k_rows, v_rows, np.asarray(positions, np.int64), positions_dev)

    def append_tokens(self, seq_ids, k_rows: torch.Tensor, v_rows: torch.Tensor, positions) -> None:
        """Batched decode append: row j of k_rows/v_rows is one new token of
        sequence seq_ids[j] at positions[j].  All host bookkeeping (segment
        reservation) happens first, then one scatter per arena array, so a
        decode step costs a handful of launches instead of several per token.
        Repeated sequences or out-of-order positions take the per-token path."""
        ids = [int(s) for s in seq_ids]
        pos = np.asarray(positions, np.int64).reshape(-1)
        n = len(ids)
        if n == 0:
            return
        if pos.shape[0] != n or k_rows.shape[0] != n or v_rows.shape[0] != n:
            raise ValueError("append_tokens needs one k/v row and position per sequence id")
        in_order = len(set(ids)) == n and all(
            p > (self._segs[s].max_pos if s in self._segs else -1) for s, p in zip(ids, pos))
        if not in_order:
            for j, sid in enumerate(ids):
                self._append_rows(sid, k_rows[j:j + 1], v_rows[j:j + 1], pos[j:j + 1])
            return
        rows = np.empty(n, np.int64)
        for j, sid in enumerate(ids):
            seg = self._reserve(sid, 1)
            rows[j] = seg.start + seg.length
            seg.length += 1
            seg.max_pos = int(pos[j])
        rows_d = _lib.h2d(rows, self.device)
        meta_d = _lib.h2d(np.stack([pos, np.asarray(ids, np.int64)]).astype(np.int32), self.device)
        self._store(0, n, k_rows, v_rows, rows_d)
        self.pos.index_copy_(0, rows_d, meta_d[0])
        self.seq.index_copy_(0, rows_d, meta_d[1])

    def _append_rows(self, seq_id, k_rows, v_rows, pos_host: np.ndarray, pos_dev=None) -> int:
        n = int(pos_host.shape[0])
        if n == 0:
            return self.cached_len(seq_id)
        if np.any(np.diff(pos_host) <= 0):
            order = np.argsort(pos_host, kind="stable")
            sel = _lib.h2d(order, self.device)
            k_rows, v_rows, pos_host = k_rows[sel], v_rows[sel], pos_host[order]
            pos_dev = None if pos_dev is None else pos_dev[sel]
        seg = self._reserve(seq_id, n)
        a = seg.start + seg.length
        self._store(a, n, k_rows, v_rows)
        if pos_dev is not None:
            self.pos[a:a + n].copy_(pos_dev)
        else:
            self.pos[a:a + n].copy_(_lib.h2d(pos_host.astype(np.int32), self.device))
        self.seq[a:a + n].fill_(int(seq_id))
        seg.length += n
        if pos_host[0] <= seg.max_pos:
            self._resort(seg)
        seg.max_pos = max(seg.max_pos, int(pos_host[-1]))
        return seg.length

    def _resort(self, seg: _Segment):
        a, b = seg.start, seg.start + seg.length
        order = torch.argsort(self.pos[a:b], stable=True)
        for t in (self.k, self.v, self.pos):
            t[a:b].copy_(t[a:b][order])

    def snapshot_padded(self, seq_id: int, max_len: int):
        """(k, v) blocks of the cached rows padded with invalid rows to max_len
        (SPEC.md:190-198); the cache itself is not modified."""
        start, length = self.segment(seq_id)
        if max_len < length:
            raise ValueError(f"max_len {max_len} below cached_len {length}")
        dev = self.device
        kd = torch.zeros((max_len, self.n_kv_heads, self.head_dim), dtype=self.dtype, device=dev)
        vd = torch.zeros_like(kd)
        self.load_rows(start, length, kd[:length], vd[:length])
        pos = torch.full((max_len,), -1, dtype=torch.int64, device=dev)
        pos[:length].copy_(self.pos[start:start + length].to(torch.int64))
        valid = torch.zeros(max_len, dtype=torch.bool, device=dev)
        valid[:length] = True
        seq = torch.full((max_len,), -1, dtype=torch.int64, device=dev)
        seq[:length] = int(seq_id)
        pos32 = torch.full((max_len,), _lib.POS_PAD_K, dtype=torch.int32, device=dev)
        seq32 = torch.full((max_len,), _lib.SEQ_PAD_K, dtype=torch.int32, device=dev)
        pos32[:length].copy_(self.pos[start:start + length])
        seq32[:length] = int(seq_id)
        kb = EmbeddingBlock(kd, pos, valid, seq, validate=False, n_valid=length)
        vb = EmbeddingBlock(vd, pos, valid, seq, validate=False, n_valid=length)
        kb._meta["k"] = (pos32, seq32)
        vb._meta["k"] = (pos32, seq32)
        return kb, vb
