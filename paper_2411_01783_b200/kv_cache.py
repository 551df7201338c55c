"""Per-rank persistent KV store on the GPU — the SPEC's ``RankKvCache``.

Reference: SPEC.md:167-219 (module ``kv_cache``; not shipped in pkg/).  One
cache per rank holds, for every sequence, only VALID key/value rows in
ascending position order.  Storage is one HBM arena per rank
(K, V as [capacity, n_kv_heads, head_dim] bf16 plus folded int32 key
metadata), each sequence owning a contiguous segment that grows by doubling,
so decode appends are O(1) and a sequence's history is a single contiguous
row range — exactly what the decode kernel (rcp_decode_attn) and the ring
message builder need.

Position bookkeeping lives on the host (every append comes from a plan whose
positions the host knows, or is checked once), so snapshots and ring messages
are built without device synchronisation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .attention import EmbeddingBlock, _device

__all__ = ["RankKvCache"]


@dataclass
class _Segment:
    start: int      # first arena row
    cap: int        # rows reserved
    length: int     # rows used
    max_pos: int    # largest cached position (-1 when empty)


class RankKvCache:
    """``append(seq_id, k_block, v_block) -> cached_len`` and
    ``snapshot_padded(seq_id, max_len) -> (k_block, v_block)`` as in SPEC.md:180-198."""

    def __init__(self, n_kv_heads: int, head_dim: int, capacity_tokens: int = 1 << 16,
                 dtype=torch.bfloat16, device=None):
        self.n_kv_heads = int(n_kv_heads)
        self.head_dim = int(head_dim)
        self.dtype = dtype
        self.device = device if device is not None else _device()
        self._cap = max(int(capacity_tokens), 1)
        self.k = torch.zeros((self._cap, n_kv_heads, head_dim), dtype=dtype, device=self.device)
        self.v = torch.zeros_like(self.k)
        self.pos = torch.full((self._cap,), _lib.POS_PAD_K, dtype=torch.int32, device=self.device)
        self.seq = torch.full((self._cap,), _lib.SEQ_PAD_K, dtype=torch.int32, device=self.device)
        self._used = 0
        self._segs: dict[int, _Segment] = {}

    # ---------------------------------------------------------------- storage
    def _grow_arena(self, need_rows: int):
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

    def _reserve(self, seq_id: int, extra: int) -> _Segment:
        seg = self._segs.get(seq_id)
        if seg is None:
            seg = _Segment(start=self._used, cap=0, length=0, max_pos=-1)
            self._segs[seq_id] = seg
        if seg.length + extra <= seg.cap:
            return seg
        new_cap = max(2 * seg.cap, seg.length + extra, 64)
        if seg.start + seg.cap == self._used:  # last segment: grow in place
            self._grow_arena(seg.start + new_cap)
            self._used = seg.start + new_cap
            seg.cap = new_cap
            return seg
        start = self._used
        self._grow_arena(start + new_cap)
        if seg.length:
            for t in (self.k, self.v, self.pos, self.seq):
                t[start:start + seg.length].copy_(t[seg.start:seg.start + seg.length])
        seg.start, seg.cap = start, new_cap
        self._used = start + new_cap
        return seg

    def reset(self) -> None:
        """Forget every sequence (keeps the arena allocation)."""
        self._used = 0
        self._segs.clear()

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
        self.k.index_copy_(0, rows_d, k_rows.to(self.dtype))
        self.v.index_copy_(0, rows_d, v_rows.to(self.dtype))
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
        self.k[a:a + n].copy_(k_rows.to(self.dtype))
        self.v[a:a + n].copy_(v_rows.to(self.dtype))
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
        kd[:length].copy_(self.k[start:start + length])
        vd[:length].copy_(self.v[start:start + length])
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
