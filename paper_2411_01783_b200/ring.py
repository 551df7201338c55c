"""Ring context-parallel protocols of arXiv 2411.01783 on B200 — the SPEC's ``ring_engine``.

Reference: SPEC.md:221-303 (not shipped in pkg/) and PAPER.md Alg. 2-4
(:283-303, :334-351, :353-370).  Two execution forms share one per-step
compute path:

* SPMD (one process per GPU): ``RingAttention(comm)`` with methods
  ``pass_kv_prefill``, ``pass_q_prefill`` and ``pass_q_decode``.  Messages are
  single flat device buffers (K | V | key metadata, or Q | query metadata) moved
  with grouped NCCL send/recv issued before the step's attention kernel, so the
  transfer of step j+1's block overlaps step j's compute; the compute stream
  waits on the transfer only before it needs the block.
* Simulated ranks (one process, one GPU, per-rank lists): ``ring_pass_kv_prefill``,
  ``ring_pass_q_prefill``, ``ring_pass_q_decode`` with the SPEC's signatures —
  the same kernels, messages read directly from the other ranks' buffers.

Merge order.  By default pass-KV folds partials in arrival order (source
ranks k, k-1, ..., k-N+1) inside the attention epilogue (rcp_attn_fwd mode
MERGE — a running merge, so no N partials are ever stored); pass-Q and decode
merge the All2All-returned partials in that same order with the same fp32
merge code, so pass-KV and pass-Q are bit-identical.
``merge_order="ascending"`` (RingAttention / the simulated drivers /
GraphedDecode) folds in ascending source rank instead — the reference's
merge_attention contract (attention.py:325-326) — bitwise
equal to merge_attention over the per-source partials; pass-KV then stores
the N partials and merges once at the end.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .attention import (EmbeddingBlock, GqaConfig, PartialAttention, _bf16, attend_into,
                        merge_rows_into)
from .kv_cache import RankKvCache
from .sharding import DecodePlan, ShardPlan, materialize_rank_block

__all__ = [
    "KvLayout",
    "QLayout",
    "RingAttention",
    "RingTopology",
    "StepTrace",
    "TorchRingComm",
    "ring_pass_kv_prefill",
    "ring_pass_q_decode",
    "ring_pass_q_prefill",
]


def _align(n: int, a: int = 256) -> int:
    return (n + a - 1) // a * a


@dataclass(frozen=True)
class RingTopology:
    """next(k) = (k+1) mod N, prev(k) = (k-1) mod N."""

    n_ranks: int

    def next(self, k: int) -> int:
        return (k + 1) % self.n_ranks

    def prev(self, k: int) -> int:
        return (k - 1) % self.n_ranks

    def source_at(self, k: int, step: int) -> int:
        """Rank whose block is resident on rank k at ring step `step`."""
        return (k - step) % self.n_ranks


@dataclass
class StepTrace:
    """Per ring step: bytes sent per rank, message kind; per call: steps."""

    records: list = field(default_factory=list)

    def add(self, step: int, rank: int, kind: str, nbytes: int, pairs: int | None = None):
        self.records.append((step, rank, kind, int(nbytes), pairs))

    @property
    def steps(self) -> int:
        return len({(r[0], r[2]) for r in self.records})

    def to_csv(self) -> str:
        lines = ["step,rank,kind,bytes,pairs"]
        for s, r, k, b, p in self.records:
            lines.append(f"{s},{r},{k},{b},{'' if p is None else p}")
        return "\n".join(lines) + "\n"


class _DevPtr:
    """A raw device address where the C-ABI wrappers expect a tensor (only
    ``data_ptr`` is used for parts, outputs and peer-mapped buffers)."""

    def __init__(self, p: int):
        self._p = int(p)

    def data_ptr(self) -> int:
        return self._p


class PeerPartials:
    """Receive buffers for pass-Q partials, one per rank, mapped on every peer.

    Rank r's buffer holds N slots of (O [S, Hq, D] fp32, LSE [S, Hq] fp32),
    slot s = the partial of r's queries against rank s's KV.  Allocated with
    rcp_ipc_alloc and opened on every other rank with rcp_ipc_open (CUDA IPC
    over NVLink), so rank s's attention kernel writes slot s of rank r's buffer
    directly — the All2All of Alg. 3 becomes the kernels' own stores."""

    def __init__(self, comm, S: int, H: int, D: int, device):
        import ctypes

        lib = _lib.load()
        n, k = comm.world, comm.rank
        self.n = n
        self.set_shape(S, H, D)
        total = self.capacity = self.bytes_for(n, S, H, D)
        own = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        with torch.cuda.device(device):
            _lib.check(lib.rcp_ipc_alloc(total, ctypes.byref(own), handle))
            handles = comm.all_gather_bytes(handle.raw)
            self.base = []
            self._opened = []
            for r in range(n):
                if r == k:
                    self.base.append(own.value)
                    continue
                p = ctypes.c_void_p()
                _lib.check(lib.rcp_ipc_open(handles[r], ctypes.byref(p)))
                self.base.append(p.value)
                self._opened.append(p.value)
        self._own = own.value
        self.device = device

    @staticmethod
    def bytes_for(n: int, S: int, H: int, D: int) -> int:
        return n * (S * H * D * 4 + _align(S * H * 4))

    def fits(self, S: int, H: int, D: int) -> bool:
        return self.bytes_for(self.n, S, H, D) <= self.capacity

    def set_shape(self, S: int, H: int, D: int) -> None:
        """Re-slot the same allocation for another (S, H, D); every rank does
        this for the same call (pass-Q messages have equal sizes), and the
        caller's stream barrier orders it after the previous call's writes."""
        self.S, self.H, self.D = S, H, D
        self.o_slot = S * H * D * 4
        self.l_slot = _align(S * H * 4)

    def o(self, owner: int, src: int) -> _DevPtr:
        return _DevPtr(self.base[owner] + src * self.o_slot)

    def lse(self, owner: int, src: int) -> _DevPtr:
        return _DevPtr(self.base[owner] + self.n * self.o_slot + src * self.l_slot)

    def close(self, comm=None) -> None:
        """Unmap the peers' buffers and free this rank's.  With ``comm`` (all
        ranks call together) every rank has finished its kernels and unmapped
        before any owner frees."""
        lib = _lib.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            for p in self._opened:
                lib.rcp_ipc_close(_DevPtr(p).data_ptr())
            self._opened = []
            if comm is not None and comm.world > 1:
                comm.stream_barrier(self.device)
                torch.cuda.synchronize()
            if self._own:
                lib.rcp_ipc_free(self._own)
        self._own = 0


@dataclass
class HostStage:
    """Inputs of one host-buffer prefill staged on the device by
    ``RingAttention.stage_host_inputs`` (copies queued, with ready events).
    k / v / q / qp / qs live in one of the ring's rotating staging slots and
    are valid for exactly one ``pass_kv_prefill_host`` call."""

    plan: ShardPlan
    k: torch.Tensor
    v: torch.Tensor
    q: torch.Tensor
    qp: torch.Tensor
    qs: torch.Tensor
    splits: list
    kv_ready: torch.cuda.Event
    q_ready: list
    slot: int
    idx: np.ndarray | None = None      # concatenated source row of every query slot (-1 pad)
    seq_off: np.ndarray | None = None  # first concatenated row of every sequence


def _slot_runs(seg: np.ndarray, seq_off: np.ndarray):
    """Split a slot range's source-row map (concatenated row index per slot,
    -1 = padding) into maximal runs: (start, end, sequence, first row in that
    sequence) for consecutive rows of one sequence, (start, end, -1, 0) for
    padding.  Vectorised: O(slots) numpy, a Python step per run only."""
    n = seg.size
    if n == 0:
        return []
    v = seg >= 0
    si = np.searchsorted(seq_off, np.where(v, seg, 0), side="right") - 1
    brk = np.ones(n, dtype=bool)
    brk[1:] = (v[1:] != v[:-1]) | (v[1:] & ((seg[1:] != seg[:-1] + 1) | (si[1:] != si[:-1])))
    starts = np.flatnonzero(brk)
    ends = np.append(starts[1:], n)
    return [(int(j), int(e), int(si[j]) if v[j] else -1, int(seg[j] - seq_off[si[j]]) if v[j] else 0)
            for j, e in zip(starts, ends)]


# ------------------------------------------------------------------ message layouts
@dataclass(frozen=True)
class KvLayout:
    """Flat KV message: K [L, Hkv, D] | V [L, Hkv, D] | pos int32 [L] | seq int32 [L]."""

    tokens: int
    n_kv_heads: int
    head_dim: int
    elem: int = 2

    @property
    def kv_bytes(self) -> int:
        return self.tokens * self.n_kv_heads * self.head_dim * self.elem

    @property
    def v_off(self) -> int:
        return _align(self.kv_bytes)

    @property
    def pos_off(self) -> int:
        return self.v_off + _align(self.kv_bytes)

    @property
    def seq_off(self) -> int:
        return self.pos_off + _align(4 * self.tokens)

    @property
    def nbytes(self) -> int:
        return self.seq_off + _align(4 * self.tokens)

    def views(self, buf: torch.Tensor, dtype=torch.bfloat16):
        shape = (self.tokens, self.n_kv_heads, self.head_dim)
        k = buf[: self.kv_bytes].view(dtype).view(shape)
        v = buf[self.v_off:self.v_off + self.kv_bytes].view(dtype).view(shape)
        pos = buf[self.pos_off:self.pos_off + 4 * self.tokens].view(torch.int32)
        seq = buf[self.seq_off:self.seq_off + 4 * self.tokens].view(torch.int32)
        return k, v, pos, seq


@dataclass(frozen=True)
class QLayout:
    """Flat query message: Q [S, Hq, D] | pos int32 [S] | seq int32 [S]."""

    tokens: int
    n_q_heads: int
    head_dim: int
    elem: int = 2

    @property
    def q_bytes(self) -> int:
        return self.tokens * self.n_q_heads * self.head_dim * self.elem

    @property
    def pos_off(self) -> int:
        return _align(self.q_bytes)

    @property
    def seq_off(self) -> int:
        return self.pos_off + _align(4 * self.tokens)

    @property
    def nbytes(self) -> int:
        return self.seq_off + _align(4 * self.tokens)

    def views(self, buf: torch.Tensor, dtype=torch.bfloat16):
        q = buf[: self.q_bytes].view(dtype).view(self.tokens, self.n_q_heads, self.head_dim)
        pos = buf[self.pos_off:self.pos_off + 4 * self.tokens].view(torch.int32)
        seq = buf[self.seq_off:self.seq_off + 4 * self.tokens].view(torch.int32)
        return q, pos, seq


MERGE_ORDERS = ("arrival", "ascending")


def merge_order_of(rank: int, n: int, mode: str = "arrival") -> list:
    """Source ranks in the order their partials are folded.  "arrival" (the
    default, k, k-1, ..., k-N+1) is the order a pass-KV ring sees its KV blocks,
    so the running merge fused into the attention epilogue needs no partials
    stored; "ascending" (0..N-1) is the reference contract of merge_attention
    (attention.py:325-326) — bitwise identical to
    merge_attention over the per-source partials, at the cost of storing the
    N partials (pass-KV) before one merge."""
    if mode == "ascending":
        return list(range(n))
    if mode != "arrival":
        raise ValueError(f"merge order must be one of {MERGE_ORDERS}, got {mode!r}")
    return [(rank - j) % n for j in range(n)]


def kv_message_len(plan: ShardPlan) -> int:
    """Equal-size KV message per rank: sum_i L^i (Alg. 2 line 2, sharding.py:95-103)."""
    return plan.message_token_slots()


def build_kv_message(plan: ShardPlan, cache: RankKvCache, buf: torch.Tensor | None = None):
    """Per sequence i: [cached rows (position-sorted) | padding] up to L^i (Alg. 2)."""
    lay = KvLayout(kv_message_len(plan), cache.n_kv_heads, cache.head_dim)
    if buf is None:
        buf = torch.empty(lay.nbytes, dtype=torch.uint8, device=cache.device)
    k, v, pos, seq = lay.views(buf, cache.dtype)
    off = 0
    for i, sh in enumerate(plan.sequences):
        L = plan.padded_len(i)
        start, n = cache.segment(sh.spec.seq_id)
        if n > L:
            raise ValueError(f"sequence {sh.spec.seq_id}: cache holds {n} rows > L^i = {L}")
        if n:
            cache.load_rows(start, n, k[off:off + n], v[off:off + n])
            pos[off:off + n].copy_(cache.pos[start:start + n])
            seq[off:off + n].copy_(cache.seq[start:start + n])
        if L > n:
            k[off + n:off + L].zero_()
            v[off + n:off + L].zero_()
            pos[off + n:off + L].fill_(_lib.POS_PAD_K)
            seq[off + n:off + L].fill_(_lib.SEQ_PAD_K)
        off += L
    return lay, buf


def append_new_tokens(plan: ShardPlan, rank: int, cache: RankKvCache, k_block: EmbeddingBlock,
                      v_block: EmbeddingBlock, slot_pos: torch.Tensor | None = None) -> None:
    """Append this rank's valid new K/V to its cache BEFORE the ring.
    Positions are host-known from the plan, so no device sync is needed;
    ``slot_pos`` (the block's folded int32 slot positions, already on the
    device) supplies them without an upload."""
    off = 0
    for i, sh in enumerate(plan.sequences):
        loc = plan.rank_local_indices(i, rank)
        slots = np.nonzero(loc >= 0)[0]
        if slots.size:
            pd = None
            if slots[-1] - slots[0] + 1 == slots.size:  # contiguous: plain slice
                a, b = off + int(slots[0]), off + int(slots[-1]) + 1
                kr, vr = k_block.data[a:b], v_block.data[a:b]
                if slot_pos is not None:
                    pd = slot_pos[a:b]
            else:
                rows = _lib.h2d(slots + off, k_block.data.device, side=True)
                kr, vr = k_block.data[rows], v_block.data[rows]
                if slot_pos is not None:
                    pd = slot_pos[rows]
            cache.append_rows(sh.spec.seq_id, kr, vr, sh.spec.cached_len + loc[slots], pd)
        off += loc.size


# ------------------------------------------------------------------ transport
class TorchRingComm:
    """Ring transport over torch.distributed (NCCL between GPUs; gloo works for
    CPU tests).  P2P ops are issued on the current stream's order: NCCL's stream
    waits for work already queued, so a transfer issued before a step's kernel
    overlaps it; ``wait`` makes the current stream wait for the transfer."""

    def __init__(self, group=None, timeout_s: float | None = None):
        import datetime
        import os

        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.topo = RingTopology(self.world)
        # Deadline of one ring transfer.  Host-blocking backends (gloo) raise
        # when it passes; for NCCL ``wait`` only orders the stream, and the
        # process group's watchdog (init_process_group(timeout=...)) enforces
        # the deadline on the device side, while ``wait_done`` below gives a
        # host-side deadline that aborts the communicator.
        t = timeout_s if timeout_s is not None else float(os.environ.get("RCP_COMM_TIMEOUT_S", "600"))
        self.timeout_s = t
        self._timeout = datetime.timedelta(seconds=t)
        self._stream_ordered = dist.get_backend(group) == "nccl"

    def _g(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def stream_barrier(self, device) -> None:
        """All ranks' work queued so far on their current streams completes
        before work queued after this on any rank (a one-element NCCL
        all-reduce on the stream; no host synchronisation)."""
        t = getattr(self, "_bar_t", None)
        if t is None or t.device != device:
            t = self._bar_t = torch.zeros(1, dtype=torch.int32, device=device)
        self.dist.all_reduce(t, group=self.group)

    def all_gather_bytes(self, data: bytes) -> list:
        out = [None] * self.world
        self.dist.all_gather_object(out, data, group=self.group)
        return out

    def exchange(self, send: torch.Tensor, recv: torch.Tensor):
        d = self.dist
        ops = [d.P2POp(d.isend, send, self._g(self.topo.next(self.rank)), self.group),
               d.P2POp(d.irecv, recv, self._g(self.topo.prev(self.rank)), self.group)]
        return d.batch_isend_irecv(ops)

    def all_to_all(self, sends: list, recvs: list):
        """sends[r] -> rank r, recvs[r] <- rank r; own entry copied locally
        (N-1 pairwise exchanges in one fixed schedule)."""
        d = self.dist
        ops = []
        for r in range(self.world):
            if r == self.rank:
                continue
            ops.append(d.P2POp(d.isend, sends[r], self._g(r), self.group))
            ops.append(d.P2POp(d.irecv, recvs[r], self._g(r), self.group))
        works = d.batch_isend_irecv(ops) if ops else []
        recvs[self.rank].copy_(sends[self.rank])
        return works

    def all_gather(self, inp: torch.Tensor, out: torch.Tensor):
        """out = concat over ranks of inp (out.shape[0] = world * inp.shape[0])."""
        m = inp.shape[0]
        w = self.dist.all_gather([out[r * m:(r + 1) * m] for r in range(self.world)], inp,
                                 group=self.group, async_op=True)
        return [w]

    def all_to_all_many(self, pairs):
        """Several All2Alls in ONE grouped launch: pairs = [(sends, recvs), ...]."""
        d = self.dist
        ops = []
        for sends, recvs in pairs:
            for r in range(self.world):
                if r == self.rank:
                    continue
                ops.append(d.P2POp(d.isend, sends[r], self._g(r), self.group))
                ops.append(d.P2POp(d.irecv, recvs[r], self._g(r), self.group))
        works = d.batch_isend_irecv(ops) if ops else []
        for sends, recvs in pairs:
            recvs[self.rank].copy_(sends[self.rank])
        return works

    def wait(self, works):
        if self._stream_ordered:
            # NCCL: make the current stream wait, never the host (a timed wait
            # would block the host until the transfer lands and serialise the
            # ring); deadlines are the watchdog's / wait_done's job
            for w in works or []:
                w.wait()
            return
        for w in works or []:
            try:
                ok = w.wait(self._timeout)
            except RuntimeError as e:
                ok = False
                err = e
            else:
                err = None
            if not ok:
                self.abort()
                raise RuntimeError(f"ring transfer not complete after {self.timeout_s} s (peer hung?); "
                                   "communicator aborted") from err

    def abort(self) -> None:
        """Abort the communicator (a hung peer must not block this rank forever)."""
        from torch.distributed.distributed_c10d import _abort_process_group

        try:
            _abort_process_group(self.group)
        except Exception:  # noqa: BLE001 - best effort; the caller raises anyway
            pass

    def wait_done(self, event, timeout_s: float | None = None, poll_s: float = 1e-3) -> None:
        """Host-side deadline for stream work (e.g. an event recorded after a
        ring step): poll until it completes; past the deadline abort the
        communicator and raise instead of blocking forever."""
        import time

        limit = time.monotonic() + (self.timeout_s if timeout_s is None else timeout_s)
        while not event.query():
            if time.monotonic() > limit:
                self.abort()
                raise RuntimeError("ring step did not complete before the deadline; communicator aborted")
            time.sleep(poll_s)


# ------------------------------------------------------------------ compute hooks
def _cuda_attend(q, q_pos, q_seq, k, v, k_pos, k_seq, cfg: GqaConfig, out, lse, mode, ws=None):
    attend_into(q, (q_pos, q_seq), k, v, (k_pos, k_seq), cfg.n_query_heads, cfg.n_kv_heads,
                cfg.scale, out, lse, mode, ws)


class Fp8QkAttend:
    """Attention callable for ``RingAttention(comm, attend=Fp8QkAttend())``:
    every ring step's Q range and received K block are quantised to e4m3 with
    per-head scales (calibrated per call) and the step runs the FP8-QK kernel
    (rcp_attn_fwd_qk8) — the opt-in FP8 mode of the CP prefill.  Messages,
    merges and everything else stay bf16 / fp32; the result is the bf16 ring's
    on the dequantised Q / K of each step."""

    def __call__(self, q, q_pos, q_seq, k, v, k_pos, k_seq, cfg: GqaConfig, out, lse, mode, ws=None):
        from .attention import attend_into_qk8, quantize_heads_e4m3

        q8, qs = quantize_heads_e4m3(q)
        k8, ks = quantize_heads_e4m3(k)
        attend_into_qk8(q8, qs, (q_pos, q_seq), k8, ks, v, (k_pos, k_seq), cfg.n_query_heads, cfg.n_kv_heads,
                        cfg.scale, out, lse, mode, ws)


def _cuda_merge(o_parts, l_parts, out, lse):
    merge_rows_into(o_parts, l_parts, out, lse)


def _cuda_decode(q, k_arena, v_arena, starts, lens, max_len, cfg: GqaConfig, out, lse, ws=None, scales=None):
    """Split-KV decode of q [B, Hq, D] against arena rows [starts[b], starts[b]+lens[b]).
    e4m3 arenas (uint8) take ``scales`` = (k_scale, v_scale) per KV head."""
    lib = _lib.load()
    B, H, D = q.shape
    need = lib.rcp_decode_workspace_bytes(B, H, max(max_len, 1))
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 32), dtype=torch.uint8, device=q.device)
    if k_arena.dtype == torch.uint8:
        if scales is None or scales[0] is None or scales[1] is None:
            raise ValueError("e4m3 kv arenas need (k_scale, v_scale)")
        _lib.count("rcp_decode_attn_fp8")
        _lib.check(lib.rcp_decode_attn_fp8(
            _lib.ptr(q), _lib.ptr(k_arena), _lib.ptr(v_arena), k_arena.stride(0), k_arena.shape[0],
            _lib.ptr(starts), _lib.ptr(lens), B, max(max_len, 1), H, cfg.n_kv_heads, D, float(cfg.scale),
            _lib.ptr(scales[0]), _lib.ptr(scales[1]), _lib.ptr(out), _lib.ptr(lse), _lib.ptr(ws), ws.numel(),
            _lib.stream_handle()))
        return
    _lib.count("rcp_decode_attn")
    _lib.check(lib.rcp_decode_attn(
        _lib.ptr(q), _lib.ptr(k_arena), _lib.ptr(v_arena), k_arena.stride(0), k_arena.shape[0],
        _lib.ptr(starts),
        _lib.ptr(lens), B, max(max_len, 1), H, cfg.n_kv_heads, D, float(cfg.scale), _lib.ptr(out),
        _lib.ptr(lse), _lib.ptr(ws), ws.numel(), _lib.stream_handle()))


class RingAttention:
    """SPMD ring attention for one rank.  ``attend``/``merge`` default to the
    sm_100a kernels; tests inject oracle callables to check the schedule on CPU."""

    def __init__(self, comm, attend=None, merge=None, decode=None, device=None, merge_order: str = "arrival"):
        if merge_order not in MERGE_ORDERS:
            raise ValueError(f"merge order must be one of {MERGE_ORDERS}, got {merge_order!r}")
        self.merge_mode = merge_order
        self.comm = comm
        self.attend = attend or _cuda_attend
        self.merge = merge or _cuda_merge
        self.decode = decode or _cuda_decode
        self.device = device
        self._bufs = {}
        self.trace: StepTrace | None = None
        # Measurement hook: True replaces every ring transfer by a local no-op
        # (each step re-reads this rank's own block) — same kernels and shapes,
        # used to compute the exposed-communication fraction;
        # "pregathered" runs each step on the very block the ring would
        # deliver, all-gathered once beforehand (pregather_kv), so the work of
        # every step is identical to the ring's and only the transfers go.
        self.no_comm = False
        self._pregathered = None
        # pass-Q partials written straight into the owners' peer-mapped
        # receive slots instead of an All2All (NCCL ranks on one node only)
        self.fused_a2a = False

    def _buf(self, key, nbytes, device):
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes or b.device != device:
            b = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._bufs[key] = b
        return b[:nbytes]

    # -------------------------------------------------------------- Alg. 2
    def pass_kv(self, q, q_pos, q_seq, kv_lay: KvLayout, kv_msg: torch.Tensor, cfg: GqaConfig,
                out: torch.Tensor, lse: torch.Tensor, dtype=torch.bfloat16, q_splits=None, q_ready=None,
                on_final=None):
        """Ring pass-KV over prepared buffers: q [S, Hq, D], kv_msg the local
        flat KV message.  Writes the merged (out, lse) for this rank's queries.

        ``q_splits`` [(a, b), ...] runs every ring step as one launch per query
        slot range (streamed host inputs): the first step's launch of range i
        waits for ``q_ready[i]`` (a CUDA event), and ``on_final(i)`` is called
        right after range i's last-step launch, when its rows are final."""
        n, k = self.comm.world, self.comm.rank
        dev = kv_msg.device
        splits = q_splits or [(0, q.shape[0])]
        bufs = [self._buf(("kv", 0), kv_lay.nbytes, dev), self._buf(("kv", 1), kv_lay.nbytes, dev)]
        cur = kv_msg
        pre = self._pregathered if self.no_comm == "pregathered" else None
        parts = None
        if self.merge_mode == "ascending" and n > 1:
            parts = [(torch.empty_like(out), torch.empty_like(lse)) for _ in range(n)]
        for step in range(n):
            works = None
            nxt = None
            if pre is not None:  # the block the ring would deliver, gathered beforehand
                cur = pre[(k - step) % n][: kv_lay.nbytes]
            elif step < n - 1 and self.no_comm:
                nxt = cur
            elif step < n - 1:
                nxt = bufs[step % 2]
                works = self.comm.exchange(cur, nxt)
                if self.trace is not None:
                    self.trace.add(step, k, "KV", kv_lay.nbytes)
            kk, vv, kp, ks = kv_lay.views(cur, dtype)
            mode = _lib.MODE_OVERWRITE if step == 0 else _lib.MODE_MERGE
            src = (k - step) % n
            o_dst, l_dst = out, lse
            if parts is not None:  # ascending merge order: keep this source's partial
                mode = _lib.MODE_OVERWRITE
                o_dst, l_dst = parts[src]
            for i, (a, b) in enumerate(splits):
                if step == 0 and q_ready is not None:
                    torch.cuda.current_stream().wait_event(q_ready[i])
                self.attend(q[a:b], q_pos[a:b], q_seq[a:b], kk, vv, kp, ks, cfg, o_dst[a:b], l_dst[a:b], mode)
                if step == n - 1 and on_final is not None and parts is None:
                    on_final(i)
            self.comm.wait(works)
            cur = nxt
        if parts is not None:
            self.merge([parts[s][0] for s in range(n)], [parts[s][1] for s in range(n)], out, lse)
            if on_final is not None:
                for i in range(len(splits)):
                    on_final(i)
        return out, lse

    def pregather_kv(self) -> None:
        """All-gather every rank's current local KV message (from the last
        prefill) for the "pregathered" measurement mode."""
        local = self._bufs[("kv", "local")]
        allb = torch.empty((self.comm.world, local.numel()), dtype=torch.uint8, device=local.device)
        self.comm.wait(self.comm.all_gather(local, allb.view(-1)))
        self._pregathered = [allb[r] for r in range(self.comm.world)]

    def _side_stream(self, key):
        s = self._bufs.get(("stream", key))
        if s is None:
            s = torch.cuda.Stream()
            self._bufs[("stream", key)] = s
        return s

    # Host-buffer serving path: staged inputs and device outputs live in
    # _HOST_SLOTS rotating slots guarded by events, so a request loop
    # allocates nothing after its first requests (device or page-locked
    # allocations between stream commands synchronise the device and would
    # break the copy / compute overlap).
    _HOST_SLOTS = 2

    def _slot_tensor(self, key, shape, dtype, device) -> torch.Tensor:
        t = self._bufs.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != torch.device(device):
            if t is not None and t.is_cuda:  # copy streams may still read / write the old block
                for name in ("h2d", "d2h"):
                    t.record_stream(self._side_stream(name))
            t = torch.empty(shape, dtype=dtype, device=device)
            self._bufs[key] = t
            self._bufs[("realloc",)] = True
        return t

    def _next_slot(self, kind: str) -> int:
        """Round-robin over the slots of ``kind`` that are not pending (staged
        but not yet consumed); a new slot when all are, so staging any number
        of requests ahead stays correct (steady state: _HOST_SLOTS slots)."""
        pending = self._bufs.setdefault(("slotpending", kind), set())
        n_slots = self._bufs.get(("slotcount", kind), self._HOST_SLOTS)
        ctr = self._bufs.get(("slotctr", kind), 0)
        for i in range(n_slots):
            c = (ctr + i) % n_slots
            if c not in pending:
                break
        else:
            c = n_slots
            self._bufs[("slotcount", kind)] = n_slots + 1
        self._bufs[("slotctr", kind)] = c + 1
        return c

    def stage_host_inputs(self, plan: ShardPlan, q_host, k_host, v_host, cfg: GqaConfig, device,
                          n_sub: int | None = None) -> "HostStage":
        """Queue the host->device copies of one prefill's inputs on the copy
        stream: K/V of this rank's chunks first, then its query slots in ranges
        (``n_sub``, default one per 8192 slots, at most 4), each range with a
        ready event.  The device buffers are one of two rotating staging slots
        (the copies into a slot wait for the compute that last read it), so
        staging may run one request ahead of the compute stream; the host
        tensors must stay unchanged until the copies have run."""
        from .sharding import _host_index_map

        k = self.comm.rank
        s_in = self._side_stream("h2d")
        H, D = cfg.n_query_heads, cfg.head_dim
        idx, posv, seqv = _host_index_map(plan, k)
        S = idx.shape[0]
        if n_sub is None:
            # each range is one attention launch per ring step, whose tail wave
            # is exposed; in a serving loop the next request is staged while
            # this one computes, so ranges only pace the D2H stream.  8B 128K
            # CP1 serving loop: 1110 / 1146 / 1154 / 1142 TF/s e2e with
            # 16 / 8 / 4 / 2 ranges (profiles/r02_e2e_ranges_cp1.txt)
            n_sub = min(4, max(1, S // 8192))
        step = max(256, -(-S // max(n_sub, 1)) // 256 * 256)
        splits = [(a, min(S, a + step)) for a in range(0, S, step)]
        q_host, k_host, v_host = ([t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t))
                                   for t in src] for src in (q_host, k_host, v_host))
        for name, src in (("q", q_host), ("k", k_host), ("v", v_host)):
            for sh, t in zip(plan.sequences, src):
                if t.shape[0] != sh.spec.new_len:
                    raise ValueError(f"sequence {sh.spec.seq_id}: {name} array has {t.shape[0]} rows, "
                                     f"expected new_len={sh.spec.new_len}")
        kvh = k_host[0].shape[1] if len(k_host) else cfg.n_kv_heads
        seq_off = np.cumsum([0] + [t.shape[0] for t in q_host])  # idx rows are concatenated
        slot = self._next_slot("stage")
        self._bufs[("slotpending", "stage")].add(slot)
        q = self._slot_tensor(("stage", slot, "q"), (S, H, D), torch.bfloat16, device)
        kd = self._slot_tensor(("stage", slot, "k"), (S, kvh, D), torch.bfloat16, device)
        vd = self._slot_tensor(("stage", slot, "v"), (S, kvh, D), torch.bfloat16, device)
        qp = self._slot_tensor(("stage", slot, "qp"), (S,), torch.int32, device)
        qs = self._slot_tensor(("stage", slot, "qs"), (S,), torch.int32, device)
        free = self._bufs.get(("stage", slot, "free"))
        realloc = self._bufs.pop(("realloc",), False)
        with torch.cuda.stream(s_in):
            if free is not None:  # the compute that last read this slot is done
                s_in.wait_event(free)
            if realloc:
                # a staging tensor was (re)allocated on the compute stream: its
                # memory may be a block the compute stream freed while still in
                # use by queued kernels, so the copies must follow that work
                s_in.wait_stream(torch.cuda.current_stream(device))

            def fill(dst, srcs, a, b):
                flat = dst.view(dst.shape[0], -1)
                for j, e, si, lo in _slot_runs(idx[a:b], seq_off):
                    if si < 0:
                        flat[a + j:a + e].zero_()
                    else:
                        flat[a + j:a + e].copy_(srcs[si].reshape(srcs[si].shape[0], -1)[lo:lo + e - j],
                                                non_blocking=True)

            fill(kd, k_host, 0, S)
            fill(vd, v_host, 0, S)
            # the slot positions go with the K/V: the cache append reads them
            # (append_new_tokens(slot_pos=qp)) after waiting only on kv_ready
            _lib.h2d(posv.astype(np.int32), device, out=qp)
            _lib.h2d(seqv.astype(np.int32), device, out=qs)
            kv_ready = torch.cuda.Event(enable_timing=True)  # timing: tools/e2e_loop_ranges.py
            kv_ready.record(s_in)
            q_ready = []
            for a, b in splits:
                fill(q, q_host, a, b)
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(s_in)
                q_ready.append(ev)
        return HostStage(plan, kd, vd, q, qp, qs, splits, kv_ready, q_ready, slot, idx, seq_off)

    def join_host_copies(self) -> None:
        """Order the caller's stream after every queued device->host copy."""
        torch.cuda.current_stream().wait_stream(self._side_stream("d2h"))

    def pass_kv_prefill_host(self, plan: ShardPlan, cache: RankKvCache, q_host, k_host, v_host,
                             cfg: GqaConfig, out_host: torch.Tensor, lse_host: torch.Tensor,
                             n_sub: int | None = None, staged: "HostStage | None" = None,
                             join: bool = True) -> None:
        """Alg. 2 for host-resident inputs and outputs, with the PCIe copies
        overlapped with the attention.

        q_host/k_host/v_host: per-sequence HOST tensors of the new tokens (pinned
        for asynchronous copies).  out_host [S, Hq, D] fp32 / lse_host [S, Hq]
        (pinned) receive this rank's merged result for its S query slots (the
        rows of ``materialize_rank_block``); or, given as per-sequence LISTS
        ([new_len_i, Hq, D] / [new_len_i, Hq]), the result in TOKEN order —
        each rank fills the rows of the tokens it owns (the host-side
        scatter of ``sharding.unshard``, done by the D2H copies themselves).  The inputs are staged by
        ``stage_host_inputs`` (or taken from ``staged``, queued earlier), every
        ring step runs one attention launch per query range as it lands, and
        each range's final rows go back on a second copy stream as soon as its
        last launch is queued.  The device result lives in one of two rotating
        output slots (the first launch into a slot waits for the copies that
        last read it).  With ``join`` (default) the caller's stream is
        ordered after those copies; a serving loop that stages the next
        request meanwhile passes ``join=False`` and calls ``join_host_copies``
        once at the end."""
        k = self.comm.rank
        dev = cache.device
        cur = torch.cuda.current_stream(dev)
        s_out = self._side_stream("d2h")
        st = staged if staged is not None else self.stage_host_inputs(plan, q_host, k_host, v_host, cfg, dev,
                                                                      n_sub)
        if st.plan is not plan and st.plan != plan:
            raise ValueError("staged inputs belong to a different plan")
        H, D = cfg.n_query_heads, cfg.head_dim
        S = st.q.shape[0]
        oslot = self._next_slot("out")
        out = self._slot_tensor(("out", oslot, "o"), (S, H, D), torch.float32, dev)
        lse = self._slot_tensor(("out", oslot, "lse"), (S, H), torch.float32, dev)
        ofree = self._bufs.get(("out", oslot, "free"))
        if ofree is not None:  # the D2H copies that last read this slot are done
            cur.wait_event(ofree)
        cur.wait_event(st.kv_ready)
        append_new_tokens(plan, k, cache, st.k, st.v, slot_pos=st.qp)
        lay = KvLayout(kv_message_len(plan), cache.n_kv_heads, cache.head_dim)
        msg = self._buf(("kv", "local"), lay.nbytes, dev)
        build_kv_message(plan, cache, msg)
        splits = st.splits

        token_order = isinstance(out_host, (list, tuple))
        if token_order:
            for sh, o_h, l_h in zip(plan.sequences, out_host, lse_host):
                if o_h.shape[0] != sh.spec.new_len or l_h.shape[0] != sh.spec.new_len:
                    raise ValueError(f"sequence {sh.spec.seq_id}: token-order outputs need {sh.spec.new_len} rows")

        o_dtype = (out_host[0] if token_order else out_host).dtype
        if o_dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("host outputs must be float32 or bfloat16")
        # bf16 host outputs: each final range is cast on the device (rcp_cast_f32_bf16)
        # and half the bytes cross PCIe; LSE stays fp32
        out_src = out if o_dtype == torch.float32 else self._slot_tensor(("out", oslot, "o16"), (S, H, D),
                                                                          torch.bfloat16, dev)

        def on_final(i):
            a, b = splits[i]
            if out_src is not out:
                _lib.count("rcp_cast_f32_bf16")
                _lib.check(_lib.load().rcp_cast_f32_bf16(_lib.ptr(out_src[a:b]), _lib.ptr(out[a:b]),
                                                         (b - a) * H * D, _lib.stream_handle(cur)))
            ev = torch.cuda.Event()
            ev.record(cur)
            s_out.wait_event(ev)
            with torch.cuda.stream(s_out):
                if not token_order:
                    out_host[a:b].copy_(out_src[a:b], non_blocking=True)
                    lse_host[a:b].copy_(lse[a:b], non_blocking=True)
                    return
                # token order: every run of consecutive slots of one sequence is
                # one contiguous run of that sequence's tokens (a chunk), so each
                # run is one D2H copy straight to its token rows; padding is skipped
                for j, e, si, lo in _slot_runs(st.idx[a:b], st.seq_off):
                    if si >= 0:
                        out_host[si][lo:lo + e - j].copy_(out_src[a + j:a + e], non_blocking=True)
                        lse_host[si][lo:lo + e - j].copy_(lse[a + j:a + e], non_blocking=True)

        self.pass_kv(st.q, st.qp, st.qs, lay, msg, cfg, out, lse, cache.dtype, q_splits=splits,
                     q_ready=st.q_ready, on_final=on_final)
        done = torch.cuda.Event()
        done.record(cur)
        self._bufs[("stage", st.slot, "free")] = done  # staging slot may be refilled
        self._bufs[("slotpending", "stage")].discard(st.slot)
        ofree = torch.cuda.Event()
        ofree.record(s_out)
        self._bufs[("out", oslot, "free")] = ofree
        if join:
            cur.wait_stream(s_out)

    def pass_kv_prefill(self, plan: ShardPlan, cache: RankKvCache, q_block: EmbeddingBlock,
                        k_block: EmbeddingBlock, v_block: EmbeddingBlock, cfg: GqaConfig) -> PartialAttention:
        """Alg. 2 for this rank: append new K/V to the cache, build the padded
        KV message, run the ring, return the merged partial of the rank's queries."""
        k = self.comm.rank
        append_new_tokens(plan, k, cache, k_block, v_block)
        lay = KvLayout(kv_message_len(plan), cache.n_kv_heads, cache.head_dim)
        msg = self._buf(("kv", "local"), lay.nbytes, cache.device)
        build_kv_message(plan, cache, msg)
        qd = _bf16(q_block.data)
        qp, qs = q_block.meta32("q")
        out = torch.empty((q_block.n_tokens, cfg.n_query_heads, cfg.head_dim), dtype=torch.float32,
                          device=qd.device)
        lse = torch.empty((q_block.n_tokens, cfg.n_query_heads), dtype=torch.float32, device=qd.device)
        self.pass_kv(qd, qp, qs, lay, msg, cfg, out, lse, cache.dtype)
        blk = EmbeddingBlock(out, q_block.positions, q_block.valid, q_block.seq_ids, validate=False,
                             n_valid=q_block.n_valid)
        return PartialAttention(blk, lse)

    # -------------------------------------------------------------- Alg. 3
    def _peer_partials(self, S, H, D, dev) -> PeerPartials:
        pp = self._bufs.get("peer")
        if pp is not None and pp.device == dev and pp.fits(S, H, D):
            pp.set_shape(S, H, D)
            return pp
        if pp is not None:  # grow: collective, every rank sees the same sizes
            pp.close(self.comm)
        pp = PeerPartials(self.comm, S, H, D, dev)
        self._bufs["peer"] = pp
        return pp

    def close(self) -> None:
        """Release the ring's buffers; with ``fused_a2a`` this unmaps and frees
        the peer-mapped partial buffers, so every rank must call it."""
        pp = self._bufs.pop("peer", None)
        if pp is not None:
            pp.close(self.comm)
        self._bufs.clear()
        self._pregathered = None

    def pass_q(self, q_lay: QLayout, q_msg: torch.Tensor, kk, vv, kp, ks, cfg: GqaConfig,
               out: torch.Tensor, lse: torch.Tensor, dtype=torch.bfloat16):
        """Ring pass-Q over prepared buffers, then All2All of the partials and the
        merge in pass-KV arrival order.  With ``self.fused_a2a`` (NCCL ranks on
        one NVLink domain) each step's attention writes its partial straight
        into the owner's peer-mapped receive slot instead (PeerPartials), and
        the All2All reduces to a stream-ordered barrier; the partials and the
        merge order are the same, so the result is bitwise identical."""
        n, k = self.comm.world, self.comm.rank
        dev = q_msg.device
        S, H, D = q_lay.tokens, cfg.n_query_heads, cfg.head_dim
        if self.fused_a2a and n > 1:
            pp = self._peer_partials(S, H, D, dev)
            self.comm.stream_barrier(dev)  # owners finished reading their slots (previous call)
            bufs = [self._buf(("q", 0), q_lay.nbytes, dev), self._buf(("q", 1), q_lay.nbytes, dev)]
            cur = q_msg
            for step in range(n):
                src = (k - step) % n
                works = None
                nxt = None
                if step < n - 1:
                    nxt = bufs[step % 2]
                    works = self.comm.exchange(cur, nxt)
                    if self.trace is not None:
                        self.trace.add(step, k, "Q", q_lay.nbytes)
                qq, qp, qs = q_lay.views(cur, dtype)
                # the partial of src's queries against this rank's KV goes to src's slot k
                self.attend(qq, qp, qs, kk, vv, kp, ks, cfg, pp.o(src, k), pp.lse(src, k), _lib.MODE_OVERWRITE)
                self.comm.wait(works)
                cur = nxt
            self.comm.stream_barrier(dev)  # every partial for this rank has landed
            if self.trace is not None:
                self.trace.add(n - 1, k, "A2A", 0)
            order = merge_order_of(k, n, self.merge_mode)
            self.merge([pp.o(k, s) for s in order], [pp.lse(k, s) for s in order], out, lse)
            return out, lse
        send_o = [torch.empty((S, H, D), dtype=torch.float32, device=dev) for _ in range(n)]
        send_l = [torch.empty((S, H), dtype=torch.float32, device=dev) for _ in range(n)]
        bufs = [self._buf(("q", 0), q_lay.nbytes, dev), self._buf(("q", 1), q_lay.nbytes, dev)]
        cur = q_msg
        for step in range(n):
            src = (k - step) % n
            works = None
            nxt = None
            if step < n - 1:
                nxt = bufs[step % 2]
                works = self.comm.exchange(cur, nxt)
                if self.trace is not None:
                    self.trace.add(step, k, "Q", q_lay.nbytes)
            qq, qp, qs = q_lay.views(cur, dtype)
            self.attend(qq, qp, qs, kk, vv, kp, ks, cfg, send_o[src], send_l[src], _lib.MODE_OVERWRITE)
            self.comm.wait(works)
            cur = nxt
        recv_o = [torch.empty_like(send_o[0]) for _ in range(n)]
        recv_l = [torch.empty_like(send_l[0]) for _ in range(n)]
        w1 = self.comm.all_to_all(send_o, recv_o)
        w2 = self.comm.all_to_all(send_l, recv_l)
        if self.trace is not None:
            self.trace.add(n - 1, k, "A2A", (n - 1) * (send_o[0].numel() + send_l[0].numel()) * 4)
        self.comm.wait(w1)
        self.comm.wait(w2)
        order = merge_order_of(k, n, self.merge_mode)
        self.merge([recv_o[s] for s in order], [recv_l[s] for s in order], out, lse)
        return out, lse

    def pass_q_prefill(self, plan: ShardPlan, cache: RankKvCache, q_block: EmbeddingBlock,
                       k_block: EmbeddingBlock, v_block: EmbeddingBlock, cfg: GqaConfig) -> PartialAttention:
        """Alg. 3 for this rank: KV stays resident (cache + new tokens), Q rotates."""
        k = self.comm.rank
        append_new_tokens(plan, k, cache, k_block, v_block)
        lay, msg = build_kv_message(plan, cache, self._buf(("kv", "local"),
                                                           KvLayout(kv_message_len(plan), cache.n_kv_heads,
                                                                    cache.head_dim).nbytes, cache.device))
        kk, vv, kp, ks = lay.views(msg, cache.dtype)
        qlay = QLayout(q_block.n_tokens, cfg.n_query_heads, cfg.head_dim)
        qmsg = self._buf(("q", "local"), qlay.nbytes, cache.device)
        qq, qp, qs = qlay.views(qmsg)
        qq.copy_(_bf16(q_block.data))
        p32, s32 = q_block.meta32("q")
        qp.copy_(p32)
        qs.copy_(s32)
        out = torch.empty((q_block.n_tokens, cfg.n_query_heads, cfg.head_dim), dtype=torch.float32,
                          device=cache.device)
        lse = torch.empty((q_block.n_tokens, cfg.n_query_heads), dtype=torch.float32, device=cache.device)
        self.pass_q(qlay, qmsg, kk, vv, kp, ks, cfg, out, lse)
        blk = EmbeddingBlock(out, q_block.positions, q_block.valid, q_block.seq_ids, validate=False,
                             n_valid=q_block.n_valid)
        return PartialAttention(blk, lse)

    # -------------------------------------------------------------- Alg. 4
    def pass_q_decode(self, plan: DecodePlan, cache: RankKvCache, q_tok: torch.Tensor,
                      k_tok: torch.Tensor, v_tok: torch.Tensor, positions, cfg: GqaConfig,
                      gather: bool = False):
        """Batched ring pass-Q decode for this rank.

        q_tok/k_tok/v_tok: [slots_per_rank, H, D] — this rank's assigned decode
        tokens in ``plan.assignments[rank]`` order (padded slots ignored);
        positions: their global positions.  The owner appends its tokens' K/V
        first (the query attends to itself), then queries rotate,
        every rank attends the visitors against its cached shard of their
        sequences, and an All2All returns the partials to the owner, merged in
        pass-KV arrival order.  Returns (out [slots, Hq, D], lse [slots, Hq]).

        ``gather=True`` replaces the N-1 sequential (Q, bid) ring steps by ONE
        all-gather of the (tiny) query blocks and ONE decode launch over every
        visiting query: on an NVSwitch domain all ranks are equidistant, and the
        partials and their merge order are those of the ring."""
        n, k = self.comm.world, self.comm.rank
        mine = plan.assignments[k]
        slots = plan.slots_per_rank
        if mine:
            cache.append_tokens([sid for sid, _b in mine], k_tok[: len(mine)], v_tok[: len(mine)],
                                [int(p) for p in positions[: len(mine)]])
        if gather and n > 1:
            return self._decode_gathered(plan, cache, q_tok, cfg)
        dev = cache.device
        H, D = cfg.n_query_heads, cfg.head_dim
        qlay = QLayout(slots, H, D)
        qmsg = self._buf(("dq", "local"), qlay.nbytes, dev)
        qq, _, _ = qlay.views(qmsg)
        qq.zero_()
        if mine:
            qq[: len(mine)].copy_(_bf16(q_tok[: len(mine)]))
        # per step: kv segment of every visiting slot (host-known from the plan)
        starts = np.zeros((n, slots), np.int64)
        lens = np.zeros((n, slots), np.int64)
        for step in range(n):
            src = (k - step) % n
            for j, (sid, _b) in enumerate(plan.assignments[src]):
                starts[step, j], lens[step, j] = cache.segment(sid)
        st_d = _lib.h2d(starts, dev)
        ln_d = _lib.h2d(lens, dev)
        max_len = int(lens.max()) if lens.size else 0
        send_o = [torch.empty((slots, H, D), dtype=torch.float32, device=dev) for _ in range(n)]
        send_l = [torch.empty((slots, H), dtype=torch.float32, device=dev) for _ in range(n)]
        bufs = [self._buf(("dq", 0), qlay.nbytes, dev), self._buf(("dq", 1), qlay.nbytes, dev)]
        cur = qmsg
        for step in range(n):
            src = (k - step) % n
            works = None
            nxt = None
            if step < n - 1:
                nxt = bufs[step % 2]
                works = self.comm.exchange(cur, nxt)
                if self.trace is not None:
                    self.trace.add(step, k, "Q", qlay.nbytes)
            q_cur, _, _ = qlay.views(cur)
            self.decode(q_cur, cache.k, cache.v, st_d[step], ln_d[step], max_len, cfg,
                        send_o[src], send_l[src], **cache.decode_kwargs())
            self.comm.wait(works)
            cur = nxt
        recv_o = [torch.empty_like(send_o[0]) for _ in range(n)]
        recv_l = [torch.empty_like(send_l[0]) for _ in range(n)]
        w1 = self.comm.all_to_all(send_o, recv_o)
        w2 = self.comm.all_to_all(send_l, recv_l)
        self.comm.wait(w1)
        self.comm.wait(w2)
        out = torch.empty((slots, H, D), dtype=torch.float32, device=dev)
        lse = torch.empty((slots, H), dtype=torch.float32, device=dev)
        order = merge_order_of(k, n, self.merge_mode)
        self.merge([recv_o[s] for s in order], [recv_l[s] for s in order], out, lse)
        return out, lse


    def _decode_gathered(self, plan: DecodePlan, cache: RankKvCache, q_tok, cfg: GqaConfig):
        n, k = self.comm.world, self.comm.rank
        mine = plan.assignments[k]
        slots = plan.slots_per_rank
        dev = cache.device
        H, D = cfg.n_query_heads, cfg.head_dim
        q_mine = self._buf(("dg", "q"), slots * H * D * 2, dev).view(torch.bfloat16).view(slots, H, D)
        q_mine.zero_()
        if mine:
            q_mine[: len(mine)].copy_(_bf16(q_tok[: len(mine)]))
        q_all = self._buf(("dg", "qall"), n * slots * H * D * 2, dev).view(torch.bfloat16).view(n * slots, H, D)
        wq = self.comm.all_gather(q_mine, q_all)
        if self.trace is not None:
            self.trace.add(0, k, "Q-allgather", q_mine.numel() * 2)
        # kv segment of every (source rank, slot) query on this rank's cache
        meta = np.zeros((2, n * slots), np.int64)
        for src in range(n):
            for j, (sid, _b) in enumerate(plan.assignments[src]):
                meta[0, src * slots + j], meta[1, src * slots + j] = cache.segment(sid)
        meta_d = _lib.h2d(meta, dev)
        max_len = int(meta[1].max()) if meta.size else 0
        part_o = torch.empty((n * slots, H, D), dtype=torch.float32, device=dev)
        part_l = torch.empty((n * slots, H), dtype=torch.float32, device=dev)
        self.comm.wait(wq)
        self.decode(q_all, cache.k, cache.v, meta_d[0], meta_d[1], max_len, cfg, part_o, part_l,
                    **cache.decode_kwargs())
        recv_o = torch.empty_like(part_o)
        recv_l = torch.empty_like(part_l)
        so = [part_o[s * slots:(s + 1) * slots] for s in range(n)]
        sl = [part_l[s * slots:(s + 1) * slots] for s in range(n)]
        ro = [recv_o[s * slots:(s + 1) * slots] for s in range(n)]
        rl = [recv_l[s * slots:(s + 1) * slots] for s in range(n)]
        w = self.comm.all_to_all_many([(so, ro), (sl, rl)])
        if self.trace is not None:
            self.trace.add(0, k, "A2A", (n - 1) * slots * H * (D + 1) * 4)
        self.comm.wait(w)
        out = torch.empty((slots, H, D), dtype=torch.float32, device=dev)
        lse = torch.empty((slots, H), dtype=torch.float32, device=dev)
        order = merge_order_of(k, n, self.merge_mode)
        self.merge([ro[s] for s in order], [rl[s] for s in order], out, lse)
        return out, lse


# ------------------------------------------------------------------ simulated ranks (SPEC signatures)
class _LocalComm:
    """In-process stand-in used by the simulated-rank drivers: exchanges are
    resolved by the driver, so this only carries rank/world."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    @staticmethod
    def wait(works):
        assert not works

    # A single-rank SPMD run (world 1) uses these through RingAttention: every
    # collective over one rank is the identity.
    def all_to_all(self, sends: list, recvs: list):
        assert self.world == 1, "_LocalComm collectives are for world 1"
        recvs[0].copy_(sends[0])

    def all_to_all_many(self, pairs):
        for sends, recvs in pairs:
            self.all_to_all(sends, recvs)

    def all_gather(self, inp: torch.Tensor, out: torch.Tensor):
        assert self.world == 1, "_LocalComm collectives are for world 1"
        out.copy_(inp.reshape(out.shape))


def ring_pass_kv_prefill(plan: ShardPlan, caches: list, q_blocks: list, k_blocks: list,
                         v_blocks: list, cfg: GqaConfig, trace: StepTrace | None = None,
                         merge_order: str = "arrival"):
    """Alg. 2 over N simulated ranks on one GPU.  Returns the
    per-rank merged PartialAttention list (and fills `trace` if given).
    ``merge_order="ascending"`` folds the per-source partials in ascending
    source rank (the reference contract) with one merge at the end."""
    n = plan.n_ranks
    for r in range(n):
        append_new_tokens(plan, r, caches[r], k_blocks[r], v_blocks[r])
    msgs = [build_kv_message(plan, caches[r]) for r in range(n)]
    outs = []
    for r in range(n):
        q = q_blocks[r]
        qd = _bf16(q.data)
        qp, qs = q.meta32("q")
        out = torch.empty((q.n_tokens, cfg.n_query_heads, cfg.head_dim), dtype=torch.float32, device=qd.device)
        lse = torch.empty((q.n_tokens, cfg.n_query_heads), dtype=torch.float32, device=qd.device)
        parts = {}
        for step in range(n):
            src = (r - step) % n
            lay, buf = msgs[src]
            kk, vv, kp, ks = lay.views(buf, caches[src].dtype)
            if merge_order == "ascending" and n > 1:
                parts[src] = (torch.empty_like(out), torch.empty_like(lse))
                _cuda_attend(qd, qp, qs, kk, vv, kp, ks, cfg, parts[src][0], parts[src][1], _lib.MODE_OVERWRITE)
            else:
                _cuda_attend(qd, qp, qs, kk, vv, kp, ks, cfg, out, lse,
                             _lib.MODE_OVERWRITE if step == 0 else _lib.MODE_MERGE)
            if trace is not None and step < n - 1:
                trace.add(step, r, "KV", lay.nbytes)
        if parts:
            order = merge_order_of(r, n, merge_order)
            _cuda_merge([parts[s][0] for s in order], [parts[s][1] for s in order], out, lse)
        outs.append(PartialAttention(EmbeddingBlock(out, q.positions, q.valid, q.seq_ids, validate=False,
                                                    n_valid=q.n_valid), lse))
    return outs


def ring_pass_q_prefill(plan: ShardPlan, caches: list, q_blocks: list, k_blocks: list,
                        v_blocks: list, cfg: GqaConfig, trace: StepTrace | None = None,
                        merge_order: str = "arrival"):
    """Alg. 3 over N simulated ranks: rank s computes O_r^s for
    every visiting Q_r against its resident KV; the All2All returns them and rank
    r merges in pass-KV arrival order — bit-identical to ring_pass_kv_prefill."""
    n = plan.n_ranks
    for r in range(n):
        append_new_tokens(plan, r, caches[r], k_blocks[r], v_blocks[r])
    msgs = [build_kv_message(plan, caches[r]) for r in range(n)]
    held = {}
    for s in range(n):  # resident KV rank
        lay, buf = msgs[s]
        kk, vv, kp, ks = lay.views(buf, caches[s].dtype)
        for step in range(n):
            r = (s - step) % n  # visiting query rank
            q = q_blocks[r]
            o = torch.empty((q.n_tokens, cfg.n_query_heads, cfg.head_dim), dtype=torch.float32, device=kk.device)
            l = torch.empty((q.n_tokens, cfg.n_query_heads), dtype=torch.float32, device=kk.device)
            qp, qs = q.meta32("q")
            _cuda_attend(_bf16(q.data), qp, qs, kk, vv, kp, ks, cfg, o, l, _lib.MODE_OVERWRITE)
            held[(r, s)] = (o, l)
            if trace is not None and step < n - 1:
                trace.add(step, s, "Q", QLayout(q.n_tokens, cfg.n_query_heads, cfg.head_dim).nbytes)
    outs = []
    for r in range(n):
        order = merge_order_of(r, n, merge_order)
        q = q_blocks[r]
        out = torch.empty_like(held[(r, r)][0])
        lse = torch.empty_like(held[(r, r)][1])
        _cuda_merge([held[(r, s)][0] for s in order], [held[(r, s)][1] for s in order], out, lse)
        if trace is not None:
            trace.add(n - 1, r, "A2A", (n - 1) * (out.numel() + lse.numel()) * 4)
        outs.append(PartialAttention(EmbeddingBlock(out, q.positions, q.valid, q.seq_ids, validate=False,
                                                    n_valid=q.n_valid), lse))
    return outs


def ring_pass_q_decode(plan: DecodePlan, caches: list, q_tok: torch.Tensor, k_tok: torch.Tensor,
                       v_tok: torch.Tensor, positions, cfg: GqaConfig, merge_order: str = "arrival"):
    """Alg. 4 over N simulated ranks.  q_tok/k_tok/v_tok are
    [B, H, D] in batch order; positions[b] the token's global position.
    Returns (out [B, Hq, D], lse [B, Hq]) in batch order."""
    n = plan.n_ranks
    B = len(plan.batch)
    for b, sid in enumerate(plan.batch):
        caches[plan.owner(b)].append_rows(sid, k_tok[b:b + 1], v_tok[b:b + 1], [int(positions[b])])
    H, D = cfg.n_query_heads, cfg.head_dim
    dev = caches[0].device
    qb = _bf16(q_tok).contiguous()
    out = torch.empty((B, H, D), dtype=torch.float32, device=dev)
    lse = torch.empty((B, H), dtype=torch.float32, device=dev)
    for b, sid in enumerate(plan.batch):
        owner = plan.owner(b)
        order = merge_order_of(owner, n, merge_order)
        parts_o, parts_l = [], []
        for s in order:
            start, length = caches[s].segment(sid)
            st = torch.tensor([start], dtype=torch.int64, device=dev)
            ln = torch.tensor([length], dtype=torch.int64, device=dev)
            o = torch.empty((1, H, D), dtype=torch.float32, device=dev)
            l = torch.empty((1, H), dtype=torch.float32, device=dev)
            _cuda_decode(qb[b:b + 1], caches[s].k, caches[s].v, st, ln, length, cfg, o, l,
                         **caches[s].decode_kwargs())
            parts_o.append(o)
            parts_l.append(l)
        _cuda_merge(parts_o, parts_l, out[b:b + 1], lse[b:b + 1])
    return out, lse
