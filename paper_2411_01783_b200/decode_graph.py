"""CUDA-graph replay of the batched decode step (Alg. 4 with all-gathered Q).

A decode step of a fixed batch is a fixed sequence of launches: append the
owners' new K/V rows to the cache arena, (N > 1) all-gather the ranks' query
slots, one split-KV decode launch over every visiting query against this
rank's shard, (N > 1) All2All of the partials, merge in ring-arrival order.
At small batch the step is bound by host launch overhead (~300 us of Python /
ctypes / allocator work per step at B = 1 against ~250 us of GPU time,
DESIGN.md), so ``GraphedDecode`` captures those launches once and replays
them; per step the host only does the cache bookkeeping and ONE pinned
host->device copy of the step's metadata (arena rows to append to,
per-query KV segments, positions and sequence ids of the appends).

Static shapes: the batch, its slot assignment pattern and the arena must not
change while a graph is live.  ``GraphedDecode`` reserves room for
``max_steps`` more tokens per sequence up front (so the arena never moves),
fixes the decode kernel's split bound at the reserved capacity, routes empty
slots (ranks with fewer tokens this iteration) to a scratch arena row, and
re-captures if the cache was reallocated anyway.  Results equal the eager
``RingAttention.pass_q_decode`` up to the split boundaries of the split-KV
reduction (tests/test_gpu_decode_graph.py checks both against the oracle).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .attention import GqaConfig, merge_rows_into
from .kv_cache import RankKvCache, _CudaArray
from .ring import _cuda_decode, merge_order_of
from .sharding import plan_decode

__all__ = ["GraphedDecode"]


def _lens_slice(g) -> slice:
    """Slice of the lens section in the step metadata (rows | starts | lens | pos | seq)."""
    S, R = g.slots, g.n * g.slots
    return slice(S + R, S + 2 * R)

_SCRATCH_SEQ = -7  # cache-internal sequence id of the scratch row (never a query's id)


def _align256(x: int) -> int:
    return (x + 255) // 256 * 256


class _PeerDecodeBuffers:
    """The decode step's exchange buffers in CUDA-IPC memory mapped on every
    rank (transport="p2p"): per rank one allocation holding
    q_all [N*S, Hq, D] bf16 | recv_o [N*S, Hq, D] fp32 | recv_l [N*S, Hq] fp32 |
    flags_q [N] | flags_o [N] (u64 epochs).  Rank k's put stores its query
    slots into block k of every rank's q_all, its routed decode combine stores
    the partials of rank s's queries into block k of rank s's recv_o / recv_l,
    and each phase ends with an epoch signal into slot k of every rank's flags
    and a wait on its own — the Q all-gather and the All2All without NCCL."""

    def __init__(self, comm, S: int, H: int, D: int, device):
        import ctypes

        lib = _lib.load()
        n, k = comm.world, comm.rank
        R = n * S
        self.n, self.k, self.S, self.H, self.D = n, k, S, H, D
        self.off_q = 0
        self.off_o = _align256(R * H * D * 2)
        self.off_l = self.off_o + _align256(R * H * D * 4)
        self.off_fq = self.off_l + _align256(R * H * 4)
        self.off_fo = self.off_fq + _align256(n * 8)
        total = self.off_fo + _align256(n * 8)
        own = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        self.device = device
        with torch.cuda.device(device):
            _lib.check(lib.rcp_ipc_alloc(total, ctypes.byref(own), handle))
            self._own = own.value
            torch.as_tensor(_CudaArray(self._own, (total,), "|u1"), device=device).zero_()
            torch.cuda.synchronize(device)
            handles = comm.all_gather_bytes(handle.raw)
            self.base, self._opened = [], []
            for r in range(n):
                if r == k:
                    self.base.append(self._own)
                    continue
                p = ctypes.c_void_p()
                _lib.check(lib.rcp_ipc_open(handles[r], ctypes.byref(p)))
                self.base.append(p.value)
                self._opened.append(p.value)
            comm.stream_barrier(device)  # every rank's flags are zero before anyone signals
            torch.cuda.synchronize(device)
        B = self.base
        dev_i64 = lambda xs: torch.tensor(xs, dtype=torch.int64, device=device)
        self.q_dst = dev_i64([B[p] + self.off_q + k * S * H * D * 2 for p in range(n)])
        self.o_dst = dev_i64([B[p] + self.off_o for p in range(n)])
        self.l_dst = dev_i64([B[p] + self.off_l for p in range(n)])
        self.fq_dst = dev_i64([B[p] + self.off_fq + k * 8 for p in range(n)])
        self.fo_dst = dev_i64([B[p] + self.off_fo + k * 8 for p in range(n)])
        self.epoch = torch.zeros(1, dtype=torch.int64, device=device)
        self.timed_out = torch.zeros(1, dtype=torch.int32, device=device)
        self.counters = torch.zeros(2, dtype=torch.int32, device=device)  # last-block counters: put, combine
        own_t = lambda off, shape, ts: torch.as_tensor(_CudaArray(self._own + off, shape, ts), device=device)
        self.q_all = own_t(self.off_q, (R, H, D), "<i2").view(torch.bfloat16)
        self.recv_o = own_t(self.off_o, (R, H, D), "<f4")
        self.recv_l = own_t(self.off_l, (R, H), "<f4")

    def flags(self, which: str) -> int:
        return self._own + (self.off_fq if which == "q" else self.off_fo)

    def close(self, comm) -> None:
        lib = _lib.load()
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            comm.stream_barrier(self.device)  # no rank still stores into a peer's buffer
            torch.cuda.synchronize()
            for p in self._opened:
                lib.rcp_ipc_close(p)
            self._opened = []
            comm.stream_barrier(self.device)  # every peer unmapped before the owner frees
            torch.cuda.synchronize()
            if self._own:
                lib.rcp_ipc_free(self._own)
            self._own = 0


class GraphedDecode:
    """Replayable decode step for ``batch`` on this rank.

    ``step(q_tok, k_tok, v_tok, positions)`` takes this rank's tokens of the
    current iteration in ``plan_decode(batch, N, it).assignments[rank]`` order
    (as ``RingAttention.pass_q_decode``) and returns views of the static
    (out [slots, Hq, D], lse [slots, Hq]) buffers, valid until the next step.
    """

    TRANSPORTS = ("nccl", "p2p")

    def __init__(self, comm, cache: RankKvCache, cfg: GqaConfig, batch, max_steps: int = 256,
                 first_iteration: int = 0, first_positions=None, merge_order: str = "arrival",
                 grouped_a2a: bool = True, transport: str = "nccl"):
        """``transport``: "nccl" (Q all-gather + grouped All2All through
        torch.distributed) or "p2p" (N > 1 on one NVLink domain: the Q put and
        the partials stored straight into the peers' CUDA-IPC buffers by the
        kernels, with device-side epoch flags; construct it and call
        ``close()`` on every rank together — both are collective)."""
        if transport not in self.TRANSPORTS:
            raise ValueError(f"transport must be one of {self.TRANSPORTS}, got {transport!r}")
        if cache.device.type != "cuda":
            raise RuntimeError("GraphedDecode needs the cache on a CUDA device")
        if getattr(cache, "fp8", False) and (cache.k_scale is None or cache.v_scale is None):
            raise ValueError("e4m3 cache has no k/v scales yet: prefill (or pass scales) before capturing")
        self.comm, self.cache, self.cfg = comm, cache, cfg
        merge_order_of(0, 1, merge_order)  # validates the mode
        self.merge_mode = merge_order
        self.grouped_a2a = grouped_a2a
        self.transport = transport if comm.world > 1 else "nccl"
        self.batch = [int(b) for b in batch]
        self.n, self.rank = comm.world, comm.rank
        self.it = int(first_iteration)
        self.slots = math.ceil(len(self.batch) / self.n)
        self.max_steps = int(max_steps)
        self.steps_left = self.max_steps
        dev = cache.device
        H, Hkv, D = cfg.n_query_heads, cfg.n_kv_heads, cfg.head_dim
        S, R = self.slots, self.n * self.slots
        # room for every future token of this graph's lifetime (owner rotation
        # gives each rank about max_steps / N of them per sequence), plus a
        # scratch row that absorbs the appends of empty slots
        per_seq = math.ceil(self.max_steps / self.n) + 1
        for sid in self.batch:
            cache._reserve(sid, per_seq)
        cache._reserve(_SCRATCH_SEQ, 1)
        self.scratch_row = cache.segment(_SCRATCH_SEQ)[0]
        self.max_len = max(cache._segs[s].cap for s in self.batch)
        # static buffers (graph inputs / outputs)
        self.q_in = torch.zeros((S, H, D), dtype=torch.bfloat16, device=dev)
        self.k_in = torch.zeros((S, Hkv, D), dtype=cache.dtype, device=dev)
        self.v_in = torch.zeros_like(self.k_in)
        # rows | starts | lens | pos | seq (one host->device copy per step)
        self.meta = torch.zeros(S + 2 * R + 2 * S, dtype=torch.int64, device=dev)
        self.q_all = torch.zeros((R, H, D), dtype=torch.bfloat16, device=dev)
        self.part_o = torch.empty((R, H, D), dtype=torch.float32, device=dev)
        self.part_l = torch.empty((R, H), dtype=torch.float32, device=dev)
        self.recv_o = torch.empty_like(self.part_o)
        self.recv_l = torch.empty_like(self.part_l)
        self.out = torch.empty((S, H, D), dtype=torch.float32, device=dev)
        self.lse = torch.empty((S, H), dtype=torch.float32, device=dev)
        lib = _lib.load()
        self.ws = torch.empty(max(int(lib.rcp_decode_workspace_bytes(R, H, self.max_len)), 32),
                              dtype=torch.uint8, device=dev)
        self.peer = _PeerDecodeBuffers(comm, S, H, D, dev) if self.transport == "p2p" else None
        self._mine_cache = {}
        import os

        self._stamps = (torch.zeros(4097, dtype=torch.int64, device=dev)
                        if os.environ.get("RCP_DECODE_STAMPS") == "1" else None)
        self.graph = None
        self._arena_ptr = None
        self._segs_at_capture = None
        # Device-resident step metadata: with the sequences' next global
        # positions known (every sequence decodes one token per step), the
        # metadata of every future step is precomputed once and the graph's
        # first launch selects the current row (rcp_step_select) — no
        # host->device upload and no metadata work on the host per step.
        self._table = None
        self._pos_next = None
        if first_positions is not None:
            self._pos_next = {int(sid): int(first_positions[sid]) for sid in self.batch}
            self._build_table()

    def _segment_key(self):
        """(start, capacity) of every batch sequence's arena segment: the
        captured decode launch's split bound (max_len) covers these only."""
        return tuple((self.cache._segs[s].start, self.cache._segs[s].cap) for s in self.batch)

    def _refit(self) -> None:
        """Re-derive the split bound and workspace from the current segments
        (a segment moved or grew between steps, e.g. an eager append)."""
        self.max_len = max(self.cache._segs[s].cap for s in self.batch)
        need = int(_lib.load().rcp_decode_workspace_bytes(self.n * self.slots, self.cfg.n_query_heads,
                                                          self.max_len))
        if self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.cache.device)

    def _build_table(self) -> None:
        """Metadata rows (rows | starts | lens | pos | seq) of steps self.it ..
        self.it + steps_left - 1, simulated from the current segments."""
        c, S, n = self.cache, self.slots, self.n
        steps = max(self.steps_left, 1)
        sim = {sid: [c._segs[sid].start, c._segs[sid].length, c._segs[sid].cap] for sid in self.batch}
        pos = dict(self._pos_next)
        table = np.empty((steps, self.meta.numel()), np.int64)
        for k in range(steps):
            plan = plan_decode(self.batch, n, self.it + k)
            rows = np.full(S, self.scratch_row, np.int64)
            pos32 = np.full(S, _lib.POS_PAD_K, np.int64)
            seq32 = np.full(S, _lib.SEQ_PAD_K, np.int64)
            for j, (sid, _b) in enumerate(plan.assignments[self.rank]):
                seg = sim[sid]
                if seg[1] >= seg[2]:
                    raise RuntimeError("GraphedDecode: reservation too small for max_steps")
                rows[j] = seg[0] + seg[1]
                seg[1] += 1
                pos32[j], seq32[j] = pos[sid], sid
            starts = np.zeros(n * S, np.int64)
            lens = np.zeros(n * S, np.int64)
            for src in range(n):
                for j, (sid, _b) in enumerate(plan.assignments[src]):
                    starts[src * S + j], lens[src * S + j] = sim[sid][0], sim[sid][1]
            for sid in self.batch:
                pos[sid] += 1
            table[k] = np.concatenate([rows, starts, lens, pos32, seq32])
        self._table = torch.from_numpy(table).to(self.cache.device)
        self._table_first_it = self.it
        self._counter = torch.zeros(1, dtype=torch.int64, device=self.cache.device)

    # ------------------------------------------------------------------ launches
    def _launches(self):
        c, S = self.cache, self.slots
        if self._table is not None:
            _lib.check(_lib.load().rcp_step_select(
                _lib.ptr(self.meta), _lib.ptr(self._table), self.meta.numel(), _lib.ptr(self._counter),
                self._table.shape[0], _lib.stream_handle()))
        R = self.n * S
        ks, vs = c.decode_kwargs().get("scales", (None, None))
        # the owners' appends: K/V rows (copied or e4m3-quantised), positions
        # and sequence ids of the step metadata, in one launch
        _lib.count("rcp_decode_append")
        _lib.check(_lib.load().rcp_decode_append(
            _lib.ptr(self.meta), S, S + 2 * R, S + 2 * R + S, _lib.ptr(self.k_in), _lib.ptr(self.v_in),
            c.k.data_ptr(), c.v.data_ptr(), c.k.stride(0), self.cfg.n_kv_heads, self.cfg.head_dim,
            _lib.ptr(c.pos), _lib.ptr(c.seq), _lib.ptr(ks), _lib.ptr(vs), _lib.stream_handle()))
        starts, lens = self.meta[S:S + R], self.meta[S + R:S + 2 * R]
        if self.n == 1:
            _cuda_decode(self.q_in, c.k, c.v, starts, lens, self.max_len, self.cfg, self.out, self.lse, self.ws,
                         **c.decode_kwargs())
            return
        if self.peer is not None:
            self._launches_p2p(starts, lens)
            return
        d = self.comm.dist
        d.all_gather_into_tensor(self.q_all, self.q_in, group=self.comm.group)
        _cuda_decode(self.q_all, c.k, c.v, starts, lens, self.max_len, self.cfg, self.part_o, self.part_l,
                     self.ws, **c.decode_kwargs())
        if self.grouped_a2a:
            # both All2Alls (partial O and LSE) as ONE grouped set of NCCL
            # send/recv pairs: one NCCL launch per step instead of two
            so = [self.part_o[s * S:(s + 1) * S] for s in range(self.n)]
            sl = [self.part_l[s * S:(s + 1) * S] for s in range(self.n)]
            ro = [self.recv_o[s * S:(s + 1) * S] for s in range(self.n)]
            rl = [self.recv_l[s * S:(s + 1) * S] for s in range(self.n)]
            self.comm.wait(self.comm.all_to_all_many([(so, ro), (sl, rl)]))
        else:
            d.all_to_all_single(self.recv_o, self.part_o, group=self.comm.group)
            d.all_to_all_single(self.recv_l, self.part_l, group=self.comm.group)
        order = merge_order_of(self.rank, self.n, self.merge_mode)
        merge_rows_into([self.recv_o[s * S:(s + 1) * S] for s in order],
                        [self.recv_l[s * S:(s + 1) * S] for s in order], self.out, self.lse)

    def _launches_p2p(self, starts, lens):
        """Q put (its last block advances the epoch and signals) -> wait ->
        decode with the combine routed into the owners' receive buffers (its
        last CTA signals) -> wait -> merge: no NCCL call, five launches."""
        lib, c, P, S = _lib.load(), self.cache, self.peer, self.slots
        st, n, H, D = _lib.stream_handle(), self.n, self.cfg.n_query_heads, self.cfg.head_dim
        cnt = P.counters.data_ptr()
        stamp = self._stamp
        stamp()
        _lib.check(lib.rcp_p2p_put(_lib.ptr(P.q_dst), n, _lib.ptr(self.q_in), S * H * D * 2, _lib.ptr(P.fq_dst),
                                   _lib.ptr(P.epoch), cnt, st))
        stamp()
        _lib.check(lib.rcp_p2p_wait(P.flags("q"), n, _lib.ptr(P.epoch), _lib.ptr(P.timed_out), st))
        stamp()
        ks, vs = c.decode_kwargs().get("scales", (None, None))
        _lib.count("rcp_decode_attn_routed")
        _lib.check(lib.rcp_decode_attn_routed(
            _lib.ptr(P.q_all), _lib.ptr(c.k), _lib.ptr(c.v), c.k.stride(0), c.k.shape[0], _lib.ptr(starts),
            _lib.ptr(lens), n * S, max(self.max_len, 1), H, self.cfg.n_kv_heads, D, float(self.cfg.scale),
            _lib.ptr(ks), _lib.ptr(vs), _lib.ptr(P.o_dst), _lib.ptr(P.l_dst), n, self.rank * S * H,
            _lib.ptr(P.fo_dst), _lib.ptr(P.epoch), cnt + 4, _lib.ptr(self.ws), self.ws.numel(), st))
        stamp()
        _lib.check(lib.rcp_p2p_wait(P.flags("o"), n, _lib.ptr(P.epoch), _lib.ptr(P.timed_out), st))
        stamp()
        order = merge_order_of(self.rank, n, self.merge_mode)
        merge_rows_into([P.recv_o[s * S:(s + 1) * S] for s in order],
                        [P.recv_l[s * S:(s + 1) * S] for s in order], self.out, self.lse)
        stamp()

    def _stamp(self) -> None:
        """Debug timeline (RCP_DECODE_STAMPS=1 at construction): %globaltimer
        after each phase of the p2p step, read with ``stamps()``."""
        if self._stamps is not None:
            _lib.check(_lib.load().rcp_debug_stamp(self._stamps.data_ptr(), self._stamps.data_ptr() + 8 * 4096,
                                                   4096, _lib.stream_handle()))

    def stamps(self):
        """(n_steps, 6) int64 ns timestamps: step start, after put, after the Q
        wait, after decode + combine, after the partials wait, after merge."""
        if self._stamps is None:
            return None
        torch.cuda.synchronize()
        k = int(self._stamps[4096].item())
        t = self._stamps[:min(k, 4096)].cpu().numpy()
        return t[: (len(t) // 6) * 6].reshape(-1, 6)

    def check_transport(self) -> None:
        """Raise if a p2p wait gave up on a peer (reads a device flag: syncs)."""
        if self.peer is not None and int(self.peer.timed_out.item()):
            raise RuntimeError("GraphedDecode: a peer never signalled (p2p wait timed out)")

    def close(self) -> None:
        """Release the p2p buffers (every rank calls it together)."""
        if self.peer is not None:
            self.peer.close(self.comm)
            self.peer = None
        self.graph = None

    def _capture(self):
        self._launches()  # warm-up: lazy inits, NCCL communicators, function attributes
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launches()
        self.graph = g
        self._arena_ptr = (self.cache.k.data_ptr(), self.cache.v.data_ptr(), self.cache.pos.data_ptr(),
                           self.cache.seq.data_ptr(), self.cache.k.shape[0])
        self._segs_at_capture = self._segment_key()

    # ------------------------------------------------------------------ per step
    def _host_meta(self, mine, positions):
        """Cache bookkeeping for this rank's appends + the step's metadata arrays."""
        c, S, n = self.cache, self.slots, self.n
        rows = np.full(S, self.scratch_row, np.int64)
        pos32 = np.full(S, _lib.POS_PAD_K, np.int64)
        seq32 = np.full(S, _lib.SEQ_PAD_K, np.int64)
        for j, (sid, _b) in enumerate(mine):
            seg = c._segs[sid]
            p = int(positions[j])
            if seg.length >= seg.cap or p <= seg.max_pos:
                raise RuntimeError("GraphedDecode: sequence outgrew its reservation or positions went "
                                   "backwards; create a new GraphedDecode")
            rows[j] = seg.start + seg.length
            seg.length += 1
            seg.max_pos = p
            pos32[j], seq32[j] = p, sid
        plan = plan_decode(self.batch, n, self.it)
        starts = np.zeros(n * S, np.int64)
        lens = np.zeros(n * S, np.int64)
        for src in range(n):
            for j, (sid, _b) in enumerate(plan.assignments[src]):
                starts[src * S + j], lens[src * S + j] = c.segment(sid)
        return np.concatenate([rows, starts, lens, pos32, seq32])

    def input_buffers(self):
        """The graph's static (q [slots, Hq, D], k, v [slots, Hkv, D]) inputs: a
        model that writes this rank's new tokens straight into rows [:m] (in
        the step's ``plan_decode`` assignment order) calls ``step(None, None,
        None, positions)`` and saves the three input copies."""
        return self.q_in, self.k_in, self.v_in

    def _mine(self, it: int):
        """This rank's (seq_id, batch index) assignments at iteration ``it``
        (plan_decode's round-robin repeats with period N: cached per it % N)."""
        key = it % self.n
        got = self._mine_cache.get(key)
        if got is None:
            got = self._mine_cache[key] = plan_decode(self.batch, self.n, it).assignments[self.rank]
        return got

    def step(self, q_tok: torch.Tensor | None, k_tok: torch.Tensor | None, v_tok: torch.Tensor | None, positions):
        """One decode step.  ``q_tok`` / ``k_tok`` / ``v_tok``: this rank's new
        tokens in assignment order, or None when the caller already wrote them
        into ``input_buffers()``."""
        if self.steps_left <= 0:
            raise RuntimeError("GraphedDecode: max_steps reached; create a new GraphedDecode")
        mine = self._mine(self.it)
        m = len(mine)
        if m and q_tok is not None:
            self.q_in[:m].copy_(q_tok[:m])
            self.k_in[:m].copy_(k_tok[:m])
            self.v_in[:m].copy_(v_tok[:m])
        if self._table is not None and (
                any(int(positions[j]) != self._pos_next[sid] for j, (sid, _b) in enumerate(mine))
                or (self.graph is not None and self._segment_key() != self._segs_at_capture)):
            # not the consecutive positions / unmoved segments the table assumed:
            # back to per-step metadata uploads (re-captured without the selector)
            self._table = None
            self.graph = None
        if self._table is not None:
            meta = None
            for j, (sid, _b) in enumerate(mine):  # host bookkeeping of this step's appends
                seg = self.cache._segs[sid]
                seg.length += 1
                seg.max_pos = int(positions[j])
            for sid in self.batch:
                self._pos_next[sid] += 1
        else:
            if self.graph is not None and self._segment_key() != self._segs_at_capture:
                self._refit()  # a segment moved / grew since capture: the baked split bound is stale
                self.graph = None
            meta = self._host_meta(mine, positions)
            if max(int(x) for x in meta[_lens_slice(self)]) > self.max_len:
                raise RuntimeError("GraphedDecode: a KV segment exceeds the captured split bound")
            _lib.h2d(meta, self.cache.device, out=self.meta)  # ordered after the previous replay
        ptrs = (self.cache.k.data_ptr(), self.cache.v.data_ptr(), self.cache.pos.data_ptr(),
                self.cache.seq.data_ptr(), self.cache.k.shape[0])  # (a grown VMM arena keeps its pointer)
        if self.graph is None or ptrs != self._arena_ptr:
            # the warm-up launch in _capture executes this step (capture only
            # records), so the step's appends and outputs happen exactly once
            self._capture()
        else:
            self.graph.replay()
        self.it += 1
        self.steps_left -= 1
        return self.out[:m], self.lse[:m]
