"""Multi-turn driver: full prefill, decode and partial prefill on one rank.

SPMD form of the SPEC's ``run_turns`` (paper §3.2's
three-stage characterisation): a conversation is a list of turns over
persistent sequences whose K/V stay sharded in each rank's ``RankKvCache``.

* a prefill turn appends new tokens to one or more sequences.  It is planned
  with ``plan_full_prefill`` when every sequence is new and
  ``plan_partial_prefill`` otherwise (the cached tokens stay where earlier
  turns put them), and run with ring pass-KV (Alg. 2) or ring pass-Q (Alg. 3):
  fixed by ``strategy``, or per turn by Alg. 1 (``perf_model.choose_strategy``)
  when ``strategy="adaptive"``;
* a decode turn adds one token to each sequence of a batch (Alg. 4,
  ``plan_decode`` ownership; the iteration counter advances per decode turn).

The runner keeps the per-rank cached-token layout of every sequence (the
``cached_layout`` argument of ``plan_partial_prefill``) and its next position,
so every rank plans identically without communication.  Each turn returns a
``TurnRecord`` with the strategy chosen and this rank's outputs; the
transcript of a whole scenario equals the single-rank replay of the
conversation (tests/test_turns_gloo.py, tests/test_gpu_turns.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import perf_model as pm
from .attention import GqaConfig
from .kv_cache import RankKvCache
from .ring import RingAttention, StepTrace
from .sharding import (SequenceSpec, materialize_rank_block, plan_decode, plan_full_prefill,
                       plan_partial_prefill)

__all__ = ["PrefillTurn", "DecodeTurn", "TurnRecord", "TurnRunner", "run_turns"]

STRATEGIES = ("pass_kv", "pass_q", "adaptive")


@dataclass(frozen=True)
class PrefillTurn:
    """New tokens for some sequences: ``q[i]`` [T_i, Hq, D], ``k[i]``/``v[i]``
    [T_i, Hkv, D] are the GLOBAL new tokens of ``seq_ids[i]`` (every rank passes
    the same tensors; each keeps its own load-balanced chunks)."""

    seq_ids: tuple
    q: tuple
    k: tuple
    v: tuple


@dataclass(frozen=True)
class DecodeTurn:
    """One new token per sequence of ``batch``: ``q`` [B, Hq, D], ``k``/``v``
    [B, Hkv, D] in batch order (global, identical on every rank)."""

    batch: tuple
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor


@dataclass
class TurnRecord:
    index: int
    kind: str                 # "full_prefill" | "partial_prefill" | "decode"
    strategy: str             # "pass_kv" | "pass_q" | "decode"
    new_tokens: int
    cached_tokens: int
    # prefill: this rank's query slots (PartialAttention over its materialised block);
    # decode: (out [slots, Hq, D], lse [slots, Hq]) for plan.assignments[rank]
    output: object = None
    assignments: tuple = ()   # decode: ((seq_id, batch_index), ...) of this rank
    trace: StepTrace = field(default_factory=StepTrace)


class TurnRunner:
    """Per-rank conversation state + turn execution over a ``RingAttention``."""

    def __init__(self, ring: RingAttention, cache: RankKvCache, cfg: GqaConfig, strategy: str = "adaptive",
                 cost_model: pm.CostModel | None = None, refined: bool = False, gather_decode: bool = False,
                 calibrate: bool = False):
        """``calibrate=True``: the adaptive rule's constants are measured on this
        box by ``perf_model.calibrate_b200`` (collective: every rank builds its
        runner together) instead of the static B200 profile."""
        if strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {strategy!r}")
        self.ring, self.cache, self.cfg = ring, cache, cfg
        self.n, self.rank = ring.comm.world, ring.comm.rank
        self.strategy, self.refined, self.gather_decode = strategy, refined, gather_decode
        model = dict(n_query_heads=cfg.n_query_heads, n_kv_heads=cfg.n_kv_heads, head_dim=cfg.head_dim)
        self.calibration = None
        if cost_model is None and calibrate:
            cost_model, self.calibration = pm.calibrate_b200(ring.comm, model, n_ranks=self.n, device=cache.device)
        self.cost_model = cost_model or pm.b200_profile(model, n_ranks=self.n)
        if self.cost_model.n_ranks != self.n:
            self.cost_model = pm.with_ranks(self.cost_model, self.n)
        self.layout: dict[int, list[int]] = {}   # seq id -> cached tokens per rank
        self.next_pos: dict[int, int] = {}       # seq id -> total cached length
        self.decode_iter = 0
        self.records: list[TurnRecord] = []

    # ------------------------------------------------------------------ prefill
    def choose(self, new_tokens: int, cached_tokens: int) -> str:
        if self.strategy != "adaptive":
            return self.strategy
        return pm.choose_strategy(pm.PrefillShape(new_tokens, cached_tokens), self.cost_model,
                                  refined=self.refined)

    def prefill(self, turn: PrefillTurn) -> TurnRecord:
        ids = tuple(int(s) for s in turn.seq_ids)
        if not ids or not (len(ids) == len(turn.q) == len(turn.k) == len(turn.v)):
            raise ValueError("prefill turn needs one (q, k, v) per sequence id")
        if len(set(ids)) != len(ids):
            raise ValueError("duplicate seq_id in prefill turn")
        seqs = [SequenceSpec(s, self.next_pos.get(s, 0), int(turn.q[i].shape[0])) for i, s in enumerate(ids)]
        full = all(s.cached_len == 0 for s in seqs)
        if full:
            plan = plan_full_prefill(seqs, self.n)
        else:
            plan = plan_partial_prefill(seqs, self.n, [self.layout.get(s.seq_id, [0] * self.n) for s in seqs])
        T = sum(s.new_len for s in seqs)
        P = sum(s.cached_len for s in seqs)
        strategy = self.choose(T, P)
        dev = self.cache.device
        qb = materialize_rank_block(plan, self.rank, list(turn.q), dev)
        kb = materialize_rank_block(plan, self.rank, list(turn.k), dev)
        vb = materialize_rank_block(plan, self.rank, list(turn.v), dev)
        rec = TurnRecord(len(self.records), "full_prefill" if full else "partial_prefill", strategy, T, P)
        self.ring.trace = rec.trace
        try:
            if strategy == "pass_kv":
                rec.output = self.ring.pass_kv_prefill(plan, self.cache, qb, kb, vb, self.cfg)
            else:
                rec.output = self.ring.pass_q_prefill(plan, self.cache, qb, kb, vb, self.cfg)
        finally:
            self.ring.trace = None
        for i, s in enumerate(seqs):
            row = self.layout.setdefault(s.seq_id, [0] * self.n)
            for r in range(self.n):
                row[r] += plan.new_token_count(i, r)
            self.next_pos[s.seq_id] = s.cached_len + s.new_len
        self.records.append(rec)
        return rec

    # ------------------------------------------------------------------ decode
    def decode(self, turn: DecodeTurn) -> TurnRecord:
        batch = tuple(int(b) for b in turn.batch)
        unknown = [s for s in batch if s not in self.next_pos]
        if unknown:
            raise ValueError(f"decode turn references unknown sequence(s) {unknown}")
        if not (turn.q.shape[0] == turn.k.shape[0] == turn.v.shape[0] == len(batch)):
            raise ValueError("decode turn needs one (q, k, v) token per batch entry")
        plan = plan_decode(list(batch), self.n, self.decode_iter)
        mine = plan.assignments[self.rank]
        idx = [b for _sid, b in mine]
        dev = self.cache.device
        take = (lambda x: x[idx].to(dev)) if idx else (lambda x: x[:0].to(dev))
        positions = [self.next_pos[sid] for sid, _b in mine]
        rec = TurnRecord(len(self.records), "decode", "decode", len(batch),
                         sum(self.next_pos[s] for s in batch), assignments=tuple(mine))
        self.ring.trace = rec.trace
        try:
            rec.output = self.ring.pass_q_decode(plan, self.cache, take(turn.q), take(turn.k), take(turn.v),
                                                 positions, self.cfg, gather=self.gather_decode)
        finally:
            self.ring.trace = None
        for b, sid in enumerate(batch):
            self.layout[sid][plan.owner(b)] += 1
            self.next_pos[sid] += 1
        self.decode_iter += 1
        self.records.append(rec)
        return rec

    def run(self, scenario) -> list[TurnRecord]:
        out = []
        for turn in scenario:
            if isinstance(turn, PrefillTurn):
                out.append(self.prefill(turn))
            elif isinstance(turn, DecodeTurn):
                out.append(self.decode(turn))
            else:
                raise TypeError(f"unknown turn type {type(turn).__name__}")
        return out


def run_turns(ring: RingAttention, cache: RankKvCache, cfg: GqaConfig, scenario, strategy: str = "adaptive",
              cost_model: pm.CostModel | None = None, refined: bool = False,
              gather_decode: bool = False) -> list[TurnRecord]:
    """SPEC.md:269-277 for this rank: run ``scenario`` (PrefillTurn / DecodeTurn
    list) and return the transcript (one TurnRecord per turn)."""
    return TurnRunner(ring, cache, cfg, strategy, cost_model, refined, gather_decode).run(scenario)
