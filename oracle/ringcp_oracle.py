"""CPU oracle for the ringcp context-parallel attention path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy, the algorithms of the reference package
``ringcp`` (``/root/reference/pkg/src/ringcp``) plus the SPEC/PAPER-only ring
protocols composed from those primitives.  It exists to CHECK the CUDA path:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import it.  The product package
``paper_2411_01783_b200`` never imports it and has no CPU fallback.

Parity pinning: every function is checked against golden vectors produced by
running the real reference (``tests/golden/make_golden.py`` imports ``ringcp``
from ``/root/reference/pkg/src`` and commits ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.

Numerics follow the reference exactly: fp64 accumulation, fp64 outputs, LSE is
the natural log, rows with no admitted key give lse = -inf and a zero row
(attention.py:176-196, 230-282), and invalid key rows are removed before any
arithmetic (attention.py:253-255) so padding is bitwise invisible.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NEG_INF = -np.inf


# --------------------------------------------------------------------------- blocks
@dataclass
class Blk:
    """Token block: data [T, H, D], int64 positions, bool valid, int64 seq ids.

    Mirrors ringcp.attention.EmbeddingBlock (attention.py:69-173) without the
    immutability machinery.
    """

    data: np.ndarray
    pos: np.ndarray
    valid: np.ndarray
    seq: np.ndarray

    @property
    def n(self) -> int:
        return int(self.data.shape[0])


def blk_from_tokens(data, positions, seq_id: int = 0) -> Blk:
    """attention.py:108-118 (from_tokens)."""
    data = np.asarray(data)
    n = data.shape[0]
    return Blk(data, np.asarray(positions, np.int64), np.ones(n, bool), np.full(n, seq_id, np.int64))


def blk_padding(n: int, heads: int, dim: int, dtype=np.float32) -> Blk:
    """attention.py:120-127 (padding): zero data, position -1, invalid, seq -1."""
    return Blk(np.zeros((n, heads, dim), dtype), np.full(n, -1, np.int64), np.zeros(n, bool),
               np.full(n, -1, np.int64))


def blk_concat(blocks: list[Blk]) -> Blk:
    """attention.py:129-138 (concat)."""
    if not blocks:
        raise ValueError("cannot concatenate zero blocks")
    return Blk(np.concatenate([b.data for b in blocks], 0), np.concatenate([b.pos for b in blocks]),
               np.concatenate([b.valid for b in blocks]), np.concatenate([b.seq for b in blocks]))


def blk_pad_to(b: Blk, n: int) -> Blk:
    """attention.py:165-173 (pad_to): append invalid rows up to n tokens."""
    if n < b.n:
        raise ValueError(f"cannot pad {b.n} tokens down to {n}")
    if n == b.n:
        return b
    return blk_concat([b, blk_padding(n - b.n, b.data.shape[1], b.data.shape[2], b.data.dtype)])


def blk_valid_only(b: Blk) -> Blk:
    """attention.py:155-163 (valid_only)."""
    m = b.valid
    return Blk(b.data[m], b.pos[m], b.valid[m], b.seq[m])


def check_block(b: Blk) -> None:
    """attention.py:85-106: finite valid rows, non-negative valid positions,
    strictly increasing positions within each sequence."""
    if b.n and not np.isfinite(b.data[b.valid]).all():
        raise ValueError("non-finite embedding data in valid rows")
    if np.any(b.pos[b.valid] < 0):
        raise ValueError("valid tokens must have non-negative positions")
    for sid in np.unique(b.seq[b.valid]):
        p = b.pos[b.valid & (b.seq == sid)]
        if np.any(np.diff(p) <= 0):
            raise ValueError(f"positions not strictly increasing within sequence {sid}")


# --------------------------------------------------------------------------- attention
def kv_head_of(n_q: int, n_kv: int) -> np.ndarray:
    """GqaConfig.query_to_kv_head (attention.py:64-66): h -> (h * n_kv) // n_q."""
    return (np.arange(n_q) * n_kv) // n_q


def default_scale(head_dim: int) -> float:
    """attention.py:61-62."""
    return 1.0 / math.sqrt(head_dim)


def admit_mask(qv, qpos, qseq, kv, kpos, kseq) -> np.ndarray:
    """_admissible (attention.py:199-206): [Tq, Tk] bool, diagonal included."""
    return (qv[:, None] & kv[None, :] & (qseq[:, None] == kseq[None, :])
            & (kpos[None, :] <= qpos[:, None]))


def admitted_pairs(q: Blk, k: Blk) -> int:
    """admitted_pair_count (attention.py:209-211)."""
    return int(admit_mask(q.valid, q.pos, q.seq, k.valid, k.pos, k.seq).sum())


def gqa(q: Blk, k: Blk, v: Blk, n_kv_heads: int, scale: float | None = None):
    """gqa_attention (attention.py:230-282).

    Returns (out [Tq, Hq, D] f64, lse [Tq, Hq] f64).  Keys with valid=False are
    removed before any arithmetic; rows that admit nothing are zero / -inf.
    """
    tq, hq, d = q.data.shape
    if scale is None:
        scale = default_scale(d)
    out = np.zeros((tq, hq, d), np.float64)
    lse = np.full((tq, hq), NEG_INF, np.float64)
    keep = k.valid
    k64 = k.data[keep].astype(np.float64)
    v64 = v.data[keep].astype(np.float64)
    if tq == 0 or k64.shape[0] == 0:
        return out, lse
    g = kv_head_of(hq, n_kv_heads)
    kh, vh = k64[:, g, :], v64[:, g, :]
    s = np.einsum("ihd,jhd->hij", q.data.astype(np.float64), kh, optimize=True) * scale
    adm = admit_mask(q.valid, q.pos, q.seq, np.ones(k64.shape[0], bool), k.pos[keep], k.seq[keep])
    s = np.where(adm[None], s, NEG_INF)
    mx = s.max(axis=2)
    has = np.isfinite(mx)
    base = np.where(has, mx, 0.0)
    w = np.where(adm[None], np.exp(s - base[:, :, None]), 0.0)
    den = w.sum(axis=2)
    num = np.einsum("hij,jhd->ihd", w, vh, optimize=True)
    num /= np.where(has, den, 1.0).T[:, :, None]
    out = np.where(has.T[:, :, None], num, 0.0)
    lse = np.where(has, base + np.log(np.where(has, den, 1.0)), NEG_INF).T
    return out, lse


def merge_pair(oa, la, ob, lb):
    """_merge_pair (attention.py:299-316): stable LSE merge of two partials."""
    m = np.maximum(la, lb)
    has = ~np.isneginf(m)
    base = np.where(has, m, 0.0)
    tot = np.exp(la - base) + np.exp(lb - base)
    lse = np.where(has, base + np.log(np.where(has, tot, 1.0)), NEG_INF)
    ref = np.where(has, lse, 0.0)
    wa = np.where(np.isneginf(la), 0.0, np.exp(la - ref))[:, :, None]
    wb = np.where(np.isneginf(lb), 0.0, np.exp(lb - ref))[:, :, None]
    return oa * wa + ob * wb, lse


def merge(parts):
    """merge_attention (attention.py:319-334): left fold in list order."""
    if not parts:
        raise ValueError("cannot merge an empty list of partials")
    o, l = parts[0]
    for ob, lb in parts[1:]:
        if ob.shape != o.shape:
            raise ValueError("partials are not query-shaped alike")
        o, l = merge_pair(o, l, ob, lb)
    return o, l


def naive_gqa_loops(q, k, v, qpos, kpos, n_kv_heads, scale, qseq=None, kseq=None):
    """Independent nested-loop oracle, restating pkg/tests/reference.py:12-55."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    tq, hq, d = q.shape
    tk = k.shape[0]
    qseq = [0] * tq if qseq is None else qseq
    kseq = [0] * tk if kseq is None else kseq
    out = np.zeros((tq, hq, d))
    lse = np.full((tq, hq), NEG_INF)
    for i in range(tq):
        keys = [j for j in range(tk) if kseq[j] == qseq[i] and kpos[j] <= qpos[i]]
        for h in range(hq):
            g = (h * n_kv_heads) // hq
            sc = [scale * float(np.dot(q[i, h], k[j, g])) for j in keys]
            if not sc:
                continue
            m = max(sc)
            e = [math.exp(x - m) for x in sc]
            t = sum(e)
            lse[i, h] = m + math.log(t)
            for w, j in zip(e, keys):
                out[i, h] += (w / t) * v[j, g]
    return out, lse


# --------------------------------------------------------------------------- sharding
def chunk_table(new_len: int, n_ranks: int):
    """_chunk_sequence (sharding.py:144-151): 2N chunks of ceil(T/2N); bounds clip at T."""
    c = -(-new_len // (2 * n_ranks))
    bounds = [(min(m * c, new_len), min((m + 1) * c, new_len)) for m in range(2 * n_ranks)]
    return c, bounds


def rank_chunks(rank: int, n_ranks: int):
    """ShardPlan.rank_chunk_indices (sharding.py:79-82)."""
    return rank, 2 * n_ranks - 1 - rank


def local_indices(new_len: int, n_ranks: int, rank: int) -> np.ndarray:
    """ShardPlan.rank_local_indices (sharding.py:105-115): [C_lo | C_hi] slots, -1 = pad."""
    c, bounds = chunk_table(new_len, n_ranks)
    out = np.full(2 * c, -1, np.int64)
    for slot_base, ch in zip((0, c), rank_chunks(rank, n_ranks)):
        a, b = bounds[ch]
        out[slot_base:slot_base + (b - a)] = np.arange(a, b)
    return out


def new_count(new_len: int, n_ranks: int, rank: int) -> int:
    """ShardPlan.new_token_count (sharding.py:84-87)."""
    _, bounds = chunk_table(new_len, n_ranks)
    return sum(bounds[ch][1] - bounds[ch][0] for ch in rank_chunks(rank, n_ranks))


def padded_len(new_len: int, cached_row, n_ranks: int) -> int:
    """ShardPlan.padded_len (sharding.py:95-100): max_j (P_j + T_j)."""
    return max(cached_row[j] + new_count(new_len, n_ranks, j) for j in range(n_ranks))


@dataclass
class Seq:
    seq_id: int
    cached_len: int
    new_len: int


def validate_prefill(seqs, n_ranks, cached_layout=None):
    """sharding.py:154-165 and 192-206."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    if not seqs:
        raise ValueError("cannot plan an empty sequence list")
    if len({s.seq_id for s in seqs}) != len(seqs):
        raise ValueError("duplicate seq_id in batch")
    for s in seqs:
        if s.new_len < 1:
            raise ValueError(f"sequence {s.seq_id} has no new tokens; decode turns use plan_decode")
    if cached_layout is None:
        for s in seqs:
            if s.cached_len != 0:
                raise ValueError(f"sequence {s.seq_id} has cached tokens; use plan_partial_prefill")
        return [[0] * n_ranks for _ in seqs]
    if len(cached_layout) != len(seqs):
        raise ValueError("cached_layout must have one row per sequence")
    for s, row in zip(seqs, cached_layout):
        if len(row) != n_ranks:
            raise ValueError("cached_layout rows must have one entry per rank")
        if any(c < 0 for c in row):
            raise ValueError("cached counts must be non-negative")
        if sum(row) != s.cached_len:
            raise ValueError(f"cached_layout for sequence {s.seq_id} sums to {sum(row)}, "
                             f"expected cached_len={s.cached_len}")
    return [list(map(int, r)) for r in cached_layout]


def materialize(seqs, n_ranks: int, rank: int, per_seq_data) -> Blk:
    """materialize_rank_block (sharding.py:211-240)."""
    pieces = []
    for s, arr in zip(seqs, per_seq_data):
        arr = np.asarray(arr)
        loc = local_indices(s.new_len, n_ranks, rank)
        ok = loc >= 0
        data = np.zeros((loc.size,) + arr.shape[1:], arr.dtype)
        data[ok] = arr[loc[ok]]
        pieces.append(Blk(data, np.where(ok, s.cached_len + loc, -1), ok,
                          np.where(ok, s.seq_id, -1)))
    return blk_concat(pieces)


def decode_owner(batch_index: int, iteration: int, n_ranks: int) -> int:
    """DecodePlan.owner (sharding.py:262-263)."""
    return (batch_index + iteration) % n_ranks


def decode_assignments(batch, n_ranks: int, iteration: int):
    """plan_decode (sharding.py:266-284): per-rank [(seq_id, batch_index)] ascending."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    if not batch:
        raise ValueError("decode batch must be non-empty")
    if iteration < 0:
        raise ValueError("iteration must be non-negative")
    if len(set(batch)) != len(batch):
        raise ValueError("duplicate seq_id in decode batch")
    per = [[] for _ in range(n_ranks)]
    for b, sid in enumerate(batch):
        per[decode_owner(b, iteration, n_ranks)].append((sid, b))
    return per


# --------------------------------------------------------------------------- kv cache (SPEC)
@dataclass
class Cache:
    """RankKvCache: valid-only, position-ordered per sequence."""

    n_kv_heads: int
    head_dim: int
    store: dict = field(default_factory=dict)

    def append(self, seq_id: int, k: Blk, v: Blk) -> int:
        k, v = blk_valid_only(k), blk_valid_only(v)
        if k.data.shape[1:] != (self.n_kv_heads, self.head_dim):
            raise ValueError("kv head geometry mismatch with cache")
        if seq_id in self.store:
            ok, ov = self.store[seq_id]
            k, v = blk_concat([ok, k]), blk_concat([ov, v])
        order = np.argsort(k.pos, kind="stable")
        k = Blk(k.data[order], k.pos[order], k.valid[order], k.seq[order])
        v = Blk(v.data[order], v.pos[order], v.valid[order], v.seq[order])
        self.store[seq_id] = (k, v)
        return k.n

    def cached_len(self, seq_id: int) -> int:
        return self.store[seq_id][0].n if seq_id in self.store else 0

    def snapshot_padded(self, seq_id: int, max_len: int):
        if seq_id not in self.store:
            e = blk_padding(0, self.n_kv_heads, self.head_dim)
            return blk_pad_to(e, max_len), blk_pad_to(e, max_len)
        k, v = self.store[seq_id]
        if max_len < k.n:
            raise ValueError("max_len below cached_len")
        return blk_pad_to(k, max_len), blk_pad_to(v, max_len)


# --------------------------------------------------------------------------- ring protocols (SPEC)
def kv_messages(seqs, layout, n_ranks, caches):
    """Per-rank KV message per Alg. 2: for
    each sequence i, [cached | new] position-sorted, padded to L^i."""
    msgs = []
    for r in range(n_ranks):
        ks, vs = [], []
        for i, s in enumerate(seqs):
            L = padded_len(s.new_len, layout[i], n_ranks)
            k, v = caches[r].snapshot_padded(s.seq_id, L)
            ks.append(k)
            vs.append(v)
        msgs.append((blk_concat(ks), blk_concat(vs)))
    return msgs


def ring_prefill(seqs, layout, n_ranks, caches, q_new, k_new, v_new, n_kv_heads, scale=None,
                 protocol="pass_kv"):
    """Composed pass-KV / pass-Q prefill over simulated ranks.

    q_new/k_new/v_new: per-sequence dense arrays of the NEW tokens.  New K/V are
    appended to the per-rank caches before the ring.  Returns the
    per-rank merged (out, lse) with merge order = ascending source rank
    (SPEC.md:289).  pass-Q computes the same partials and merges in the same
    order, so it is bit-identical.
    """
    qb = [materialize(seqs, n_ranks, r, q_new) for r in range(n_ranks)]
    for r in range(n_ranks):
        kb = materialize(seqs, n_ranks, r, k_new)
        vb = materialize(seqs, n_ranks, r, v_new)
        for s in seqs:
            sel = kb.seq == s.seq_id
            caches[r].append(s.seq_id, Blk(kb.data[sel], kb.pos[sel], kb.valid[sel], kb.seq[sel]),
                             Blk(vb.data[sel], vb.pos[sel], vb.valid[sel], vb.seq[sel]))
    msgs = kv_messages(seqs, layout, n_ranks, caches)
    outs = []
    for r in range(n_ranks):
        if protocol == "pass_kv":
            parts = [gqa(qb[r], msgs[s][0], msgs[s][1], n_kv_heads, scale) for s in range(n_ranks)]
        else:  # pass_q: rank s computes O_r^s with resident KV_s; All2All returns them to r
            parts = [gqa(qb[r], msgs[s][0], msgs[s][1], n_kv_heads, scale) for s in range(n_ranks)]
        outs.append(merge(parts))
    return qb, outs


def ring_decode(batch, n_ranks, iteration, caches, q_tok, k_tok, v_tok, positions, n_kv_heads,
                scale=None):
    """Composed ring pass-Q decode (Alg. 4).

    q_tok/k_tok/v_tok: [B, H, D] one new token per sequence; positions[b] its
    global position.  The plan_decode owner appends the token's K/V first (the
    query attends to itself), then each sequence's output is the merge over
    ranks (ascending) of attention against that rank's cached shard.
    """
    for b, sid in enumerate(batch):
        o = decode_owner(b, iteration, n_ranks)
        one = lambda x: blk_from_tokens(x[b:b + 1], [positions[b]], sid)
        caches[o].append(sid, one(k_tok), one(v_tok))
    outs = []
    for b, sid in enumerate(batch):
        qb = blk_from_tokens(q_tok[b:b + 1], [positions[b]], sid)
        parts = []
        for r in range(n_ranks):
            L = caches[r].cached_len(sid)
            k, v = caches[r].snapshot_padded(sid, L)
            parts.append(gqa(qb, k, v, n_kv_heads, scale))
        outs.append(merge(parts))
    return outs


# --------------------------------------------------------------------------- heuristic (SPEC/PAPER)
def size_threshold(n_q: int, n_kv: int) -> float:
    """Eq. 1: 2 N_KV / N_H."""
    return 2.0 * n_kv / n_q


def pass_kv_overlap_min_T(n_ranks, peak_flops, n_q, n_kv, elem_bytes, bw) -> float:
    """Eq. 2: N C N_KV e / (2 N_H BW)."""
    return n_ranks * peak_flops * n_kv * elem_bytes / (2.0 * n_q * bw)


def pass_q_overlap_min_ctx(n_ranks, peak_flops, elem_bytes, bw) -> float:
    """Eq. 3: N e C / (4 BW)."""
    return n_ranks * elem_bytes * peak_flops / (4.0 * bw)


def choose_strategy(new_len, cached_len, n_ranks, n_q, n_kv, peak_flops, bw, elem_bytes=2) -> str:
    """Alg. 1: pass-KV iff T >= Eq.2 or
    miss >= Eq.1; ties favour pass-KV."""
    miss = new_len / (new_len + cached_len)
    if new_len >= pass_kv_overlap_min_T(n_ranks, peak_flops, n_q, n_kv, elem_bytes, bw):
        return "pass_kv"
    if miss >= size_threshold(n_q, n_kv):
        return "pass_kv"
    return "pass_q"


def attention_flops(new_len, cached_len, model_dim) -> float:
    """Table 2: 4 T D (T + P)."""
    return 4.0 * new_len * model_dim * (new_len + cached_len)


def comm_bytes(new_len, cached_len, model_dim, n_q, n_kv, elem_bytes, kind) -> float:
    """Table 2."""
    if kind == "Q":
        return float(new_len * model_dim * elem_bytes)
    return 2.0 * (new_len + cached_len) * model_dim * (n_kv / n_q) * elem_bytes


# --------------------------------------------------------------------------- large-T (sampled rows)
def gqa_grouped(q: Blk, k: Blk, v: Blk, n_kv_heads: int, scale: float | None = None):
    """gqa_attention (attention.py:230-282) evaluated per KV-head group with
    fp64 matrix products instead of the [H, Tq, Tk] einsum, so a few query
    rows against 10^5-10^6 keys run on BLAS.  Same semantics as ``gqa``:
    padding keys dropped first (attention.py:253-255), mask = _admissible
    (attention.py:199-206), row max / exp / sum / PV in fp64, natural-log LSE,
    zero / -inf rows without keys.  Agrees with ``gqa`` to ~1e-15 (summation
    order differs); pinned by tests/test_oracle_sampled.py."""
    tq, hq, d = q.data.shape
    if scale is None:
        scale = default_scale(d)
    out = np.zeros((tq, hq, d), np.float64)
    lse = np.full((tq, hq), NEG_INF, np.float64)
    keep = k.valid
    if tq == 0 or not keep.any():
        return out, lse
    kpos, kseq = k.pos[keep], k.seq[keep]
    adm = admit_mask(q.valid, q.pos, q.seq, np.ones(kpos.size, bool), kpos, kseq)  # [Tq, Tk]
    if not adm.any():
        return out, lse
    heads_of = kv_head_of(hq, n_kv_heads)
    for g in range(n_kv_heads):
        hs = np.flatnonzero(heads_of == g)
        kg = k.data[keep][:, g, :].astype(np.float64)            # [Tk, D]
        vg = v.data[keep][:, g, :].astype(np.float64)
        qg = q.data[:, hs, :].astype(np.float64).reshape(tq * hs.size, d)
        s = (qg @ kg.T).reshape(tq, hs.size, -1) * scale          # [Tq, G, Tk]
        s = np.where(adm[:, None, :], s, NEG_INF)
        mx = s.max(axis=2)
        has = np.isfinite(mx)
        base = np.where(has, mx, 0.0)
        w = np.where(adm[:, None, :], np.exp(s - base[:, :, None]), 0.0)
        den = w.sum(axis=2)
        num = (w.reshape(tq * hs.size, -1) @ vg).reshape(tq, hs.size, d)
        num /= np.where(has, den, 1.0)[:, :, None]
        out[:, hs, :] = np.where(has[:, :, None], num, 0.0)
        lse[:, hs] = np.where(has, base + np.log(np.where(has, den, 1.0)), NEG_INF)
    return out, lse


def sampled_rows_attention(q_rows: Blk, k: Blk, v: Blk, n_kv_heads: int, scale: float | None = None,
                           block: int = 16384):
    """Exact fp64 attention of a few query rows against a long key sequence:
    the reference's recipe for large T — gqa_attention on
    consecutive key blocks (attention.py:230-282), folded left in ascending
    block order with merge_attention (attention.py:319-334).  Blocks whose
    smallest valid position exceeds every query position admit nothing and
    are skipped (merging an all -inf partial is the exact identity of
    _merge_pair, attention.py:299-316).  Returns (out [R, Hq, D], lse [R, Hq])."""
    parts = []
    qmax = int(q_rows.pos[q_rows.valid].max()) if q_rows.valid.any() else -1
    for a in range(0, k.n, block):
        b = min(k.n, a + block)
        kv = k.valid[a:b]
        if not kv.any() or int(k.pos[a:b][kv].min()) > qmax:
            continue
        kb = Blk(k.data[a:b], k.pos[a:b], k.valid[a:b], k.seq[a:b])
        vb = Blk(v.data[a:b], v.pos[a:b], v.valid[a:b], v.seq[a:b])
        parts.append(gqa_grouped(q_rows, kb, vb, n_kv_heads, scale))
    if not parts:
        tq, hq, d = q_rows.data.shape
        return np.zeros((tq, hq, d)), np.full((tq, hq), NEG_INF)
    return merge(parts)


def sample_rows(n_tokens: int, n_ranks: int, count: int, seed: int = 0) -> np.ndarray:
    """Query rows worth checking at scale: first / last token, both sides of
    every 2N-chunk boundary (sharding.py:144-151), then random rows up to
    ``count`` (the boundaries are always included)."""
    c = -(-n_tokens // (2 * n_ranks))
    rows = {0, n_tokens - 1}
    for m in range(1, 2 * n_ranks):
        b = m * c
        if 0 < b < n_tokens:
            rows.update((b - 1, b))
    rng = np.random.default_rng(seed)
    while len(rows) < count and len(rows) < n_tokens:
        rows.add(int(rng.integers(0, n_tokens)))
    return np.array(sorted(rows), np.int64)


# --------------------------------------------------------------------------- FP8 (e4m3) KV rows
# Not in the reference (its numerics are fp64 / bf16); the FP8 KV-cache mode is
# SURVEY §8f rank 4 (FP8 on the attention path).  Restated from
# the OCP 8-bit floating point spec (E4M3 "fn": bias 7, no infinities,
# S.1111.111 = NaN, max 448, subnormals m * 2^-9) and the PTX conversion
# semantics the kernels use (cvt.rn.satfinite.e4m3x2.f32: round to nearest
# even, |x| > 448 -> 448, NaN -> NaN).  Pinned against torch.float8_e4m3fn in
# tests/test_oracle_fp8.py.
E4M3_MAX = 448.0


def e4m3_encode(x) -> np.ndarray:
    """float32 values -> e4m3 bytes (RNE, satfinite)."""
    v = np.asarray(x, np.float32).astype(np.float64)
    sign = np.signbit(v).astype(np.uint8) << 7
    a = np.abs(v)
    nan = np.isnan(a)
    a = np.where(nan, 0.0, a)
    _, ex = np.frexp(np.where(a > 0, a, 1.0))           # a = m * 2^ex, m in [0.5, 1)
    e = np.maximum(ex - 1, -6)                          # binade (subnormals share 2^-6's quantum)
    q = np.ldexp(1.0, e - 3)                            # spacing of 3 mantissa bits
    r = np.minimum(np.rint(a / q) * q, E4M3_MAX)        # RNE, then saturate
    _, rex = np.frexp(np.where(r > 0, r, 1.0))
    E = rex - 1
    normal = r >= 2.0 ** -6
    man_n = np.rint((r / np.ldexp(1.0, E) - 1.0) * 8).astype(np.int64)
    bits_n = ((E + 7) << 3) | man_n
    bits_s = np.rint(r / 2.0 ** -9).astype(np.int64)
    bits = np.where(normal, bits_n, bits_s).astype(np.uint8)
    return np.where(nan, np.uint8(0x7F), bits | sign).astype(np.uint8)


def e4m3_decode(b) -> np.ndarray:
    """e4m3 bytes -> float64 values (NaN for S.1111.111)."""
    b = np.asarray(b, np.uint8).astype(np.int64)
    s = np.where(b & 0x80, -1.0, 1.0)
    E = (b >> 3) & 15
    m = b & 7
    val = np.where(E == 0, m * 2.0 ** -9, (1.0 + m / 8.0) * np.ldexp(1.0, E - 7))
    return np.where((b & 0x7F) == 0x7F, np.nan, s * val)


def pow2_ceil_f32(v) -> np.ndarray:
    """Smallest power of two >= v for positive normal float32 v (bit-exact:
    round the exponent up unless the mantissa is zero)."""
    u = np.asarray(v, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFFFF) & 0xFF800000).astype(np.uint32).view(np.float32)


def e4m3_scale(rows, n_kv_heads: int) -> np.ndarray:
    """Per-KV-head calibration scale (rcp_kv_calibrate_e4m3): max(absmax,
    2^-24) / 448 in float32, rounded UP to a power of two.  A power-of-two
    scale keeps the head's absmax within e4m3's range and makes e4m3 * scale
    exactly representable in bf16, so the bf16 rows the prefill reads and the
    scaled e4m3 the decode kernel reads are the same values."""
    r = np.asarray(rows, np.float32).reshape(-1, n_kv_heads, np.asarray(rows).shape[-1])
    amax = np.abs(r).max(axis=(0, 2)) if r.shape[0] else np.zeros(n_kv_heads, np.float32)
    v = (np.maximum(amax, np.float32(2.0 ** -24)).astype(np.float32) / np.float32(E4M3_MAX)).astype(np.float32)
    return pow2_ceil_f32(v)


def quantize_e4m3(rows, scale) -> np.ndarray:
    """rows [n, H, D] (float32 / bf16 values) -> e4m3 bytes: RNE(x * inv[h])
    with inv = 1 / scale[h] and the product in IEEE float32
    (rcp_kv_quantize_e4m3)."""
    r = np.asarray(rows, np.float32)
    inv = (np.float32(1.0) / np.asarray(scale, np.float32)).astype(np.float32).reshape(1, -1, 1)
    return e4m3_encode((r * inv).astype(np.float32))


def dequantize_e4m3(bits, scale) -> np.ndarray:
    """e4m3 bytes [n, H, D] -> exact float64 values scale[h] * e4m3."""
    return e4m3_decode(bits) * np.asarray(scale, np.float64).reshape(1, -1, 1)


def f32_to_bf16_values(x) -> np.ndarray:
    """Round float32 to bf16 (nearest even), returned as float32 values."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def dequantize_e4m3_bf16(bits, scale) -> np.ndarray:
    """rcp_kv_dequantize_e4m3: float32(e4m3) * float32(scale) in fp32, rounded to bf16."""
    v = e4m3_decode(bits).astype(np.float32) * np.asarray(scale, np.float32).reshape(1, -1, 1)
    return f32_to_bf16_values(v.astype(np.float32))
