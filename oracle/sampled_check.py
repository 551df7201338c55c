"""Large-T parity check of the CUDA path on sampled query rows — TEST INFRASTRUCTURE.

Used by tests/test_gpu_scale.py and ``bench.py --check`` (outside the timed
region) as the CHECKER only: it reads device outputs back and compares them
with ``ringcp_oracle.sampled_rows_attention`` (the reference's gqa_attention
over key blocks folded with merge_attention, attention.py:230-282 / 319-334)
on rows picked by ``ringcp_oracle.sample_rows`` (first / last token, both
sides of every 2N-chunk boundary, random rows).

Workload shape: ONE sequence of T new tokens, full prefill (positions 0..T-1,
seq id 0), sharded by plan_full_prefill over N ranks; rank r's output is in
slot order (materialize_rank_block, sharding.py:105-115, 211-240).
"""

from __future__ import annotations

import time

import numpy as np

from . import ringcp_oracle as orc


def token_to_slot(t: int, T: int, n_ranks: int) -> tuple[int, int]:
    """(rank, slot) holding token t of a single-sequence full prefill
    (rank r owns chunks r and 2N-1-r, sharding.py:79-82, 105-115)."""
    c = -(-T // (2 * n_ranks))
    ch = t // c
    if ch < n_ranks:
        return ch, t - ch * c
    return 2 * n_ranks - 1 - ch, c + (t - ch * c)


def check_rank_rows(T: int, n_ranks: int, rank: int, out, lse, q_dev, k_dev, v_dev, n_kv_heads: int,
                    scale: float, rows=None, count: int = 32, seed: int = 0, block: int = 16384,
                    k_host=None, v_host=None) -> dict:
    """Compare rank ``rank``'s device (out [S, Hq, D], lse [S, Hq]) with the
    fp64 oracle on the sampled rows this rank owns.  q_dev / k_dev / v_dev are
    the full token-order inputs (any device / dtype; read back as fp32, i.e.
    the exact bf16 values the kernels consumed).  Returns max |dO|, max |dLSE|
    and the rows checked."""
    import torch

    if rows is None:
        rows = orc.sample_rows(T, n_ranks, count, seed)
    mine = [(int(t), *token_to_slot(int(t), T, n_ranks)) for t in rows]
    mine = [(t, s) for t, r, s in mine if r == rank]
    if not mine:
        return {"rows": 0, "max_dO": 0.0, "max_dLSE": 0.0}
    toks = np.array([t for t, _ in mine], np.int64)
    slots = torch.tensor([s for _, s in mine], dtype=torch.long, device=out.device)
    got_o = out.index_select(0, slots).double().cpu().numpy()
    got_l = lse.index_select(0, slots).double().cpu().numpy()
    qr = q_dev.index_select(0, torch.from_numpy(toks).to(q_dev.device)).float().cpu().numpy()
    qb = orc.blk_from_tokens(qr, toks)
    t0 = time.perf_counter()
    # the sampled_rows_attention recipe, with key blocks read back one at a
    # time (a 1M-token K/V never has to sit in host memory as fp32)
    parts = []
    for a in range(0, min(T, int(toks.max()) + 1), block):
        b = min(T, a + block)
        kh = k_host[a:b] if k_host is not None else k_dev[a:b].float().cpu().numpy()
        vh = v_host[a:b] if v_host is not None else v_dev[a:b].float().cpu().numpy()
        pos = np.arange(a, b)
        parts.append(orc.gqa_grouped(qb, orc.blk_from_tokens(kh, pos), orc.blk_from_tokens(vh, pos),
                                     n_kv_heads, scale))
    want_o, want_l = orc.merge(parts)
    dt = time.perf_counter() - t0
    fin = np.isfinite(want_l)
    if not np.array_equal(np.isneginf(got_l), ~fin):
        d_lse = float("inf")
    else:
        d_lse = float(np.abs(got_l[fin] - want_l[fin]).max()) if fin.any() else 0.0
    return {"rows": int(toks.size), "max_dO": float(np.abs(got_o - want_o).max()), "max_dLSE": d_lse,
            "oracle_s": dt}


def check_plan_rows(plan, rank: int, out, lse, q_seqs, k_seqs, v_seqs, n_kv_heads: int, scale: float,
                    rows_per_seq: int = 8, seed: int = 0, block: int = 16384) -> dict:
    """Fused multi-sequence form of ``check_rank_rows``: sequence i of the plan
    (new tokens only, full prefill) has token-ordered inputs q_seqs[i] /
    k_seqs[i] / v_seqs[i]; rank ``rank``'s outputs are in the plan's slot order
    (sequences concatenated, 2·chunk_len slots each).  Sampled rows of every
    sequence that this rank owns are compared with the fp64 oracle over that
    sequence's keys only (attention never crosses sequences)."""
    import torch

    worst_o, worst_l, rows, off = 0.0, 0.0, 0, 0
    for i, sh in enumerate(plan.sequences):
        T = sh.spec.new_len
        loc = plan.rank_local_indices(i, rank)
        cand = orc.sample_rows(T, plan.n_ranks, rows_per_seq, seed + i)
        slot_of = {int(t): s for s, t in enumerate(loc) if t >= 0}
        mine = [(int(t), off + slot_of[int(t)]) for t in cand if int(t) in slot_of]
        off += loc.size
        if not mine:
            continue
        toks = np.array([t for t, _ in mine], np.int64)
        slots = torch.tensor([s for _, s in mine], dtype=torch.long, device=out.device)
        got_o = out.index_select(0, slots).double().cpu().numpy()
        got_l = lse.index_select(0, slots).double().cpu().numpy()
        qd = q_seqs[i]
        qr = qd.index_select(0, torch.from_numpy(toks).to(qd.device)).float().cpu().numpy()
        qb = orc.blk_from_tokens(qr, toks)
        parts = []
        for a in range(0, min(T, int(toks.max()) + 1), block):
            b = min(T, a + block)
            pos = np.arange(a, b)
            parts.append(orc.gqa_grouped(qb, orc.blk_from_tokens(k_seqs[i][a:b].float().cpu().numpy(), pos),
                                         orc.blk_from_tokens(v_seqs[i][a:b].float().cpu().numpy(), pos),
                                         n_kv_heads, scale))
        want_o, want_l = orc.merge(parts)
        fin = np.isfinite(want_l)
        if not np.array_equal(np.isneginf(got_l), ~fin):
            worst_l = float("inf")
        elif fin.any():
            worst_l = max(worst_l, float(np.abs(got_l[fin] - want_l[fin]).max()))
        worst_o = max(worst_o, float(np.abs(got_o - want_o).max()))
        rows += len(mine)
    return {"rows": rows, "max_dO": worst_o, "max_dLSE": worst_l}
