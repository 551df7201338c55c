"""Pin the CPU oracle to golden vectors produced by the real reference ``ringcp``
(tests/golden/make_golden.py).  CPU only."""

import math

import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from tests import _golden as G


def test_gqa_oracle_matches_reference_bitwise():
    z = G.npz("gqa.npz")
    for name in z["names"]:
        c = G.gqa_case(z, name)
        out, lse = orc.gqa(c["q"], c["k"], c["v"], c["hkv"], c["scale"])
        np.testing.assert_array_equal(out, c["out"], err_msg=name)
        np.testing.assert_array_equal(lse, c["lse"], err_msg=name)
        assert orc.admitted_pairs(c["q"], c["k"]) == c["pairs"], name


def test_loop_oracle_agrees_with_vector_oracle():
    z = G.npz("gqa.npz")
    for name in ["causal8", "single_key", "fully_masked", "cross_seq"]:
        c = G.gqa_case(z, name)
        keep = c["k"].valid
        out, lse = orc.naive_gqa_loops(c["q"].data, c["k"].data[keep], c["v"].data[keep], c["q"].pos,
                                       c["k"].pos[keep], c["hkv"], c["scale"], c["q"].seq, c["k"].seq[keep])
        assert np.abs(out - c["out"]).max() < 1e-12
        fin = np.isfinite(c["lse"])
        assert np.array_equal(np.isneginf(lse), ~fin)
        if fin.any():
            assert np.abs(lse[fin] - c["lse"][fin]).max() < 1e-12


def test_merge_oracle_matches_reference_bitwise():
    z = G.npz("merge.npz")
    for name in z["names"]:
        n = int(z[f"{name}__n"])
        parts = [(z[f"{name}__p{p}__out"], z[f"{name}__p{p}__lse"]) for p in range(n)]
        out, lse = orc.merge(parts)
        np.testing.assert_array_equal(out, z[f"{name}__out"])
        np.testing.assert_array_equal(lse, z[f"{name}__lse"])


def test_shard_plans_match_reference():
    cases = G.js("shard.json")
    z = G.npz("shard.npz")
    for ci, c in enumerate(cases):
        n = c["n_ranks"]
        seqs = [orc.Seq(s["seq_id"], s["cached_len"], s["new_len"]) for s in c["sequences"]]
        layout = [s["rank_cached_counts"] for s in c["sequences"]]
        for i, (s, sj) in enumerate(zip(seqs, c["sequences"])):
            ch, bounds = orc.chunk_table(s.new_len, n)
            assert ch == sj["chunk_len"]
            assert [list(b) for b in bounds] == sj["chunks"]
            assert orc.padded_len(s.new_len, layout[i], n) == sj["padded_len"]
            assert [orc.new_count(s.new_len, n, r) for r in range(n)] == sj["rank_new_counts"]
            for r in range(n):
                assert orc.local_indices(s.new_len, n, r).tolist() == c["local_indices"][i][r]
        assert sum(2 * orc.chunk_table(s.new_len, n)[0] for s in seqs) == c["total_query_slots"]
        if f"s{ci}__in0" in z:
            data = [z[f"s{ci}__in{i}"] for i in range(len(seqs))]
            for r in range(n):
                b = orc.materialize(seqs, n, r, data)
                np.testing.assert_array_equal(b.data, z[f"s{ci}__r{r}__data"])
                np.testing.assert_array_equal(b.pos, z[f"s{ci}__r{r}__pos"])
                np.testing.assert_array_equal(b.valid, z[f"s{ci}__r{r}__valid"])
                np.testing.assert_array_equal(b.seq, z[f"s{ci}__r{r}__seq"])


def test_decode_plans_match_reference():
    for c in G.js("decode.json"):
        got = orc.decode_assignments(c["batch"], c["n_ranks"], c["iteration"])
        assert [[list(e) for e in a] for a in got] == c["assignments"]
        assert math.ceil(len(c["batch"]) / c["n_ranks"]) == c["slots_per_rank"]


def test_ring_oracle_matches_reference_composition():
    z = G.npz("ring.npz")
    for name in z["names"]:
        meta = [int(x) for x in z[f"{name}__meta"]]
        n, hq, hkv, lens = meta[0], meta[1], meta[2], meta[3:]
        seqs = [orc.Seq(i, 0, t) for i, t in enumerate(lens)]
        qd = [z[f"{name}__q{i}"] for i in range(len(lens))]
        kd = [z[f"{name}__k{i}"] for i in range(len(lens))]
        vd = [z[f"{name}__v{i}"] for i in range(len(lens))]
        layout = [[0] * n for _ in seqs]
        for proto in ("pass_kv", "pass_q"):
            caches = [orc.Cache(hkv, 128) for _ in range(n)]
            qb, outs = orc.ring_prefill(seqs, layout, n, caches, qd, kd, vd, hkv, protocol=proto)
            for r in range(n):
                np.testing.assert_array_equal(qb[r].data, z[f"{name}__r{r}__q__data"])
                np.testing.assert_array_equal(outs[r][0], z[f"{name}__r{r}__out"])
                np.testing.assert_array_equal(outs[r][1], z[f"{name}__r{r}__lse"])


def test_ring_oracle_equals_dense_unsharded():
    """Composed ring (pass-KV / pass-Q) == one dense causal attention."""
    rng = np.random.default_rng(9)
    for n, lens in [(2, [64]), (3, [50, 31]), (4, [128, 9])]:
        seqs = [orc.Seq(10 + i, 0, t) for i, t in enumerate(lens)]
        qd = [rng.standard_normal((t, 4, 16)) for t in lens]
        kd = [rng.standard_normal((t, 2, 16)) for t in lens]
        vd = [rng.standard_normal((t, 2, 16)) for t in lens]
        caches = [orc.Cache(2, 16) for _ in range(n)]
        qb, outs = orc.ring_prefill(seqs, [[0] * n for _ in seqs], n, caches, qd, kd, vd, 2)
        for i, s in enumerate(seqs):
            full_q = orc.blk_from_tokens(qd[i], np.arange(lens[i]), s.seq_id)
            full_k = orc.blk_from_tokens(kd[i], np.arange(lens[i]), s.seq_id)
            full_v = orc.blk_from_tokens(vd[i], np.arange(lens[i]), s.seq_id)
            want_o, want_l = orc.gqa(full_q, full_k, full_v, 2)
            for r in range(n):
                sel = qb[r].valid & (qb[r].seq == s.seq_id)
                pos = qb[r].pos[sel]
                assert np.abs(outs[r][0][sel] - want_o[pos]).max() < 1e-12
                assert np.abs(outs[r][1][sel] - want_l[pos]).max() < 1e-12


def test_decode_oracle_equals_dense():
    rng = np.random.default_rng(4)
    n, batch, T = 2, [3, 5, 8], 20
    seqs = [orc.Seq(s, 0, T) for s in batch]
    qd = [rng.standard_normal((T, 4, 16)) for _ in batch]
    kd = [rng.standard_normal((T + 6, 2, 16)) for _ in batch]
    vd = [rng.standard_normal((T + 6, 2, 16)) for _ in batch]
    caches = [orc.Cache(2, 16) for _ in range(n)]
    orc.ring_prefill(seqs, [[0] * n for _ in seqs], n, caches, qd, [k[:T] for k in kd], [v[:T] for v in vd], 2)
    for it in range(6):
        qt = rng.standard_normal((len(batch), 4, 16))
        kt = np.stack([k[T + it] for k in kd])
        vt = np.stack([v[T + it] for v in vd])
        outs = orc.ring_decode(batch, n, it, caches, qt, kt, vt, [T + it] * len(batch), 2)
        for b in range(len(batch)):
            fq = orc.blk_from_tokens(qt[b:b + 1], [T + it])
            fk = orc.blk_from_tokens(kd[b][:T + it + 1], np.arange(T + it + 1))
            fv = orc.blk_from_tokens(vd[b][:T + it + 1], np.arange(T + it + 1))
            wo, wl = orc.gqa(fq, fk, fv, 2)
            assert np.abs(outs[b][0] - wo).max() < 1e-12
            assert np.abs(outs[b][1] - wl).max() < 1e-12
    # round-robin decode balance: per-sequence per-rank appended counts differ by <= 1
    counts = [[caches[r].cached_len(s) for r in range(n)] for s in batch]
    for row in counts:
        assert max(row) - min(row) <= 1 + T  # prefill split is balanced, decode adds <= 1 skew


def test_heuristic_paper_examples():
    # Eq. 1 for Llama3-405B
    assert orc.size_threshold(128, 8) == 0.125
    # Eq. 2 example: N=1, C=8e14, 1/16, e=2, BW=5e10 -> 1000
    assert orc.pass_kv_overlap_min_T(1, 8e14, 16, 1, 2, 5e10) == pytest.approx(1000)
    # Eq. 3 example: N=1, e=2, C=8e14, BW=5e10 -> 8000
    assert orc.pass_q_overlap_min_ctx(1, 8e14, 2, 5e10) == pytest.approx(8000)
    # full prefill -> pass-KV
    assert orc.choose_strategy(1000, 0, 4, 128, 8, 8e14, 5e10) == "pass_kv"
