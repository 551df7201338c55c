"""GPU: device sharding bit-exact vs the reference, ring pass-KV / pass-Q /
decode over simulated ranks vs the reference-composed oracle."""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rc():
    import paper_2411_01783_b200 as rc

    return rc


def test_materialize_bit_exact_vs_reference(rc):
    import torch

    from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block,
                                                plan_full_prefill, plan_partial_prefill)

    cases = G.js("shard.json")
    z = G.npz("shard.npz")
    for ci, c in enumerate(cases):
        if f"s{ci}__in0" not in z:
            continue
        seqs = [SequenceSpec(s["seq_id"], s["cached_len"], s["new_len"]) for s in c["sequences"]]
        n = c["n_ranks"]
        plan = (plan_full_prefill(seqs, n) if c["kind"] == "full" else
                plan_partial_prefill(seqs, n, [s["rank_cached_counts"] for s in c["sequences"]]))
        data = [z[f"s{ci}__in{i}"] for i in range(len(seqs))]
        for r in range(n):
            for src in ("host", "device"):
                arrs = data if src == "host" else [torch.from_numpy(a).cuda() for a in data]
                b = materialize_rank_block(plan, r, arrs)
                np.testing.assert_array_equal(b.data.cpu().numpy(), z[f"s{ci}__r{r}__data"])
                np.testing.assert_array_equal(b.positions.cpu().numpy(), z[f"s{ci}__r{r}__pos"])
                np.testing.assert_array_equal(b.valid.cpu().numpy(), z[f"s{ci}__r{r}__valid"])
                np.testing.assert_array_equal(b.seq_ids.cpu().numpy(), z[f"s{ci}__r{r}__seq"])


@pytest.mark.parametrize("T,n", [(4096, 2), (1000, 4), (8192, 8), (333, 3)])
def test_device_gather_kernel_bit_exact_d128(rc, T, n):
    """rcp_shard_gather at kernel geometry (16-byte rows) vs the oracle restatement."""
    import torch

    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    rng = np.random.default_rng(T)
    x = rng.standard_normal((T, 2, 128)).astype(np.float32)
    plan = plan_full_prefill([SequenceSpec(3, 0, T)], n)
    xd = torch.from_numpy(x).cuda()
    for r in range(n):
        b = materialize_rank_block(plan, r, [xd])
        want = orc.materialize([orc.Seq(3, 0, T)], n, r, [x])
        np.testing.assert_array_equal(b.data.cpu().numpy(), want.data)
        np.testing.assert_array_equal(b.positions.cpu().numpy(), want.pos)
        np.testing.assert_array_equal(b.valid.cpu().numpy(), want.valid)
        np.testing.assert_array_equal(b.seq_ids.cpu().numpy(), want.seq)
        p32, s32 = b.meta32("q")
        assert np.array_equal(p32.cpu().numpy(), np.where(want.valid, want.pos, -1))


def _ring_inputs(rc, name):
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    z = G.npz("ring.npz")
    meta = [int(x) for x in z[f"{name}__meta"]]
    n, hq, hkv, lens = meta[0], meta[1], meta[2], meta[3:]
    plan = plan_full_prefill([SequenceSpec(i, 0, t) for i, t in enumerate(lens)], n)
    cfg = rc.GqaConfig(hq, hkv, 128)
    dev = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    qd = [dev(z[f"{name}__q{i}"]) for i in range(len(lens))]
    kd = [dev(z[f"{name}__k{i}"]) for i in range(len(lens))]
    vd = [dev(z[f"{name}__v{i}"]) for i in range(len(lens))]
    qb = [materialize_rank_block(plan, r, qd) for r in range(n)]
    kb = [materialize_rank_block(plan, r, kd) for r in range(n)]
    vb = [materialize_rank_block(plan, r, vd) for r in range(n)]
    caches = lambda: [RankKvCache(hkv, 128, capacity_tokens=256) for _ in range(n)]
    return z, n, plan, cfg, qb, kb, vb, caches


@pytest.mark.parametrize("name", ["ring_n2_t256", "ring_n3_fused", "ring_n4_t512"])
def test_ring_prefill_matches_reference_composition(rc, name):
    from paper_2411_01783_b200.ring import StepTrace, ring_pass_kv_prefill, ring_pass_q_prefill

    z, n, plan, cfg, qb, kb, vb, caches = _ring_inputs(rc, name)
    tr = StepTrace()
    kv = ring_pass_kv_prefill(plan, caches(), qb, kb, vb, cfg, trace=tr)
    pq = ring_pass_q_prefill(plan, caches(), qb, kb, vb, cfg)
    for r in range(n):
        o = kv[r].output.data.cpu().numpy()
        l = kv[r].lse.cpu().numpy()
        assert np.abs(o - z[f"{name}__r{r}__out"]).max() <= G.O_TOL
        assert G.lse_err(l, z[f"{name}__r{r}__lse"]) <= G.LSE_TOL
        # protocol equivalence: pass-KV and pass-Q bit-identical
        assert np.array_equal(o, pq[r].output.data.cpu().numpy())
        assert np.array_equal(l, pq[r].lse.cpu().numpy())
    # message-count law: N-1 KV sends per rank, equal sizes within a step
    assert len(tr.records) == n * (n - 1)
    assert len({rec[3] for rec in tr.records}) == 1


@pytest.mark.parametrize("kv_dtype", ["bf16", "e4m3"])
def test_partial_prefill_and_decode_vs_oracle(rc, kv_dtype):
    """Multi-turn: full prefill -> 5 decode steps -> partial prefill, vs the
    composed oracle.  e4m3: FP8 caches with fixed per-head
    scales; the oracle sees every K/V row quantised and dequantised (the
    prefill messages and the decode kernel both read the cached e4m3 rows)."""
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_kv_prefill, ring_pass_q_decode, ring_pass_q_prefill
    from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_decode,
                                                plan_full_prefill, plan_partial_prefill)

    rng = np.random.default_rng(21)
    n, hq, hkv = 3, 8, 2
    cfg = rc.GqaConfig(hq, hkv, 128)
    bf = lambda a: _bf16(a)
    batch = [4, 9]
    T0 = [300, 170]
    if kv_dtype == "e4m3":
        sc = np.array([2.0 ** -6, 2.0 ** -5], np.float32)  # powers of two: the bf16 prefill rows are exact
        caches_g = [RankKvCache(hkv, 128, capacity_tokens=128, kv_dtype="e4m3", k_scale=sc, v_scale=sc)
                    for _ in range(n)]
        kvq = lambda a: orc.dequantize_e4m3(orc.quantize_e4m3(a, sc), sc)  # what the cache holds
    else:
        caches_g = [RankKvCache(hkv, 128, capacity_tokens=128) for _ in range(n)]
        kvq = lambda a: a
    caches_o = [orc.Cache(hkv, 128) for _ in range(n)]
    # turn 1: full prefill
    seqs = [SequenceSpec(s, 0, t) for s, t in zip(batch, T0)]
    q = [bf(rng.standard_normal((t, hq, 128))) for t in T0]
    k = [bf(rng.standard_normal((t, hkv, 128))) for t in T0]
    v = [bf(rng.standard_normal((t, hkv, 128))) for t in T0]
    plan = plan_full_prefill(seqs, n)
    dev = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    qb = [materialize_rank_block(plan, r, [dev(x) for x in q]) for r in range(n)]
    kb = [materialize_rank_block(plan, r, [dev(x) for x in k]) for r in range(n)]
    vb = [materialize_rank_block(plan, r, [dev(x) for x in v]) for r in range(n)]
    got = ring_pass_kv_prefill(plan, caches_g, qb, kb, vb, cfg)
    oseqs = [orc.Seq(s, 0, t) for s, t in zip(batch, T0)]
    _, want = orc.ring_prefill(oseqs, [[0] * n for _ in oseqs], n, caches_o, q, [kvq(x) for x in k],
                               [kvq(x) for x in v], hkv)
    for r in range(n):
        assert np.abs(got[r].output.data.cpu().numpy() - want[r][0]).max() <= G.O_TOL
        assert G.lse_err(got[r].lse.cpu().numpy(), want[r][1]) <= G.LSE_TOL
    # turn 2: decode steps
    lens = list(T0)
    for it in range(5):
        dp = plan_decode(batch, n, it)
        qt = bf(rng.standard_normal((len(batch), hq, 128)))
        kt = bf(rng.standard_normal((len(batch), hkv, 128)))
        vt = bf(rng.standard_normal((len(batch), hkv, 128)))
        pos = list(lens)
        o, l = ring_pass_q_decode(dp, caches_g, dev(qt), dev(kt), dev(vt), pos, cfg)
        wo = orc.ring_decode(batch, n, it, caches_o, qt, kvq(kt), kvq(vt), pos, hkv)
        for b in range(len(batch)):
            assert np.abs(o[b].cpu().numpy() - wo[b][0][0]).max() <= G.O_TOL
            assert G.lse_err(l[b].cpu().numpy(), wo[b][1][0]) <= G.LSE_TOL
        lens = [x + 1 for x in lens]
    # turn 3: partial prefill (new tokens continue after the cached history)
    T1 = [40, 23]
    layout = [[caches_g[r].cached_len(s) for r in range(n)] for s in batch]
    seqs = [SequenceSpec(s, P, t) for s, P, t in zip(batch, lens, T1)]
    plan = plan_partial_prefill(seqs, n, layout)
    q = [bf(rng.standard_normal((t, hq, 128))) for t in T1]
    k = [bf(rng.standard_normal((t, hkv, 128))) for t in T1]
    v = [bf(rng.standard_normal((t, hkv, 128))) for t in T1]
    qb = [materialize_rank_block(plan, r, [dev(x) for x in q]) for r in range(n)]
    kb = [materialize_rank_block(plan, r, [dev(x) for x in k]) for r in range(n)]
    vb = [materialize_rank_block(plan, r, [dev(x) for x in v]) for r in range(n)]
    caches_g2 = caches_g  # pass-Q needs its own caches: rebuild by replay is costly; compare pass-KV here
    got = ring_pass_kv_prefill(plan, caches_g2, qb, kb, vb, cfg)
    oseqs = [orc.Seq(s, P, t) for s, P, t in zip(batch, lens, T1)]
    _, want = orc.ring_prefill(oseqs, layout, n, caches_o, q, [kvq(x) for x in k], [kvq(x) for x in v], hkv)
    for r in range(n):
        assert np.abs(got[r].output.data.cpu().numpy() - want[r][0]).max() <= G.O_TOL
        assert G.lse_err(got[r].lse.cpu().numpy(), want[r][1]) <= G.LSE_TOL


def _bf16(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("hq,hkv,lens", [(128, 8, [5000, 70, 0, 1]), (32, 8, [4099, 64]),
                                         (16, 1, [20000]), (40, 1, [3000, 17]), (64, 2, [5000])])
def test_decode_kernel_vs_oracle(rc, hq, hkv, lens):
    """rcp_decode_attn directly: one query per sequence against its cache
    segment (ragged lengths, empty segment, tail blocks, several splits)."""
    import torch

    from paper_2411_01783_b200.ring import _cuda_decode

    rng = np.random.default_rng(sum(lens) + hq)
    cap = sum(lens) + 256
    k = _bf16(rng.standard_normal((cap, hkv, 128)))
    v = _bf16(rng.standard_normal((cap, hkv, 128)))
    q = _bf16(rng.standard_normal((len(lens), hq, 128)))
    starts = np.cumsum([0] + lens[:-1]) + 3
    cfg = rc.GqaConfig(hq, hkv, 128)
    dev = lambda a: torch.from_numpy(a).cuda()
    out = torch.empty((len(lens), hq, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((len(lens), hq), dtype=torch.float32, device="cuda")
    _cuda_decode(dev(q).to(torch.bfloat16), dev(k).to(torch.bfloat16), dev(v).to(torch.bfloat16),
                 dev(starts.astype(np.int64)), dev(np.array(lens, np.int64)), max(lens), cfg, out, lse)
    for b, n in enumerate(lens):
        s0 = starts[b]
        qb = orc.blk_from_tokens(q[b:b + 1], [n])
        kb = orc.blk_from_tokens(k[s0:s0 + n], np.arange(n))
        vb = orc.blk_from_tokens(v[s0:s0 + n], np.arange(n))
        wo, wl = orc.gqa(qb, kb, vb, hkv)
        assert np.abs(out[b].cpu().numpy() - wo[0]).max() <= G.O_TOL
        assert G.lse_err(lse[b].cpu().numpy(), wl[0]) <= G.LSE_TOL


@pytest.mark.parametrize("lens,n,cached", [([4096], 2, [0]), ([1000, 333], 4, [0, 0]), ([8192], 8, [0]),
                                           ([9], 4, [0]), ([700, 50, 2000], 3, [100, 0, 7])])
def test_shard_scatter_inverts_gather_bit_exact(rc, lens, n, cached):
    """Device scatter (rcp_shard_scatter) is the exact inverse of the device
    gather: the N ranks' scatters rebuild every sequence bitwise, and each
    rank's scatter writes exactly the oracle's local indices of that rank."""
    import torch

    from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_partial_prefill,
                                                scatter_rank_block, unshard)

    rng = np.random.default_rng(sum(lens) + n)
    specs = [SequenceSpec(i + 3, c, t) for i, (t, c) in enumerate(zip(lens, cached))]
    layout = [[c // n + (1 if r < c % n else 0) for r in range(n)] for c in cached]
    plan = plan_partial_prefill(specs, n, layout)
    for shape, dt in (((2, 128), np.float32), ((8, 128), np.float32), ((1, 4), np.float32), ((1, 2), np.float32)):
        xs = [rng.standard_normal((t,) + shape).astype(dt) for t in lens]
        xd = [torch.from_numpy(x).cuda() for x in xs]
        blocks = [materialize_rank_block(plan, r, xd).data for r in range(n)]
        back = unshard(plan, blocks)
        for x, b in zip(xs, back):
            np.testing.assert_array_equal(b.cpu().numpy(), x)
        # one rank alone writes exactly its own rows (others untouched)
        for r in range(n):
            outs = [torch.full((t,) + shape, -7.0, device="cuda") for t in lens]
            scatter_rank_block(plan, r, blocks[r], outs)
            for i, (x, o) in enumerate(zip(xs, outs)):
                loc = orc.local_indices(lens[i], n, r)
                loc = loc[loc >= 0]
                got = o.cpu().numpy()
                np.testing.assert_array_equal(got[loc], x[loc])
                mask = np.ones(lens[i], bool)
                mask[loc] = False
                assert np.all(got[mask] == -7.0)


def test_ring_outputs_unshard_to_token_order(rc):
    """End to end: a simulated CP3 ring's slot-ordered outputs (O fp32 rows and
    LSE rows), scattered back to token order on the device, match the oracle's
    token-ordered single-block attention."""
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_kv_prefill
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill, unshard

    T, n, hq, hkv = 1000, 3, 8, 2
    rng = np.random.default_rng(5)
    arrs = [_bf16_exact(rng.standard_normal((T, h, 128)).astype(np.float32)) for h in (hq, hkv, hkv)]
    dev = [torch.from_numpy(a).cuda().to(torch.bfloat16) for a in arrs]
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    cfg = rc.GqaConfig(hq, hkv, 128)
    blocks = [[materialize_rank_block(plan, r, [t]) for r in range(n)] for t in dev]
    outs = ring_pass_kv_prefill(plan, [RankKvCache(hkv, 128, capacity_tokens=T) for _ in range(n)], *blocks, cfg)
    o_tok = unshard(plan, [p.output.data for p in outs])[0]
    l_tok = unshard(plan, [p.lse for p in outs])[0]
    q, k, v = (orc.blk_from_tokens(a, np.arange(T)) for a in arrs)
    want_o, want_l = orc.gqa(q, k, v, hkv)
    assert np.abs(o_tok.cpu().numpy() - want_o).max() <= G.O_TOL
    assert G.lse_err(l_tok.cpu().numpy(), want_l) <= G.LSE_TOL


def _bf16_exact(x):
    from tests.golden.make_golden_inputs import bf16_exact

    return bf16_exact(x)


@pytest.mark.parametrize("name", ["ring_n3_fused", "ring_n4_t512"])
def test_ascending_merge_order_matches_merge_attention_bitwise(rc, name):
    """merge_order="ascending": the ring result is bitwise merge_attention over
    the per-source partials in ascending source rank (attention.py:325-326,
    SPEC.md:79, 289), for pass-KV and pass-Q alike; the default arrival order
    stays within tolerance of it."""
    import torch

    from paper_2411_01783_b200.ring import build_kv_message, ring_pass_kv_prefill, ring_pass_q_prefill

    z, n, plan, cfg, qb, kb, vb, caches = _ring_inputs(rc, name)
    kv = ring_pass_kv_prefill(plan, caches(), qb, kb, vb, cfg, merge_order="ascending")
    pq = ring_pass_q_prefill(plan, caches(), qb, kb, vb, cfg, merge_order="ascending")
    arr = ring_pass_kv_prefill(plan, caches(), qb, kb, vb, cfg)
    # reference-style composition: one attention per source message (the ring's
    # own per-step launch), then merge_attention over the partials in ascending
    # source rank
    from paper_2411_01783_b200.ring import _cuda_attend, append_new_tokens

    cs = caches()
    for r in range(n):
        append_new_tokens(plan, r, cs[r], kb[r], vb[r])
    msgs = [build_kv_message(plan, cs[r]) for r in range(n)]
    for r in range(n):
        parts = []
        qp, qs = qb[r].meta32("q")
        for s in range(n):
            lay, buf = msgs[s]
            kk, vv, kp, ks = lay.views(buf)
            o = torch.empty((qb[r].n_tokens, cfg.n_query_heads, 128), device="cuda")
            l = torch.empty((qb[r].n_tokens, cfg.n_query_heads), device="cuda")
            _cuda_attend(qb[r].data.to(torch.bfloat16), qp, qs, kk, vv, kp, ks, cfg, o, l, 0)
            parts.append(rc.PartialAttention(rc.EmbeddingBlock(o, qb[r].positions, qb[r].valid, qb[r].seq_ids,
                                                               validate=False), l))
        want = rc.merge_attention(parts)
        assert torch.equal(kv[r].output.data, want.output.data)
        assert torch.equal(kv[r].lse, want.lse)
        assert torch.equal(pq[r].output.data, want.output.data)
        assert torch.equal(pq[r].lse, want.lse)
        assert float((arr[r].output.data - want.output.data).abs().max()) <= 1e-5
