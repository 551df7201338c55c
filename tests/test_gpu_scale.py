"""GPU parity at BASELINE scale (VERDICT r1 "next" #1; SURVEY §8c large-T oracle).

* cfg1 exactly (BASELINE configs[0]): pass-KV / pass-Q, CP=2 simulated ranks,
  T=4096, 8 Q / 1 KV heads, default_rng(0) inputs rounded to bf16, against the
  FULL composed oracle (every row).
* cfg2 shape (8B, 32/8 heads) at 128K tokens: the bench's own path at CP1
  (RingAttention.pass_kv_prefill, world 1) and the CP8 ring over 8 simulated
  ranks (64 launches of 16384 x 16384, fused running merge), plus single
  launches at the CP8 step shapes (diagonal / off-diagonal, normal and peaky Q).
* 405B shape (128/8 heads) at 128K over 4 simulated ranks.

Large cases are checked on sampled rows (first / last token, both sides of
every chunk boundary, random rows) against the fp64 oracle
(oracle/sampled_check.py); tolerance |dO| <= 2e-2, |dLSE| <= 1e-3.
"""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from oracle.sampled_check import check_rank_rows
from tests import _golden as G
from tests.golden.make_golden_inputs import bf16_exact

pytestmark = pytest.mark.gpu

D = 128


@pytest.fixture(autouse=True)
def _free():
    import torch

    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _inputs(T, hq, hkv, seeds=(11, 12, 13), q_scale=1.0):
    """Synthetic bf16 inputs exactly as bench.py makes them (torch CUDA generator)."""
    import torch

    g = torch.Generator(device="cuda")
    out = []
    for h, s in zip((hq, hkv, hkv), seeds):
        g.manual_seed(s)
        out.append(torch.randn((T, h, D), generator=g, device="cuda", dtype=torch.bfloat16))
    if q_scale != 1.0:
        out[0] = (out[0].float() * q_scale).to(torch.bfloat16)
    return out


def _ok(res):
    assert res["max_dO"] <= G.O_TOL, res
    assert res["max_dLSE"] <= G.LSE_TOL, res


def test_cfg1_exact_full_oracle():
    """BASELINE configs[0]: pass-KV full prefill, CP=2 simulated ranks, T=4096,
    8 Q / 1 KV head, head_dim 128 — every output row vs the composed oracle."""
    import torch

    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_kv_prefill, ring_pass_q_prefill
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    T, n, hq, hkv = 4096, 2, 8, 1
    rng = np.random.default_rng(0)
    q = bf16_exact(rng.standard_normal((T, hq, D)).astype(np.float32))
    k = bf16_exact(rng.standard_normal((T, hkv, D)).astype(np.float32))
    v = bf16_exact(rng.standard_normal((T, hkv, D)).astype(np.float32))
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    cfg = rc.GqaConfig(hq, hkv, D)
    dev = [torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (q, k, v)]
    blocks = [[materialize_rank_block(plan, r, [t]) for r in range(n)] for t in dev]
    kv = ring_pass_kv_prefill(plan, [RankKvCache(hkv, D, capacity_tokens=T) for _ in range(n)], *blocks, cfg)
    pq = ring_pass_q_prefill(plan, [RankKvCache(hkv, D, capacity_tokens=T) for _ in range(n)], *blocks, cfg)
    _, want = orc.ring_prefill([orc.Seq(0, 0, T)], [[0] * n], n, [orc.Cache(hkv, D) for _ in range(n)],
                               [q], [k], [v], hkv)
    for r in range(n):
        o = kv[r].output.data.cpu().numpy()
        l = kv[r].lse.cpu().numpy()
        assert np.abs(o - want[r][0]).max() <= G.O_TOL
        assert G.lse_err(l, want[r][1]) <= G.LSE_TOL
        assert np.array_equal(o, pq[r].output.data.cpu().numpy())
        assert np.array_equal(l, pq[r].lse.cpu().numpy())


def test_8b_128k_cp1_bench_path_sampled():
    """The exact path bench.py times at N=1 (RingAttention.pass_kv_prefill,
    world 1: device shard gather, cache append, KV message, one launch)."""
    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    T, hq, hkv = 131072, 32, 8
    q, k, v = _inputs(T, hq, hkv)
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], 1)
    cfg = rc.GqaConfig(hq, hkv, D)
    ring = RingAttention(_LocalComm(0, 1))
    cache = RankKvCache(hkv, D, capacity_tokens=T + 4096, device=q.device)
    part = ring.pass_kv_prefill(plan, cache, *(materialize_rank_block(plan, 0, [t]) for t in (q, k, v)), cfg)
    res = check_rank_rows(T, 1, 0, part.output.data, part.lse, q, k, v, hkv, cfg.scale, count=32)
    assert res["rows"] >= 32
    _ok(res)


def test_8b_128k_cp8_simulated_ring_sampled():
    """CP8 over 8 simulated ranks at 128K: 64 launches of 16384 x 16384 with the
    fused running merge; pass-Q bitwise equal to pass-KV."""
    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_kv_prefill, ring_pass_q_prefill
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    import torch

    T, n, hq, hkv = 131072, 8, 32, 8
    q, k, v = _inputs(T, hq, hkv)
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    cfg = rc.GqaConfig(hq, hkv, D)
    blocks = [[materialize_rank_block(plan, r, [t]) for r in range(n)] for t in (q, k, v)]
    caches = lambda: [RankKvCache(hkv, D, capacity_tokens=T // n + 256) for _ in range(n)]
    outs = ring_pass_kv_prefill(plan, caches(), *blocks, cfg)
    kh, vh = k.float().cpu().numpy(), v.float().cpu().numpy()
    rows = orc.sample_rows(T, n, 48, seed=1)
    total = 0
    for r in range(n):
        res = check_rank_rows(T, n, r, outs[r].output.data, outs[r].lse, q, k, v, hkv, cfg.scale, rows=rows,
                              k_host=kh, v_host=vh)
        total += res["rows"]
        _ok(res)
    assert total == len(rows)
    pq = ring_pass_q_prefill(plan, caches(), *blocks, cfg)
    for r in range(n):
        assert torch.equal(outs[r].output.data, pq[r].output.data)
        assert torch.equal(outs[r].lse, pq[r].lse)


@pytest.mark.parametrize("src,q_scale", [(0, 1.0), (5, 1.0), (0, 4.0), (3, 4.0)])
def test_cp8_step_launch_shape(src, q_scale):
    """One attention launch at a CP8 ring-step shape (rank 0's 16384 query
    slots against rank src's 16384-slot KV message; src=0 is the diagonal
    step), OVERWRITE mode, normal and peaky (x4) queries."""
    import torch

    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200 import _lib
    from paper_2411_01783_b200.attention import attend_into
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    T, n, hq, hkv = 131072, 8, 32, 8
    q, k, v = _inputs(T, hq, hkv, q_scale=q_scale)
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    cfg = rc.GqaConfig(hq, hkv, D)
    qb = materialize_rank_block(plan, 0, [q])
    kb = materialize_rank_block(plan, src, [k]).valid_only()
    vb = materialize_rank_block(plan, src, [v]).valid_only()
    out = torch.empty(qb.n_tokens, hq, D, device="cuda")
    lse = torch.empty(qb.n_tokens, hq, device="cuda")
    attend_into(qb.data, qb.meta32("q"), kb.data, vb.data, kb.meta32("k"), hq, hkv, cfg.scale, out, lse,
                _lib.MODE_OVERWRITE)
    # oracle: rank 0's sampled query rows against exactly this key block
    slots = np.array([0, 1, 8191, 8192, 16383] + list(np.random.default_rng(src).integers(0, 16384, 11)))
    toks = plan.rank_local_indices(0, 0)[slots]
    kt = plan.rank_local_indices(0, src)
    kt = kt[kt >= 0]
    qr = q[torch.from_numpy(toks).cuda()].float().cpu().numpy()
    kh = k[torch.from_numpy(kt).cuda()].float().cpu().numpy()
    vh = v[torch.from_numpy(kt).cuda()].float().cpu().numpy()
    want_o, want_l = orc.sampled_rows_attention(orc.blk_from_tokens(qr, toks), orc.blk_from_tokens(kh, kt),
                                                orc.blk_from_tokens(vh, kt), hkv, cfg.scale)
    sl = torch.from_numpy(slots).cuda()
    assert np.abs(out[sl].double().cpu().numpy() - want_o).max() <= G.O_TOL
    assert G.lse_err(lse[sl].cpu().numpy(), want_l) <= G.LSE_TOL


def test_405b_128k_cp4_simulated_ring_sampled():
    """405B-shaped GQA layer (128 Q / 8 KV heads) at 128K over 4 simulated ranks."""
    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_kv_prefill
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    T, n, hq, hkv = 131072, 4, 128, 8
    q, k, v = _inputs(T, hq, hkv)
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    cfg = rc.GqaConfig(hq, hkv, D)
    blocks = [[materialize_rank_block(plan, r, [t]) for r in range(n)] for t in (q, k, v)]
    outs = ring_pass_kv_prefill(plan, [RankKvCache(hkv, D, capacity_tokens=T // n + 256) for _ in range(n)],
                                *blocks, cfg)
    kh, vh = k.float().cpu().numpy(), v.float().cpu().numpy()
    rows = orc.sample_rows(T, n, 16, seed=2)
    for r in range(n):
        _ok(check_rank_rows(T, n, r, outs[r].output.data, outs[r].lse, q, k, v, hkv, cfg.scale, rows=rows,
                            k_host=kh, v_host=vh))
