"""RankKvCache on the device: the SPEC's append / snapshot_padded examples
(SPEC.md:180-198), the round-trip and capacity-balance invariants
(SPEC.md:200-203), VMM growth without moving or copying cached rows, and
eviction / segment reuse."""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc

pytestmark = pytest.mark.gpu

H, D = 2, 128


def _blk(rc, n, positions, seq=0, seed=0):
    import torch

    rng = np.random.default_rng(seed)
    data = torch.from_numpy(rng.standard_normal((n, H, D)).astype(np.float32)).to(torch.bfloat16)
    return rc.EmbeddingBlock(data.cuda(), np.asarray(positions), np.ones(n, bool), np.full(n, seq))


@pytest.fixture(scope="module")
def rc():
    import paper_2411_01783_b200 as rc

    return rc


def test_spec_append_examples(rc):
    from paper_2411_01783_b200.kv_cache import RankKvCache

    c = RankKvCache(H, D, capacity_tokens=8)
    k = _blk(rc, 4, np.arange(4))
    assert c.append(0, k, k) == 4  # empty cache, append 4 tokens -> cached_len 4
    # chunks {0..3} then {12..15}: retrieval yields positions sorted ascending
    k2 = _blk(rc, 4, np.arange(12, 16), seed=1)
    assert c.append(0, k2, k2) == 8
    kb, vb = c.snapshot_padded(0, 8)
    assert kb.positions.cpu().tolist() == [0, 1, 2, 3, 12, 13, 14, 15]
    # out-of-order append (chunk 12..15 before 4..7) is re-sorted
    k3 = _blk(rc, 4, np.arange(4, 8), seed=2)
    c.append(0, k3, k3)
    assert c.snapshot_padded(0, 12)[0].positions.cpu().tolist() == list(range(8)) + list(range(12, 16))
    # shape / head-count mismatch is an error
    with pytest.raises(ValueError):
        bad = rc.EmbeddingBlock(np.zeros((2, H + 1, D), np.float32), np.arange(2), np.ones(2, bool), np.zeros(2))
        c.append(0, bad, bad)
    c.close()


def test_spec_snapshot_examples_and_round_trip(rc):
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache

    c = RankKvCache(H, D, capacity_tokens=16)
    k = _blk(rc, 10, np.arange(10), seed=3)
    v = _blk(rc, 10, np.arange(10), seed=4)
    c.append(0, k, v)
    kb, vb = c.snapshot_padded(0, 16)  # cached_len 10, max_len 16 -> 6 padding rows
    assert kb.n_tokens == 16 and kb.n_valid == 10
    assert kb.valid.cpu().tolist() == [True] * 10 + [False] * 6
    assert kb.positions.cpu().tolist()[10:] == [-1] * 6 and kb.seq_ids.cpu().tolist()[10:] == [-1] * 6
    kb2, vb2 = c.snapshot_padded(0, 10)  # cached_len = max_len -> zero padding; round trip exact
    assert kb2.n_tokens == 10
    assert torch.equal(kb2.data, k.data) and torch.equal(vb2.data, v.data)
    with pytest.raises(ValueError):
        c.snapshot_padded(0, 9)  # max_len < cached_len
    # the snapshot is a copy: the cache is not modified by changing it
    kb2.data.zero_()
    assert torch.equal(c.snapshot_padded(0, 10)[0].data, k.data)
    c.close()


def test_vmm_growth_keeps_base_pointer_and_rows(rc):
    """Growing past the mapped capacity maps more memory behind the same base
    pointer: no cached row is copied or moved."""
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache

    c = RankKvCache(H, D, capacity_tokens=64, max_tokens=1 << 22)
    assert c.growth == "vmm"
    k = _blk(rc, 1000, np.arange(1000), seq=5, seed=6)
    c.append(5, k, k)
    base = (c.k.data_ptr(), c.v.data_ptr(), c.pos.data_ptr())
    cap0 = c.k.shape[0]
    big = _blk(rc, 300000, np.arange(1000, 301000), seq=7, seed=7)
    c.append(7, big, big)  # forces growth far beyond the first mapping
    assert c.k.shape[0] > cap0
    assert (c.k.data_ptr(), c.v.data_ptr(), c.pos.data_ptr()) == base
    st, ln = c.segment(5)
    assert torch.equal(c.k[st:st + ln], k.data)
    st, ln = c.segment(7)
    assert torch.equal(c.k[st:st + ln], big.data)
    assert c.pos[st:st + ln].cpu().tolist()[:3] == [1000, 1001, 1002]
    c.close()


def test_evict_reuses_segment(rc):
    from paper_2411_01783_b200.kv_cache import RankKvCache

    c = RankKvCache(H, D, capacity_tokens=64)
    for sid in range(3):
        k = _blk(rc, 100, np.arange(100), seq=sid, seed=sid)
        c.append(sid, k, k)
    st1, _ = c.segment(1)
    used = c._used
    assert c.evict(1) == 100 and c.cached_len(1) == 0
    k = _blk(rc, 90, np.arange(90), seq=9, seed=9)
    c.append(9, k, k)  # fits in the freed segment (first fit)
    assert c.segment(9)[0] == st1 and c._used == used
    kb, _ = c.snapshot_padded(9, 90)
    assert kb.positions.cpu().tolist() == list(range(90))
    c.close()


@pytest.mark.parametrize("n,B,k", [(4, 3, 2), (8, 5, 3), (3, 7, 4)])
def test_capacity_balance_after_ring_decode(rc, n, B, k):
    """after k·N iterations of Alg. 4 on a B-sequence batch the
    spread of cached rows over ranks is at most B, and every decoded token is
    cached exactly once (Σ-invariant), on the device caches the ring uses."""
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache, capacity_balance
    from paper_2411_01783_b200.ring import ring_pass_q_decode
    from paper_2411_01783_b200.sharding import plan_decode

    hq = 4
    cfg = rc.GqaConfig(hq, H, D)
    caches = [RankKvCache(H, D, capacity_tokens=64) for _ in range(n)]
    batch = list(range(B))
    pos = {b: 0 for b in batch}
    rng = np.random.default_rng(n * 100 + B)
    for it in range(k * n):
        plan = plan_decode(batch, n, it)
        q, kk, vv = (torch.from_numpy(rng.standard_normal((B, h, D)).astype(np.float32)).to(torch.bfloat16).cuda()
                     for h in (hq, H, H))
        ring_pass_q_decode(plan, caches, q, kk, vv, [pos[b] for b in batch], cfg)
        for b in batch:
            pos[b] += 1
    rep = capacity_balance(caches, batch)
    assert rep["spread"] <= B, rep
    assert all(v == k * n for v in rep["per_seq_total"].values()), rep
    # the oracle's round-robin gives the same per-rank rows
    want = [0] * n
    for it in range(k * n):
        for r, a in enumerate(orc.decode_assignments(batch, n, it)):
            want[r] += len(a)
    assert rep["per_rank"] == want
    for c in caches:
        c.close()
