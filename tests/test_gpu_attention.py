"""GPU parity of gqa_attention / merge_attention (C-ABI kernels) vs the oracle
and the golden vectors produced by the real reference."""


import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rc():
    import torch

    import paper_2411_01783_b200 as rc

    torch.manual_seed(0)
    return rc


def to_dev(rc, b: orc.Blk, bf16=True):
    import torch

    data = torch.from_numpy(np.ascontiguousarray(b.data)).cuda()
    if bf16:
        data = data.to(torch.bfloat16)
    return rc.EmbeddingBlock(data, b.pos, b.valid, b.seq)


D128 = ["d128_ragged200", "fused_r0_r0", "fused_r0_r1", "cached_offset", "peaky",
        "zigzag_q0_k0", "zigzag_q0_k1", "zigzag_q1_k0", "zigzag_q1_k1", "empty_k", "all_pad_k"]


@pytest.mark.parametrize("name", D128)
def test_gqa_matches_reference_golden(rc, name):
    z = G.npz("gqa.npz")
    c = G.gqa_case(z, name)
    cfg = rc.GqaConfig(c["hq"], c["hkv"], c["d"])
    part = rc.gqa_attention(to_dev(rc, c["q"]), to_dev(rc, c["k"]), to_dev(rc, c["v"]), cfg)
    out = part.output.data.cpu().numpy()
    lse = part.lse.cpu().numpy()
    assert np.abs(out - c["out"]).max() <= G.O_TOL
    assert G.lse_err(lse, c["lse"]) <= G.LSE_TOL
    # structural: rows without keys are exactly zero / -inf
    empty = np.isneginf(c["lse"])
    assert np.all(out[empty] == 0.0)


@pytest.mark.parametrize("tq,tk,hq,hkv,qoff", [
    (128, 128, 4, 1, 0), (256, 256, 8, 2, 0), (384, 1000, 4, 4, 700), (77, 333, 16, 1, 300),
    (1024, 1024, 8, 1, 0), (2048, 2048, 32, 8, 0),
])
def test_gqa_random_vs_oracle(rc, tq, tk, hq, hkv, qoff):
    rng = np.random.default_rng(tq * 7 + tk)
    def mk(n, h, pos):
        x = orc.blk_from_tokens(rng.standard_normal((n, h, 128)).astype(np.float32), pos)
        x.data = _bf16_exact(x.data)
        return x
    q = mk(tq, hq, np.arange(qoff, qoff + tq))
    k = mk(tk, hkv, np.arange(tk))
    v = mk(tk, hkv, np.arange(tk))
    want_o, want_l = orc.gqa(q, k, v, hkv)
    cfg = rc.GqaConfig(hq, hkv, 128)
    part = rc.gqa_attention(to_dev(rc, q), to_dev(rc, k), to_dev(rc, v), cfg)
    assert np.abs(part.output.data.cpu().numpy() - want_o).max() <= G.O_TOL
    assert G.lse_err(part.lse.cpu().numpy(), want_l) <= G.LSE_TOL


def _bf16_exact(x):
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def test_q_zero_mask_kat(rc):
    """Q = 0: every admitted key has score 0, so LSE = ln(#admitted) exactly and
    O = mean of admitted V rows (SURVEY finding 8)."""
    rng = np.random.default_rng(5)
    T = 640
    plan_q = orc.materialize([orc.Seq(0, 0, T)], 2, 0, [np.zeros((T, 4, 128), np.float32)])
    vd = _bf16_exact(rng.standard_normal((T, 1, 128)).astype(np.float32))
    kb = orc.materialize([orc.Seq(0, 0, T)], 2, 1, [vd])
    vb = kb
    o, l = orc.gqa(plan_q, kb, vb, 1)
    cfg = rc.GqaConfig(4, 1, 128)
    part = rc.gqa_attention(to_dev(rc, plan_q), to_dev(rc, kb), to_dev(rc, vb), cfg)
    lse = part.lse.cpu().numpy()
    adm = orc.admit_mask(plan_q.valid, plan_q.pos, plan_q.seq, kb.valid, kb.pos, kb.seq).sum(1)
    want = np.where(adm > 0, np.log(np.maximum(adm, 1)), -np.inf)
    assert G.lse_err(lse, np.repeat(want[:, None], 4, 1)) <= 1e-5
    assert np.abs(part.output.data.cpu().numpy() - o).max() <= 1e-2


def test_padding_bitwise_invisible(rc):
    """test_attention.py:81-106 on device: padding rows anywhere in K/V change no bit."""
    rng = np.random.default_rng(11)
    q = orc.blk_from_tokens(_bf16_exact(rng.standard_normal((300, 4, 128)).astype(np.float32)), np.arange(300))
    k = orc.blk_from_tokens(_bf16_exact(rng.standard_normal((300, 2, 128)).astype(np.float32)), np.arange(300))
    v = orc.blk_from_tokens(_bf16_exact(rng.standard_normal((300, 2, 128)).astype(np.float32)), np.arange(300))
    cfg = rc.GqaConfig(4, 2, 128)
    base = rc.gqa_attention(to_dev(rc, q), to_dev(rc, k), to_dev(rc, v), cfg)

    def pad(b, where):
        p = orc.blk_padding(7, b.data.shape[1], 128)
        p.data[:] = np.nan  # padding data may be non-finite (only valid rows are checked)
        return orc.Blk(np.concatenate([b.data[:where], p.data, b.data[where:]]),
                       np.concatenate([b.pos[:where], p.pos, b.pos[where:]]),
                       np.concatenate([b.valid[:where], p.valid, b.valid[where:]]),
                       np.concatenate([b.seq[:where], p.seq, b.seq[where:]]))

    for where in (0, 130, 300):
        got = rc.gqa_attention(to_dev(rc, q), to_dev(rc, pad(k, where)), to_dev(rc, pad(v, where)), cfg)
        assert np.array_equal(got.output.data.cpu().numpy(), base.output.data.cpu().numpy())
        assert np.array_equal(got.lse.cpu().numpy(), base.lse.cpu().numpy())


def test_merge_matches_golden(rc):
    import torch

    z = G.npz("merge.npz")
    for name in z["names"]:
        n = int(z[f"{name}__n"])
        parts = []
        for p in range(n):
            out = z[f"{name}__p{p}__out"].astype(np.float32)
            lse = z[f"{name}__p{p}__lse"].astype(np.float32)
            blk = rc.EmbeddingBlock.from_tokens(torch.from_numpy(out), np.arange(out.shape[0]))
            parts.append(rc.PartialAttention(blk, torch.from_numpy(lse)))
        m = rc.merge_attention(parts)
        if n == 1:
            assert m is parts[0]
        assert np.abs(m.output.data.cpu().numpy() - z[f"{name}__out"]).max() <= 1e-5
        assert G.lse_err(m.lse.cpu().numpy(), z[f"{name}__lse"]) <= 1e-5


def test_split_merge_equals_unsplit(rc):
    """Block-split invariance (test_attention.py:238-280) at D=128 on device."""
    rng = np.random.default_rng(3)
    T = 700
    q = orc.blk_from_tokens(_bf16_exact(rng.standard_normal((200, 8, 128)).astype(np.float32)), np.arange(T, T + 200))
    k = orc.blk_from_tokens(_bf16_exact(rng.standard_normal((T, 2, 128)).astype(np.float32)), np.arange(T))
    cfg = rc.GqaConfig(8, 2, 128)
    whole = rc.gqa_attention(to_dev(rc, q), to_dev(rc, k), to_dev(rc, k), cfg)
    cuts = [0, 129, 130, 400, T]
    parts = []
    for a, b in zip(cuts, cuts[1:]):
        kb = orc.Blk(k.data[a:b], k.pos[a:b], k.valid[a:b], k.seq[a:b])
        parts.append(rc.gqa_attention(to_dev(rc, q), to_dev(rc, kb), to_dev(rc, kb), cfg))
    m = rc.merge_attention(parts)
    assert np.abs(m.output.data.cpu().numpy() - whole.output.data.cpu().numpy()).max() <= 1e-2
    assert np.abs(m.lse.cpu().numpy() - whole.lse.cpu().numpy()).max() <= 1e-4


def test_errors(rc):
    with pytest.raises(ValueError, match="divisible"):
        rc.GqaConfig(3, 2, 128)
    with pytest.raises(ValueError, match="empty"):
        rc.merge_attention([])
    rng = np.random.default_rng(1)
    cfg = rc.GqaConfig(2, 1, 128)
    mk = lambda n, h: rc.EmbeddingBlock.from_tokens(rng.standard_normal((n, h, 128)).astype(np.float32), np.arange(n))
    with pytest.raises(ValueError, match="mismatch"):
        rc.gqa_attention(mk(2, 2), mk(2, 1), mk(3, 1), cfg)
    with pytest.raises(ValueError):
        rc.gqa_attention(mk(2, 2), mk(2, 2), mk(2, 2), cfg)
