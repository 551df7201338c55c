"""Randomised soak of the attention kernel against a plain fp32 torch reference.

60 random cases (fixed seeds): 1..2500 query rows, 1..3000 keys, one to three
sequences per block with padding rows between them, random monotone
positions (gaps, shared positions across sequences), GQA ratios 1..16, and
both modes (overwrite; merge into a random running (O, LSE)).  The reference
is the masked softmax of the reference's attention.py:230-282 in fp32 on the
GPU (same bf16 inputs); tolerances are the suite's bf16 ones.  Meant to catch
rare schedule / barrier races that fixed shapes would miss.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAD_Q, PAD_K, POS_PAD_K = -(2 ** 31), -(2 ** 31) + 1, 2 ** 31 - 1


def _block(rng, n, n_seq, seq_ids, pad_seq, pad_pos):
    """n rows split over up to n_seq sequences with a few padding rows."""
    pos = np.empty(n, np.int64)
    seq = np.empty(n, np.int64)
    cuts = np.sort(rng.choice(np.arange(1, n), size=min(n_seq - 1, max(n - 1, 0)), replace=False)) if n > 1 else []
    bounds = [0, *cuts, n]
    for i in range(len(bounds) - 1):
        a, b = bounds[i], bounds[i + 1]
        start = int(rng.integers(0, 500))
        steps = rng.integers(1, 3, size=b - a)  # strictly increasing positions with gaps
        pos[a:b] = start + np.cumsum(steps) - steps[0]
        seq[a:b] = seq_ids[i % len(seq_ids)]
    pad = rng.random(n) < 0.05
    pos32 = np.where(pad, pad_pos, pos).astype(np.int32)
    seq32 = np.where(pad, pad_seq, seq).astype(np.int32)
    return pos32, seq32


def _reference(q, k, v, qp, qs, kp, ks, hq, hkv, scale):
    """fp32 masked softmax attention; rows without admitted keys -> O 0, LSE -inf."""
    g = hq // hkv
    qf = q.float().transpose(0, 1)                             # [Hq, Tq, D]
    kf = k.float().transpose(0, 1).repeat_interleave(g, 0)     # [Hq, Tk, D]
    vf = v.float().transpose(0, 1).repeat_interleave(g, 0)
    s = torch.matmul(qf, kf.transpose(1, 2)) * scale           # [Hq, Tq, Tk]
    ok = (qs[:, None] == ks[None, :]) & (kp[None, :] <= qp[:, None]) & (qs[:, None] != PAD_Q)
    s = s.masked_fill(~ok[None], float("-inf"))
    lse = torch.logsumexp(s, dim=-1)                           # [Hq, Tq]
    p = torch.exp(s - torch.where(torch.isfinite(lse), lse, torch.zeros_like(lse))[..., None])
    p = torch.where(ok[None], p, torch.zeros_like(p))
    o = torch.matmul(p, vf)
    return o.transpose(0, 1), lse.transpose(0, 1)


@pytest.mark.parametrize("case", range(60))
def test_attention_random_soak(case):
    from paper_2411_01783_b200.attention import attend_into
    from paper_2411_01783_b200 import _lib

    rng = np.random.default_rng(1000 + case)
    hkv = int(rng.choice([1, 2, 4, 8]))
    g = int(rng.choice([1, 2, 4, 8, 16]))
    hq = hkv * g
    if hq > 64:
        hq, g = 64, 64 // hkv
    tq = int(rng.integers(1, 2500))
    tk = int(rng.integers(1, 3000))
    seq_ids = [int(x) for x in rng.choice(50, size=3, replace=False)]
    n_seq = int(rng.integers(1, 4))
    qp, qs = _block(rng, tq, n_seq, seq_ids, PAD_Q, -1)
    kp, ks = _block(rng, tk, n_seq, seq_ids, PAD_K, POS_PAD_K)
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(case)
    q = torch.randn(tq, hq, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    k = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    v = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    qp_d, qs_d = torch.from_numpy(qp).to(dev), torch.from_numpy(qs).to(dev)
    kp_d, ks_d = torch.from_numpy(kp).to(dev), torch.from_numpy(ks).to(dev)
    scale = 1.0 / math.sqrt(128)
    merge = bool(case % 3 == 2)
    out = torch.randn(tq, hq, 128, device=dev) if merge else torch.empty(tq, hq, 128, device=dev)
    lse = torch.randn(tq, hq, device=dev) if merge else torch.empty(tq, hq, device=dev)
    o0, l0 = out.clone(), lse.clone()
    attend_into(q, (qp_d, qs_d), k, v, (kp_d, ks_d), hq, hkv, scale, out, lse,
                _lib.MODE_MERGE if merge else _lib.MODE_OVERWRITE)
    ro, rl = _reference(q, k, v, qp_d.long(), qs_d.long(), kp_d.long(), ks_d.long(), hq, hkv, scale)
    if merge:  # exact LSE merge of the running (o0, l0) with the new partial
        m = torch.maximum(l0, rl)
        m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
        wa, wb = torch.exp(l0 - m), torch.exp(rl - m)
        tot = wa + wb
        rl = torch.log(tot) + m
        ro = (o0 * wa[..., None] + ro * wb[..., None]) / tot[..., None]
    torch.cuda.synchronize()
    valid = torch.from_numpy(qs != PAD_Q).to(dev)
    assert torch.isfinite(out[valid]).all()
    assert (out[valid] - ro[valid]).abs().max().item() <= 2e-2
    fin = torch.isfinite(rl) & valid[:, None]
    assert torch.equal(torch.isfinite(lse) & valid[:, None], fin)
    if fin.any():
        assert (lse[fin] - rl[fin]).abs().max().item() <= 1e-3
