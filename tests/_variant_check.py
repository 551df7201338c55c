"""Run by tests/test_gpu_variants.py in a fresh process with RCP_ATTN_VERSION
set (the library reads it once): a few attention cases of the selected
kernel variant against the fp32 torch reference of the soak test."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_01783_b200 import _lib  # noqa: E402
from paper_2411_01783_b200.attention import attend_into  # noqa: E402
from tests.test_gpu_attention_soak import _block, _reference, PAD_Q, PAD_K, POS_PAD_K  # noqa: E402

assert _lib.load().rcp_attn_version() == int(os.environ["RCP_ATTN_VERSION"]), "kernel form not selected"
worst_o, worst_l = 0.0, 0.0
for case in range(8):
    rng = np.random.default_rng(500 + case)
    hkv = int(rng.choice([1, 2, 8]))
    g = int(rng.choice([1, 4, 8]))
    hq = hkv * g
    tq = int(rng.integers(200, 2100))
    tk = int(rng.integers(200, 2600))
    seq_ids = [3, 9]
    qp, qs = _block(rng, tq, 2, seq_ids, PAD_Q, -1)
    kp, ks = _block(rng, tk, 2, seq_ids, PAD_K, POS_PAD_K)
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(case)
    q = torch.randn(tq, hq, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    k = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    v = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=gen)
    qp_d, qs_d = torch.from_numpy(qp).to(dev), torch.from_numpy(qs).to(dev)
    kp_d, ks_d = torch.from_numpy(kp).to(dev), torch.from_numpy(ks).to(dev)
    scale = 1.0 / math.sqrt(128)
    merge = case % 2 == 1
    out = torch.randn(tq, hq, 128, device=dev) if merge else torch.empty(tq, hq, 128, device=dev)
    lse = torch.randn(tq, hq, device=dev) if merge else torch.empty(tq, hq, device=dev)
    o0, l0 = out.clone(), lse.clone()
    attend_into(q, (qp_d, qs_d), k, v, (kp_d, ks_d), hq, hkv, scale, out, lse,
                _lib.MODE_MERGE if merge else _lib.MODE_OVERWRITE)
    ro, rl = _reference(q, k, v, qp_d.long(), qs_d.long(), kp_d.long(), ks_d.long(), hq, hkv, scale)
    if merge:
        m = torch.maximum(l0, rl)
        m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
        wa, wb = torch.exp(l0 - m), torch.exp(rl - m)
        tot = wa + wb
        rl = torch.log(tot) + m
        ro = (o0 * wa[..., None] + ro * wb[..., None]) / tot[..., None]
    torch.cuda.synchronize()
    valid = torch.from_numpy(qs != PAD_Q).to(dev)
    worst_o = max(worst_o, float((out[valid] - ro[valid]).abs().max()))
    fin = torch.isfinite(rl) & valid[:, None]
    assert torch.equal(torch.isfinite(lse) & valid[:, None], fin), case
    if fin.any():
        worst_l = max(worst_l, float((lse[fin] - rl[fin]).abs().max()))
print(f"version {os.environ.get('RCP_ATTN_VERSION')}: max |dO| {worst_o:.2e}, max |dLSE| {worst_l:.2e}")
assert worst_o <= 2e-2 and worst_l <= 1e-3
