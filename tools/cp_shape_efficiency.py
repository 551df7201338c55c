"""Attention efficiency at CP-N per-step shapes, emulated on one GPU.

Runs the simulated-rank ring (ring_pass_kv_prefill: all N ranks' steps in
sequence on one GPU) for the 8B-shaped 128K prefill, so the total work equals
the whole problem while every kernel launch has the CP-N per-step shape.
Reports TF/s (total algorithmic FLOPs / time) per N.

  python tools/cp_shape_efficiency.py [T]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import ring_pass_kv_prefill  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
hq, hkv, D = 32, 8, 128
cfg = rc.GqaConfig(hq, hkv, D)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(T, hq, D, device="cuda", dtype=torch.bfloat16, generator=g)
k = torch.randn(T, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
v = torch.randn(T, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
flops = 4.0 * D * hq * T * (T + 1) / 2
for n in (1, 2, 4, 8):
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    qb = [materialize_rank_block(plan, r, [q]) for r in range(n)]
    kb = [materialize_rank_block(plan, r, [k]) for r in range(n)]
    vb = [materialize_rank_block(plan, r, [v]) for r in range(n)]
    ts = []
    for it in range(3):
        caches = [RankKvCache(hkv, D, capacity_tokens=T // n + 4096) for _ in range(n)]
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        ring_pass_kv_prefill(plan, caches, qb, kb, vb, cfg)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
        del caches
    ms = min(ts[1:])
    print(f"CP{n} shapes: {ms:.1f} ms for the whole problem -> {flops / ms / 1e9:.0f} TF/s "
          f"({n * n} launches of {T // n} x {T // n})", flush=True)
