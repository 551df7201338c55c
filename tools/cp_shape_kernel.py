"""Per-launch attention kernel efficiency at CP-N ring-step shapes.

For the 8B-shaped 128K prefill and N in (1, 2, 4, 8): rank 0's query block
against every rank's key/value block (the N launches rank 0 makes in a
pass-KV ring), each launch timed alone with CUDA events (median of 5) on
admitted-pair FLOPs.  Separates kernel efficiency at small launch shapes from
the host/ring overheads cp_shape_efficiency.py includes.

  python tools/cp_shape_kernel.py [T] [merge]

With "merge" every launch folds into a running (O, LSE) (RCP_MODE_MERGE, what
ring steps after the first do).
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200 import _lib  # noqa: E402
from paper_2411_01783_b200.attention import admitted_pair_count, attend_into  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
MODE = _lib.MODE_MERGE if "merge" in sys.argv[2:] else _lib.MODE_OVERWRITE
hq, hkv, D = 32, 8, 128
cfg = rc.GqaConfig(hq, hkv, D)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(T, hq, D, device="cuda", dtype=torch.bfloat16, generator=g)
k = torch.randn(T, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
v = torch.randn(T, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
for n in (1, 2, 4, 8):
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], n)
    qb = materialize_rank_block(plan, 0, [q])
    tot_f, tot_ms = 0.0, 0.0
    parts = []
    for src in range(n):
        kb = materialize_rank_block(plan, src, [k])
        vb = materialize_rank_block(plan, src, [v])
        kk, vv = kb.valid_only(), vb.valid_only()
        flops = 4.0 * D * hq * admitted_pair_count(qb, kk)
        out = torch.zeros(qb.n_tokens, hq, D, device="cuda")
        lse = torch.zeros(qb.n_tokens, hq, device="cuda")
        ws = torch.empty(max(_lib.load().rcp_attn_workspace_bytes(qb.n_tokens, kk.n_tokens), 32),
                         dtype=torch.uint8, device="cuda")
        ts = []
        for it in range(7):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            attend_into(qb.data, qb.meta32("q"), kk.data, vv.data, kk.meta32("k"), hq, hkv, cfg.scale,
                        out, lse, MODE, workspace=ws)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = statistics.median(ts[2:])
        tot_f += flops
        tot_ms += ms
        parts.append(f"src{src} {ms:.2f} ms {flops / ms / 1e9:.0f}")
    print(f"CP{n}: rank-0 launches {qb.n_tokens} x {T // n}: " + "; ".join(parts) +
          f" | sum {tot_ms:.2f} ms -> {tot_f / tot_ms / 1e9:.0f} TF/s", flush=True)
