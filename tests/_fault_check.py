"""Run by tests/test_gpu_negative_controls.py in a fresh process with RCP_FAULT
set (the library reads it once): the parity harness's checks on a small case,
printed as one JSON line.  Under a fault some check MUST fail."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01783_b200 as rc  # noqa: E402
from oracle import ringcp_oracle as orc  # noqa: E402
from tests import _golden as G  # noqa: E402
from tests.golden.make_golden_inputs import bf16_exact  # noqa: E402

# 1) gqa_attention vs the fp64 oracle (causal, 1024 tokens, GQA 8/2)
T, hq, hkv = 1024, 8, 2
rng = np.random.default_rng(0)
q, k, v = (orc.blk_from_tokens(bf16_exact(rng.standard_normal((T, h, 128)).astype(np.float32)), np.arange(T))
           for h in (hq, hkv, hkv))
want_o, want_l = orc.gqa(q, k, v, hkv)
dev = [rc.EmbeddingBlock(torch.from_numpy(b.data).cuda().to(torch.bfloat16), b.pos, b.valid, b.seq) for b in (q, k, v)]
part = rc.gqa_attention(*dev, rc.GqaConfig(hq, hkv, 128))
d_o = float(np.abs(part.output.data.cpu().numpy() - want_o).max())
d_l = G.lse_err(part.lse.cpu().numpy(), want_l)

# 2) protocol equivalence: pass-KV (fused running merge) == pass-Q (All2All + merge kernel), bitwise
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import ring_pass_kv_prefill, ring_pass_q_prefill  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402

z = G.npz("ring.npz")
name = "ring_n3_fused"
meta = [int(x) for x in z[f"{name}__meta"]]
n, rhq, rhkv, lens = meta[0], meta[1], meta[2], meta[3:]
plan = plan_full_prefill([SequenceSpec(i, 0, t) for i, t in enumerate(lens)], n)
cfg = rc.GqaConfig(rhq, rhkv, 128)
todev = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
blocks = [[materialize_rank_block(plan, r, [todev(z[f"{name}__{x}{i}"]) for i in range(len(lens))]) for r in range(n)]
          for x in "qkv"]
caches = lambda: [RankKvCache(rhkv, 128, capacity_tokens=256) for _ in range(n)]
kv = ring_pass_kv_prefill(plan, caches(), *blocks, cfg)
pq = ring_pass_q_prefill(plan, caches(), *blocks, cfg)
bitwise = all(torch.equal(kv[r].output.data, pq[r].output.data) and torch.equal(kv[r].lse, pq[r].lse)
              for r in range(n))
ring_err = max(float(np.abs(kv[r].output.data.cpu().numpy() - z[f"{name}__r{r}__out"]).max()) for r in range(n))
print(json.dumps({"fault": os.environ.get("RCP_FAULT", ""), "max_dO": d_o, "max_dLSE": d_l,
                  "parity_ok": d_o <= G.O_TOL and d_l <= G.LSE_TOL and ring_err <= G.O_TOL,
                  "ring_bitwise_kv_eq_q": bitwise}))
