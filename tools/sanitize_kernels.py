"""One small launch of every product kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):

  compute-sanitizer --tool memcheck python tools/sanitize_kernels.py

K1 attention (every form: RCP_ATTN_VERSION=4 default, 12, 13 via env) with
ragged / padded / fused-sequence metadata in overwrite and merge mode; K0 shard
gather + scatter; K2 merge (fixed-N and generic); K4 split-KV decode +
combine; fold / fill / step-select helpers.  Small shapes: the tools replay
every access."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200 import _lib  # noqa: E402
from paper_2411_01783_b200.attention import attend_into, merge_rows_into  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import _cuda_decode  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill, unshard  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
rn = lambda *s: torch.randn(s, generator=g, device=dev, dtype=torch.bfloat16)

# K1: two fused sequences with padding in the middle, GQA 8/2, overwrite + merge
tq, tk, hq, hkv = 300, 420, 8, 2
qpos = torch.tensor(list(range(100, 250)) + [-1] * 10 + list(range(0, 140)), dtype=torch.int32, device=dev)
qseq = torch.tensor([3] * 150 + [_lib.SEQ_PAD_Q] * 10 + [9] * 140, dtype=torch.int32, device=dev)
kpos = torch.tensor(list(range(0, 260)) + [_lib.POS_PAD_K] * 20 + list(range(0, 140)), dtype=torch.int32, device=dev)
kseq = torch.tensor([3] * 260 + [_lib.SEQ_PAD_K] * 20 + [9] * 140, dtype=torch.int32, device=dev)
q, k, v = rn(tq, hq, 128), rn(tk, hkv, 128), rn(tk, hkv, 128)
o = torch.empty(tq, hq, 128, device=dev)
lse = torch.empty(tq, hq, device=dev)
attend_into(q, (qpos, qseq), k, v, (kpos, kseq), hq, hkv, 128 ** -0.5, o, lse, _lib.MODE_OVERWRITE)
attend_into(q, (qpos, qseq), k, v, (kpos, kseq), hq, hkv, 128 ** -0.5, o, lse, _lib.MODE_MERGE)
torch.cuda.synchronize()
print("K1 ok", os.environ.get("RCP_ATTN_VERSION", "default"))

# K0 gather / scatter
plan = plan_full_prefill([SequenceSpec(0, 0, 1000), SequenceSpec(1, 0, 333)], 3)
x = [rn(1000, 2, 128), rn(333, 2, 128)]
blocks = [materialize_rank_block(plan, r, x) for r in range(3)]
back = unshard(plan, [b.data for b in blocks])
assert all(torch.equal(a, b) for a, b in zip(x, back))
print("K0 ok")

# K2 merge: fixed-N (3) and generic (9) forms
parts_o = [torch.randn(257, 4, 128, device=dev) for _ in range(9)]
parts_l = [torch.randn(257, 4, device=dev) for _ in range(9)]
mo, ml = torch.empty(257, 4, 128, device=dev), torch.empty(257, 4, device=dev)
merge_rows_into(parts_o[:3], parts_l[:3], mo, ml)
merge_rows_into(parts_o, parts_l, mo, ml)
torch.cuda.synchronize()
print("K2 ok")

# K4 decode over a small cache (GQA 16/2), three sequences incl. an empty one
cfg = rc.GqaConfig(16, 2, 128)
cache = RankKvCache(2, 128, capacity_tokens=64)
for sid, L in ((0, 700), (1, 65)):
    cache.append_rows(sid, rn(L, 2, 128), rn(L, 2, 128), np.arange(L))
starts = torch.tensor([cache.segment(0)[0], cache.segment(1)[0], 0], dtype=torch.int64, device=dev)
lens = torch.tensor([700, 65, 0], dtype=torch.int64, device=dev)
do, dl = torch.empty(3, 16, 128, device=dev), torch.empty(3, 16, device=dev)
_cuda_decode(rn(3, 16, 128), cache.k, cache.v, starts, lens, 700, cfg, do, dl)
torch.cuda.synchronize()
cache.close()
print("K4 ok")
