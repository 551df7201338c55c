"""One causal GQA attention launch for ncu captures (warm-up launch first).

  ncu --set full --import-source on -k regex:attn_fwd --launch-skip 1 -c 1 \
      -o gpurun_out/attn python tools/profile_attn.py 65536
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_01783_b200.attention import attend_into  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
HQ, HKV = 32, 8
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(T, HQ, 128, device=dev, dtype=torch.bfloat16, generator=g)
k = torch.randn(T, HKV, 128, device=dev, dtype=torch.bfloat16, generator=g)
v = torch.randn(T, HKV, 128, device=dev, dtype=torch.bfloat16, generator=g)
pos = torch.arange(T, device=dev, dtype=torch.int32)
seq = torch.zeros(T, device=dev, dtype=torch.int32)
out = torch.empty(T, HQ, 128, device=dev, dtype=torch.float32)
lse = torch.empty(T, HQ, device=dev, dtype=torch.float32)
for _ in range(2):
    attend_into(q, (pos, seq), k, v, (pos, seq), HQ, HKV, 128 ** -0.5, out, lse, 0)
torch.cuda.synchronize()
print("ok", float(lse[-1, 0]))
