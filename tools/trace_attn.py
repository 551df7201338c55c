"""Pipeline timeline of attn_fwd_kernel from the RCP_TRACE build.

Builds are separate: paper_2411_01783_b200/_ringcp_b200_trace.so is compiled
with -DRCP_TRACE=1 (see tools/build_trace.sh).  Runs one causal attention of
T tokens and prints, for the first traced CTAs, per-iteration cycle deltas of
the MMA issue points, the softmax windows and the TMA loads.
"""

import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_01783_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_2411_01783_b200", "_ringcp_b200_trace.so")
lib = _lib.load()
lib.rcp_debug_set_trace.argtypes = [ctypes.c_void_p]

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200.attention import attend_into  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
HQ, HKV = 32, 8
dev = torch.device("cuda")
q = torch.randn(T, HQ, 128, device=dev, dtype=torch.bfloat16)
k = torch.randn(T, HKV, 128, device=dev, dtype=torch.bfloat16)
v = torch.randn(T, HKV, 128, device=dev, dtype=torch.bfloat16)
pos = torch.arange(T, device=dev, dtype=torch.int32)
seq = torch.zeros(T, device=dev, dtype=torch.int32)
out = torch.empty(T, HQ, 128, device=dev, dtype=torch.float32)
lse = torch.empty(T, HQ, device=dev, dtype=torch.float32)
tr = torch.zeros(8 * 64 * 16, dtype=torch.int64, device=dev)
for i in range(2):
    lib.rcp_debug_set_trace(tr.data_ptr() if i == 1 else None)
    attend_into(q, (pos, seq), k, v, (pos, seq), HQ, HKV, 128 ** -0.5, out, lse, 0)
torch.cuda.synchronize()
t = tr.view(8, 64, 16).cpu().numpy()
names = ["PV0 issue", "PV1 issue", "S0 ready", "P0 done", "S1 ready", "P1 done", "K load", "V load"]
for cta in range(2):
    base = t[cta, 0, 6]
    print(f"CTA {cta}: cycles relative to first K load")
    print("it  " + " ".join(f"{n:>10s}" for n in names))
    for it in range(0, 64, 4):
        print(f"{it:3d} " + " ".join(f"{(x - base) if x else -1:10d}" for x in t[cta, it, :8]))
    it0, it1 = 16, 60
    per_it = (t[cta, it1, 0] - t[cta, it0, 0]) / (it1 - it0)
    sm0 = np.mean(t[cta, it0:it1, 3] - t[cta, it0:it1, 2])
    sm1 = np.mean(t[cta, it0:it1, 5] - t[cta, it0:it1, 4])
    wait0 = np.mean(t[cta, it0 + 1:it1 + 1, 2] - t[cta, it0:it1, 0])
    print(f"  cycles/iteration {per_it:.0f} (TC ideal 1024 per 64-key block); softmax0 {sm0:.0f}, softmax1 {sm1:.0f}; "
          f"PV0 issue -> next S0 ready {wait0:.0f}")

d = t[0, 16:60]
print("softmax0 phases (cycles): ld->s", np.mean(d[:, 8] - d[:, 2]), " max/m", np.mean(d[:, 9] - d[:, 8]),
      " exp loop", np.mean(d[:, 10] - d[:, 9]), " sum/rescale", np.mean(d[:, 11] - d[:, 10]),
      " st wait+fence", np.mean(d[:, 3] - d[:, 11]))
print("MMA loop (cycles): top->V ready", np.mean(d[1:, 12] - d[:-1, 14]), " V->PV0 issue (wait P0)", np.mean(d[:, 0] - d[:, 12]),
      " PV0 -> PV1 issue (S0 + wait P1)", np.mean(d[:, 1] - d[:, 0]), " PV1 -> commits done", np.mean(d[:, 13] - d[:, 1]),
      " S1 issue", np.mean(d[:, 14] - d[:, 13]))
