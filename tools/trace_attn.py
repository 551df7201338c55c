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

_lib.LIB_PATH = os.path.join(ROOT, "paper_2411_01783_b200", os.environ.get("RCP_TRACE_LIB", "_ringcp_b200_trace.so"))
lib = _lib.load()
lib.rcp_debug_set_trace.argtypes = [ctypes.c_void_p]

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

VER = os.environ.get("RCP_ATTN_VERSION", "6")
if VER == "6":
    for cta in (0, 1):
        d = t[cta, 8:56]
        print(f"v6 CTA {cta}: cycles/block {np.mean(np.diff(d[:, 2])):.0f} (TC ideal 2048 per 128-key block, 2 tiles); "
              f"softmax0 {np.mean(d[:, 3] - d[:, 2]):.0f}, softmax1 {np.mean(d[:, 5] - d[:, 4]):.0f}")
        print(f"   softmax0 phases: ld {np.mean(d[:, 8] - d[:, 2]):.0f}, mask+max {np.mean(d[:, 9] - d[:, 8]):.0f}, "
              f"exp+st {np.mean(d[:, 10] - d[:, 9]):.0f}, sum/rescale {np.mean(d[:, 11] - d[:, 10]):.0f}, "
              f"st wait+arrive {np.mean(d[:, 3] - d[:, 11]):.0f}")
        print(f"   P0(it) -> S0(it+1) ready {np.mean(d[1:, 2] - d[:-1, 3]):.0f}; P1(it) -> S1(it+1) ready "
              f"{np.mean(d[1:, 4] - d[:-1, 5]):.0f}; P0 done -> PV0 issued {np.mean(d[:, 0] - d[:, 3]):.0f}; "
              f"P1 done -> PV1 issued {np.mean(d[:, 1] - d[:, 5]):.0f}")
        print(f"   MMA: top->V ready {np.mean(d[1:, 12] - d[:-1, 14]):.0f}, V->PV0 (wait P0) {np.mean(d[:, 0] - d[:, 12]):.0f}, "
              f"PV0->PV1 (S0 + wait P1) {np.mean(d[:, 1] - d[:, 0]):.0f}, PV1->commits {np.mean(d[:, 13] - d[:, 1]):.0f}, "
              f"S1 issue {np.mean(d[1:, 14] - d[1:, 13]):.0f}; loads lead {np.mean(d[:, 0] - d[:, 7]):.0f}")
    sys.exit(0)
if VER == "8":
    for cta in (0, 1):
        d = t[cta]
        for x in (0, 1):
            its = np.arange(8 + x, 56, 2)
            s_seen, p_done = d[its, 2 + 2 * x], d[its, 3 + 2 * x]
            print(f"v8 CTA {cta} group {x}: cycles per own block {np.mean(np.diff(s_seen)):.0f} "
                  f"(2 blocks of the pair per period; TC ideal 2 x 1024); softmax {np.mean(p_done - s_seen):.0f}; "
                  f"P done -> next own S seen {np.mean(s_seen[1:] - p_done[:-1]):.0f}")
        if cta == 0:
            its = np.arange(8, 56)
            print(f"   leader: P(it) wait done -> PV issued {np.mean(d[its, 1] - d[its, 0]):.0f} (PV+S issue incl. K wait)")
    sys.exit(0)
if os.environ.get("RCP_TRACE_PERWARP"):
    for cta in (0, 1):
        d = t[cta, 8:56]
        base = d[:, 8]
        print(f"CTA {cta}: P-arrive of softmax warps 4..11 relative to warp 4 (mean over blocks):",
              " ".join(f"w{4 + w}:{np.mean(d[:, 8 + w] - base):+.0f}" for w in range(8)))
    sys.exit(0)
if VER == "5":
    for cta in (0, 1):
        d = t[cta, 8:56]
        rk = cta & 1
        s_rdy, p_done = d[:, 2 + 2 * rk], d[:, 3 + 2 * rk]
        print(f"v5 CTA {cta}: cycles/block {np.mean(np.diff(s_rdy)):.0f} (TC ideal 1024 per 128-key block); "
              f"softmax {np.mean(p_done - s_rdy):.0f}; S ready -> next S ready waits {np.mean(s_rdy[1:] - p_done[:-1]):.0f}")
        print(f"   softmax: S ready -> max exchanged {np.mean(d[:, 12 + rk] - s_rdy):.0f}")
        if rk == 0:
            print(f"   softmax: P done -> arrive issued {np.mean(d[:, 15] - p_done):.0f}; arrive -> next S seen "
                  f"{np.mean(s_rdy[1:] - d[:-1, 15]):.0f}")
        if rk == 0:
            print(f"   MMA latency (observer warp): S(it) issue end -> S done {np.mean(d[2:, 11] - d[:-2, 10]):.0f}; "
                  f"PV(it) issue end -> PV done {np.mean(d[:-1, 14] - d[:-1, 8]):.0f}; "
                  f"S done -> softmax sees it {np.mean(s_rdy - d[:, 11]):.0f}")
        if rk == 0:
            print(f"   leader MMA: P->PV issue {np.mean(d[:, 0] - p_done):.0f}, PV issue {np.mean(d[:, 8] - d[:, 0]):.0f}, "
                  f"commits+wait K {np.mean(d[:, 9] - d[:, 8]):.0f}, S issue {np.mean(d[:, 10] - d[:, 9]):.0f}, "
                  f"loop top->P wait done {np.mean(d[1:, 0] - d[:-1, 1]):.0f}, loads lead {np.mean(d[:, 0] - d[:, 7]):.0f}")
            print(f"   S(it) issued (end of iter it-2) -> S(it) ready at softmax: {np.mean(d[2:, 2] - d[:-2, 10]):.0f}; "
                  f"PV(it-1) issue -> S(it+1) issued: {np.mean(d[1:, 10] - d[:-1, 0]):.0f}")
    sys.exit(0)
d = t[0, 16:60]
print("softmax0 phases (cycles): ld->s", np.mean(d[:, 8] - d[:, 2]), " max/m", np.mean(d[:, 9] - d[:, 8]),
      " exp loop", np.mean(d[:, 10] - d[:, 9]), " sum/rescale", np.mean(d[:, 11] - d[:, 10]),
      " st wait+fence", np.mean(d[:, 3] - d[:, 11]))
print("MMA loop (cycles): top->V ready", np.mean(d[1:, 12] - d[:-1, 14]), " V->PV0 issue (wait P0)", np.mean(d[:, 0] - d[:, 12]),
      " PV0 -> PV1 issue (S0 + wait P1)", np.mean(d[:, 1] - d[:, 0]), " PV1 -> commits done", np.mean(d[:, 13] - d[:, 1]),
      " S1 issue", np.mean(d[:, 14] - d[:, 13]))
