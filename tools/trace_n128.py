"""Pipeline timeline of the 128-key attention kernel (v12) from the RCP_TRACE build
(tools/build_trace.sh).  One causal attention of T tokens (8B shape); for the
first traced CTAs prints per-block cycle deltas of the two tiles' S-ready /
P-done points, the softmax phases and the MMA issue points.

  RCP_ATTN_VERSION=12 python tools/trace_n128.py [T]
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
t = tr.view(8, 64, 16).cpu().numpy().astype(np.int64)
for cta in (range(3) if os.environ.get("RCP_ATTN_VERSION") != "13" else []):
    d = t[cta, 8:60]
    s0, p0, s1, p1 = d[:, 2], d[:, 3], d[:, 4], d[:, 5]
    print(f"CTA {cta}: cycles per 128-key block {np.mean(np.diff(s0)):.0f} (tensor ideal 2048 for 2 tiles)")
    print(f"  softmax (S ready -> P arrive): tile0 {np.mean(p0 - s0):.0f}, tile1 {np.mean(p1 - s1):.0f}")
    print(f"  tile0 phases: ld {np.mean(d[:, 8] - s0):.0f}, mask+max {np.mean(d[:, 9] - d[:, 8]):.0f}, "
          f"turn wait (v16) {np.mean(d[:, 11] - d[:, 9]):.0f}, exp+st {np.mean(d[:, 10] - d[:, 11]):.0f}, "
          f"sum+st wait+arrive {np.mean(p0 - d[:, 10]):.0f}")
    print(f"  P0 -> PV0 issued {np.mean(d[:, 0] - p0):.0f}; PV0 issued -> S0(+1) issued {np.mean(d[:, 12] - d[:, 0]):.0f}; "
          f"S0(+1) issued -> S0(+1) ready {np.mean(s0[1:] - d[:-1, 12]):.0f}")
    print(f"  P1 -> PV1 issued {np.mean(d[:, 1] - p1):.0f}; PV1 issued -> S1(+1) issued {np.mean(d[:, 13] - d[:, 1]):.0f}; "
          f"S1(+1) issued -> S1(+1) ready {np.mean(s1[1:] - d[:-1, 13]):.0f}")
    print(f"  offset S1 ready - S0 ready {np.mean(s1 - s0):.0f}; K load lead over PV0 {np.mean(d[:, 0] - d[:, 6]):.0f}")

if os.environ.get("RCP_ATTN_VERSION") == "13":
    # v13 events: 0 PV(it) issued, 1 S(it+3) issued (leader, index it); 2/4 S seen by
    # group 0/1, 3/5 P arrive of group 0/1, 8 max done, 9 handoff+rescale done,
    # 10 exps+st done (group 0) — group events indexed it >> 1
    for cta in (0, 2):
        d = t[cta]
        pv = d[8:56, 0]
        print(f"v13 pair {cta // 2}: cycles per 128-key block {np.mean(np.diff(pv)):.0f} (tensor ideal 1024 per SM)")
        for gg in (0, 1):
            s_seen, p_arr = d[4:28, 2 + 2 * gg], d[4:28, 3 + 2 * gg]
            print(f"  group {gg}: softmax (S seen -> P arrive) {np.mean(p_arr - s_seen):.0f}; "
                  f"P arrive -> next own S seen {np.mean(s_seen[1:] - p_arr[:-1]):.0f}")
        g0 = d[4:28]
        print(f"  group 0 phases: ld+max {np.mean(g0[:, 8] - g0[:, 2]):.0f}, exps {np.mean(g0[:, 9] - g0[:, 8]):.0f}, "
              f"handoff wait {np.mean(g0[:, 10] - g0[:, 9]):.0f}, fixups+tail {np.mean(g0[:, 3] - g0[:, 10]):.0f}")
        its = np.arange(8, 56, 2)
        print(f"  leader: P0(it) arrive -> PV(it) issued {np.mean(d[its, 0] - d[its // 2, 3]):.0f}")

if os.environ.get("RCP_ATTN_VERSION") == "14":
    # v14 events (per block it): 0 PV issued, 1 S(it+3) issued (leader); 2/4 S seen by group 0/1,
    # 9 exps done (group 0), 3/5 P arrive of group 0/1
    for cta in (0, 2):
        d = t[cta, 8:60]
        print(f"v14 pair {cta // 2}: cycles per 128-key block {np.mean(np.diff(d[:, 0])):.0f} (tensor ideal 1024 per SM)")
        print(f"  group 0: S seen -> exps done {np.mean(d[:, 9] - d[:, 2]):.0f}, exps done -> P arrive "
              f"{np.mean(d[:, 3] - d[:, 9]):.0f}, P arrive -> next S seen {np.mean(d[1:, 2] - d[:-1, 3]):.0f}")
        print(f"  group 1: S seen -> P arrive {np.mean(d[:, 5] - d[:, 4]):.0f}; leader P -> PV issued "
              f"{np.mean(d[:, 0] - np.maximum(d[:, 3], d[:, 5])):.0f}")
