"""The bench's e2e serving loop at several query-range counts (one GPU).

Runs K requests of the 8B-shape 128K CP1 prefill through
RingAttention.pass_kv_prefill_host from pinned host buffers, each request
staged one ahead (as bench.py does), for n_sub in a list, and prints ms per
request next to the device-input step time — how much of the e2e overhead is
split-launch tails versus copies.

  python tools/e2e_loop_ranges.py [K] [n_sub ...]
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import RingAttention, _LocalComm  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
SUBS = [int(x) for x in sys.argv[2:]] or [16, 8, 4, 2, 1]
T, hq, hkv, D = 131072, 32, 8, 128
cfg = rc.GqaConfig(hq, hkv, D)
plan = plan_full_prefill([SequenceSpec(0, 0, T)], 1)
g = torch.Generator(device="cuda").manual_seed(0)
dev = {n: torch.randn(T, h, D, device="cuda", dtype=torch.bfloat16, generator=g) for n, h in
       (("q", hq), ("k", hkv), ("v", hkv))}
host = {n: t.cpu().pin_memory() for n, t in dev.items()}
S = plan.total_query_slots()
out_h = torch.empty((S, hq, D), dtype=torch.float32).pin_memory()
lse_h = torch.empty((S, hq), dtype=torch.float32).pin_memory()
cache = RankKvCache(hkv, D, capacity_tokens=S + 4096)
ring = RingAttention(_LocalComm(0, 1))
flops = 4.0 * D * hq * T * (T + 1) / 2


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def device_steps(n):
    blocks = [materialize_rank_block(plan, 0, [dev[x]]) for x in ("q", "k", "v")]
    for _ in range(n):
        cache.reset()
        ring.pass_kv_prefill(plan, cache, *blocks, cfg)


def loop(n, n_sub):
    def stage():
        return ring.stage_host_inputs(plan, [host["q"]], [host["k"]], [host["v"]], cfg, "cuda", n_sub=n_sub)

    st = stage()
    for i in range(n):
        cache.reset()
        ring.pass_kv_prefill_host(plan, cache, [host["q"]], [host["k"]], [host["v"]], cfg, out_h, lse_h,
                                  staged=st, join=False)
        st = stage() if i + 1 < n else None
    ring.join_host_copies()


launch_ev = []
if os.environ.get("TIMELINE") == "2":  # time every attention launch
    _attend = ring.attend

    def _timed_attend(*a, **kw):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _attend(*a, **kw)
        e1.record()
        launch_ev.append((e0, e1))

    ring.attend = _timed_attend


def timeline(n, n_sub):
    """Per request: compute window (events on the compute stream around the
    call) and when its D2H finished, relative to the loop start (ms)."""
    cur = torch.cuda.current_stream()
    s_out = ring._side_stream("d2h")
    launch_ev.clear()
    t0 = torch.cuda.Event(enable_timing=True)
    ev = []
    host_t = []
    landed = []
    torch.cuda.synchronize()
    t0.record()
    h0 = time.perf_counter()

    def stage():
        return ring.stage_host_inputs(plan, [host["q"]], [host["k"]], [host["v"]], cfg, "cuda", n_sub=n_sub)

    jit = os.environ.get("STAGE_JIT")  # stage each request just before its compute
    st = stage()
    for i in range(n):
        cache.reset()
        if jit and i > 0:
            st = stage()
        a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        landed.append((st.kv_ready, st.q_ready[0], st.q_ready[-1]))
        a.record(cur)
        ring.pass_kv_prefill_host(plan, cache, [host["q"]], [host["k"]], [host["v"]], cfg, out_h, lse_h,
                                  staged=st, join=False)
        b.record(cur)
        c.record(s_out)
        ev.append((a, b, c))
        h1 = time.perf_counter()
        if not jit:
            st = stage() if i + 1 < n else None
        host_t.append(f"{1e3 * (h1 - h0):.0f}/{1e3 * (time.perf_counter() - h0):.0f}")
    ring.join_host_copies()
    torch.cuda.synchronize()
    rows = [f"{t0.elapsed_time(a):.0f}-{t0.elapsed_time(b):.0f} (d2h {t0.elapsed_time(c):.0f})" for a, b, c in ev]
    print(f"  n_sub {n_sub}: compute windows " + ", ".join(rows), flush=True)
    if launch_ev:
        L = len(launch_ev) // n
        for r in range(n):
            le = launch_ev[r * L:(r + 1) * L]
            busy = sum(a.elapsed_time(b) for a, b in le)
            wa, wb, _ = ev[r]
            print(f"    request {r}: first launch +{wa.elapsed_time(le[0][0]):.1f} ms after window start, "
                  f"launches {busy:.1f} ms busy, gaps {sum(le[i][1].elapsed_time(le[i + 1][0]) for i in range(L - 1)):.1f} ms, "
                  f"last launch -> window end {le[-1][1].elapsed_time(wb):.1f} ms", flush=True)
        launch_ev.clear()
    print("    host: request issued / next staged at " + ", ".join(host_t) + " ms", flush=True)
    try:
        print("    inputs landed (K/V, first range, last range): " + ", ".join(
            f"{t0.elapsed_time(x):.0f}/{t0.elapsed_time(y):.0f}/{t0.elapsed_time(z):.0f}" for x, y, z in landed),
            flush=True)
    except RuntimeError as e:  # the first request was staged before t0
        print("    inputs landed: n/a", e)


device_steps(2)
ms_dev = timed(lambda: device_steps(K)) / K
print(f"device inputs: {ms_dev:.1f} ms/step ({flops / ms_dev / 1e9:.0f} TF/s)", flush=True)
for n_sub in SUBS:
    loop(2, n_sub)
    ms = timed(lambda: loop(K, n_sub)) / K
    print(f"host e2e, n_sub {n_sub:2d}: {ms:.1f} ms/step ({flops / ms / 1e9:.0f} TF/s)", flush=True)
    if os.environ.get("TIMELINE"):
        timeline(int(os.environ.get("TL_N", "5")), n_sub)
