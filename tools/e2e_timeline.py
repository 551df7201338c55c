"""Timeline of one host-buffer prefill step (RingAttention.pass_kv_prefill_host).

Prints, relative to the step start (CUDA events): K/V resident, each query
range resident, each range's final attention launch done, and the end of the
step (device->host copies included); plus the device-only time of the same
attention with the query ranges split (no copies) and unsplit.

  python tools/e2e_timeline.py [T] [n_sub]
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import RingAttention, _LocalComm  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
n_sub = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hq, hkv, D = 32, 8, 128
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

marks = []
orig_pass_kv = ring.pass_kv


def pass_kv_marked(*a, **kw):
    user = kw.get("on_final")

    def on_final(i):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((f"range {i} final launch done", e))
        user(i)

    kw["on_final"] = on_final
    for i, ev in enumerate(kw.get("q_ready") or []):
        e = torch.cuda.Event(enable_timing=True)
        torch.cuda.current_stream().wait_event(ev)
        e.record()
        marks.append((f"range {i} Q resident (compute stream)", e))
    return orig_pass_kv(*a, **kw)


for ns in (2, 4, 8, 16):  # plain step time per range count (no instrumentation)
    ts = []
    for it in range(4):
        cache.reset()
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        ring.pass_kv_prefill_host(plan, cache, [host["q"]], [host["k"]], [host["v"]], cfg, out_h, lse_h, n_sub=ns)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print(f"n_sub {ns:2d}: step {min(ts[1:]):.2f} ms")

ring.pass_kv = pass_kv_marked
for it in range(3):
    marks.clear()
    cache.reset()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    s.record()
    ring.pass_kv_prefill_host(plan, cache, [host["q"]], [host["k"]], [host["v"]], cfg, out_h, lse_h, n_sub=n_sub)
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    torch.cuda.synchronize()
if True:
    for name, ev in marks:
        print(f"{s.elapsed_time(ev):8.2f} ms  {name}")
    print(f"{s.elapsed_time(e):8.2f} ms  step end (D2H included)")

ring.pass_kv = orig_pass_kv
for splits_n in (1, n_sub):
    ts = []
    for it in range(3):
        cache.reset()
        qb = materialize_rank_block(plan, 0, [dev["q"]])
        kb = materialize_rank_block(plan, 0, [dev["k"]])
        vb = materialize_rank_block(plan, 0, [dev["v"]])
        from paper_2411_01783_b200.ring import KvLayout, append_new_tokens, build_kv_message, kv_message_len

        append_new_tokens(plan, 0, cache, kb, vb)
        lay = KvLayout(kv_message_len(plan), hkv, D)
        msg = torch.empty(lay.nbytes, dtype=torch.uint8, device="cuda")
        build_kv_message(plan, cache, msg)
        qp, qs = qb.meta32("q")
        out = torch.empty((S, hq, D), dtype=torch.float32, device="cuda")
        lse = torch.empty((S, hq), dtype=torch.float32, device="cuda")
        step = max(256, -(-S // splits_n) // 256 * 256)
        splits = [(a, min(S, a + step)) for a in range(0, S, step)]
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        ring.pass_kv(qb.data, qp, qs, lay, msg, cfg, out, lse, q_splits=splits)
        s1.record()
        torch.cuda.synchronize()
        ts.append(s0.elapsed_time(s1))
    print(f"device-only attention, {len(splits)} launch(es): {min(ts):.2f} ms")
