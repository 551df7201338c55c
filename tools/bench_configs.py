"""Benchmarks for BASELINE configs #4 and #5 (launch with torchrun, one rank per GPU).

  partial  cfg4: partial prefill on a persistent KV cache, P + T = 131072,
           KV-cache miss rate sweep; times ring pass-KV and ring pass-Q for the
           same turn and reports what the Alg. 1 heuristic (B200 profile) picks.
  decode   cfg5: ring pass-Q batched decode, B sequences of `--context` cached
           tokens sharded over the ranks (balanced prefill layout); times one
           decode step (append + Q ring + split-KV attention + All2All + merge).

Each measurement: warm-up, then per-step CUDA events on the compute stream,
median over steps, max over ranks.  Prints one JSON line per point on rank 0.
"""

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from paper_2411_01783_b200 import perf_model as pm  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import RingAttention, TorchRingComm, _LocalComm  # noqa: E402
from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_decode,  # noqa: E402
                                            plan_full_prefill, plan_partial_prefill)

D = 128


def setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world


def max_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def timed(fn, reset, steps, warmup, world):
    for _ in range(warmup):
        reset()
        fn()
    ts = []
    for _ in range(steps):
        reset()
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(max_over_ranks(s.elapsed_time(e), world))
    return statistics.median(ts)


def randn(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)


def run_partial(args, rank, world):
    hq, hkv = args.hq, args.hkv
    cfg = rc.GqaConfig(hq, hkv, D)
    total = args.context
    comm = TorchRingComm() if world > 1 else _LocalComm(0, 1)
    ring = RingAttention(comm)
    model = dict(n_query_heads=hq, n_kv_heads=hkv, head_dim=D)
    m = pm.b200_profile(model, n_ranks=world)
    calib = None
    if args.calibrate:  # the heuristic's constants measured in this run (perf_model.calibrate_b200)
        m, calib = pm.calibrate_b200(comm if world > 1 else _LocalComm(0, 1), model, n_ranks=world)
        if rank == 0:
            print(json.dumps({"calibration": calib}), flush=True)
    quantum = 2 * world * 128
    for miss in args.miss:
        T = max(quantum, int(round(miss * total / quantum)) * quantum)
        P = total - T
        # history: a balanced prefill of P tokens placed the cache (rank r holds chunks r, 2N-1-r)
        cache = RankKvCache(hkv, D, capacity_tokens=(P + T) // world + 8192)
        layout = [[0] * world]
        if P > 0:
            hplan = plan_full_prefill([SequenceSpec(0, 0, P)], world)
            kh = materialize_rank_block(hplan, rank, [randn((P, hkv, D), 21)])
            vh = materialize_rank_block(hplan, rank, [randn((P, hkv, D), 22)])
            loc = hplan.rank_local_indices(0, rank)
            sl = np.nonzero(loc >= 0)[0]
            cache.append_rows(0, kh.data[sl[0]:sl[-1] + 1], vh.data[sl[0]:sl[-1] + 1], loc[sl])
            layout = [[hplan.new_token_count(0, r) for r in range(world)]]
        plan = plan_partial_prefill([SequenceSpec(0, P, T)], world, layout)
        qn, kn, vn = randn((T, hq, D), 31), randn((T, hkv, D), 32), randn((T, hkv, D), 33)
        qb = materialize_rank_block(plan, rank, [qn])
        kb = materialize_rank_block(plan, rank, [kn])
        vb = materialize_rank_block(plan, rank, [vn])
        base_len = cache.cached_len(0)
        reset = lambda: cache.truncate(0, base_len)
        res = {}
        for proto in ("pass_kv", "pass_q"):
            fn = (lambda: ring.pass_kv_prefill(plan, cache, qb, kb, vb, cfg)) if proto == "pass_kv" else \
                 (lambda: ring.pass_q_prefill(plan, cache, qb, kb, vb, cfg))
            res[proto] = timed(fn, reset, args.steps, args.warmup, world)
        fused = None
        if args.fused and world > 1:
            # pass-Q with the partials written straight into the owners' peer
            # slots (no All2All): must equal the All2All version bit for bit
            reset()
            ref = ring.pass_q_prefill(plan, cache, qb, kb, vb, cfg)
            ring.fused_a2a = True
            reset()
            got = ring.pass_q_prefill(plan, cache, qb, kb, vb, cfg)
            torch.cuda.synchronize()
            same = torch.tensor([int(torch.equal(ref.output.data, got.output.data) and torch.equal(ref.lse, got.lse))],
                                device="cuda")
            dist.all_reduce(same, op=dist.ReduceOp.MIN)
            assert int(same.item()) == 1, "fused pass-Q differs from the All2All version"
            fused = timed(lambda: ring.pass_q_prefill(plan, cache, qb, kb, vb, cfg), reset, args.steps,
                          args.warmup, world)
            ring.fused_a2a = False
        shape = pm.PrefillShape(T, P)
        pick = pm.choose_strategy(shape, m)
        pick_ref = pm.choose_strategy(shape, m, refined=True)
        flops = 4.0 * D * hq * (T * P + T * (T + 1) / 2)
        if rank == 0:
            best = min(res, key=res.get)
            print(json.dumps({
                "config": "cfg4-partial-prefill", "cp": world, "n_q_heads": hq, "n_kv_heads": hkv,
                "P": P, "T": T, "miss": T / total, "pass_kv_ms": res["pass_kv"], "pass_q_ms": res["pass_q"],
                "pass_q_fused_a2a_ms": fused,
                "winner": best, "heuristic": pick, "heuristic_refined": pick_ref,
                "tflops_per_gpu_best": flops / (res[best] * 1e-3) / 1e12 / world}), flush=True)
        del cache


def run_decode(args, rank, world):
    hq, hkv = args.hq, args.hkv
    cfg = rc.GqaConfig(hq, hkv, D)
    comm = TorchRingComm() if world > 1 else _LocalComm(0, 1)
    ring = RingAttention(comm)
    local = args.context // world
    for B in args.batch:
        cache = RankKvCache(hkv, D, capacity_tokens=B * (local + 128), kv_dtype=args.kv_dtype)
        batch = list(range(B))
        hplan = plan_full_prefill([SequenceSpec(0, 0, args.context)], world)
        loc = hplan.rank_local_indices(0, rank)
        pos = loc[loc >= 0]
        for b in batch:  # each sequence: its balanced shard of the history (random data)
            cache._reserve(b, local + 128)  # room for the decode steps: no segment moves later
            cache.append_rows(b, randn((local, hkv, D), 100 + b), randn((local, hkv, D), 200 + b), pos)
        lens = {b: cache.cached_len(b) for b in batch}
        dp = plan_decode(batch, world, 0)
        mine = dp.assignments[rank]
        n_mine = max(len(mine), 1)
        qt, kt, vt = randn((n_mine, hq, D), 7), randn((n_mine, hkv, D), 8), randn((n_mine, hkv, D), 9)
        positions = [args.context] * len(mine)

        def reset():
            for b in batch:
                cache.truncate(b, lens[b])

        def step():
            return ring.pass_q_decode(dp, cache, qt[: len(mine)], kt[: len(mine)], vt[: len(mine)], positions, cfg,
                                      gather=args.gather)

        if args.graph:
            # CUDA-graph replay of the step (decode_graph.GraphedDecode): one
            # capture, then every timed step is a replay; the cache keeps
            # growing by one token per sequence per step, as in serving.
            from paper_2411_01783_b200.decode_graph import GraphedDecode

            pos0 = {b: max(lens[b], args.context) for b in batch}
            # consecutive positions per step: the step metadata is precomputed on the
            # device and selected by the graph (no per-step upload / host metadata)
            gd = GraphedDecode(comm, cache, cfg, batch, max_steps=args.warmup + 2 * args.steps + 4,
                               first_positions=None if args.no_table else pos0, grouped_a2a=not args.separate_a2a,
                               transport=args.transport)

            if args.inplace:  # the model writes its new tokens into the graph's input buffers
                for dst, src in zip(gd.input_buffers(), (qt, kt, vt)):
                    m0 = min(dst.shape[0], src.shape[0])
                    dst[:m0].copy_(src[:m0])

            def step():  # noqa: F811 - graphed variant
                it = gd.it
                own = plan_decode(batch, world, it).assignments[rank]
                p = [pos0[sid] + it for sid, _b in own]
                if args.inplace:
                    return gd.step(None, None, None, p)
                return gd.step(qt[: len(own)], kt[: len(own)], vt[: len(own)], p)

            reset = lambda: None  # noqa: E731 - appends are part of the measured step
        ms = timed(step, reset, args.steps, args.warmup, world)
        b2b = None
        if args.graph:
            # back to back: the host issues step i+1 while the GPU runs step i
            # (a serving loop); per-step time = max(host issue, GPU time)
            barrier(world)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            nb = max(1, min(args.steps, gd.steps_left - 1))
            for _ in range(nb):
                step()
            e.record()
            torch.cuda.synchronize()
            b2b = max_over_ranks(s.elapsed_time(e) / nb, world)
        elem = 1 if args.kv_dtype == "e4m3" else 2
        kv_bytes = B * local * hkv * D * 2 * elem  # this rank's K+V read per decode step
        if rank == 0:
            print(json.dumps({
                "config": "cfg5-ring-pass-q-decode", "cp": world, "batch": B, "context": args.context,
                "q_transport": "allgather" if (args.gather or args.graph) else "ring",
                "cuda_graph": bool(args.graph), "device_step_table": bool(args.graph and not args.no_table),
                "transport": args.transport if (args.graph and world > 1) else None,
                "inputs": "in place" if (args.graph and args.inplace) else "copied per step",
                "n_q_heads": hq, "n_kv_heads": hkv, "kv_dtype": args.kv_dtype, "step_ms": ms, "step_ms_back_to_back": b2b,
                "kv_bytes_per_rank": kv_bytes, "hbm_gbs_effective": kv_bytes / (ms * 1e-3) / 1e9}), flush=True)
        if args.graph:
            gd.check_transport()
            gd.close()
        del cache
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["partial", "decode"])
    ap.add_argument("--hq", type=int, default=128)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--miss", type=float, nargs="*", default=[0.01, 0.025, 0.05, 0.10, 0.125, 0.2, 0.5, 1.0])
    ap.add_argument("--batch", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--gather", action="store_true", help="decode: all-gather Q instead of the Q ring")
    ap.add_argument("--graph", action="store_true", help="decode: replay the step from a CUDA graph")
    ap.add_argument("--separate-a2a", action="store_true",
                    help="decode --graph: two All2All collectives instead of one grouped send/recv set")
    ap.add_argument("--no-table", action="store_true",
                    help="decode --graph: upload the step metadata each step instead of the device table")
    ap.add_argument("--calibrate", action="store_true",
                    help="partial: feed Alg. 1 the attention / link / All2All constants measured in this run")
    ap.add_argument("--fused", action="store_true",
                    help="partial: also time pass-Q with peer-memory partials (no All2All), checked bitwise")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="decode --graph at N > 1: NCCL collectives or kernel stores into CUDA-IPC peer buffers")
    ap.add_argument("--inplace", action="store_true",
                    help="decode --graph: inputs written once into GraphedDecode.input_buffers() (no per-step copies)")
    ap.add_argument("--kv-dtype", choices=["bf16", "e4m3"], default="bf16",
                    help="decode: KV-cache storage (e4m3 = FP8 KV, per-head scales calibrated at prefill)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    rank, world = setup()
    try:
        (run_partial if args.mode == "partial" else run_decode)(args, rank, world)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
