"""GraphedDecode vs eager ring pass-Q decode over NCCL (torchrun, one rank per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/decode_graph_check.py

Two identical per-rank caches (each sequence's balanced shard of a random
history); per step the eager all-gather decode and the graph replay get the
same tokens, and their outputs must agree (they differ only in split-KV
boundaries).  Then both are timed (CUDA events, median, max over ranks).
"""

import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.decode_graph import GraphedDecode
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, TorchRingComm
    from paper_2411_01783_b200.sharding import SequenceSpec, plan_decode, plan_full_prefill

    hq, hkv, D = 128, 8, 128
    context = int(os.environ.get("CTX", "65536"))
    cfg = GqaConfig(hq, hkv, D)
    comm = TorchRingComm()
    res = []
    for B in (1, 4, 8):
        batch = list(range(B))
        hplan = plan_full_prefill([SequenceSpec(0, 0, context)], world)
        loc = hplan.rank_local_indices(0, rank)
        pos = loc[loc >= 0]
        local_len = len(pos)
        # GD_KV=e4m3: FP8 KV caches (scales calibrated by the identical first appends)
        caches = [RankKvCache(hkv, D, capacity_tokens=B * (local_len + 128), kv_dtype=os.environ.get("GD_KV", "bf16"))
                  for _ in range(2)]
        g = torch.Generator(device="cuda").manual_seed(100 + rank)
        for b in batch:
            k = torch.randn(local_len, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
            v = torch.randn(local_len, hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
            for c in caches:
                c._reserve(b, local_len + 64)
                c.append_rows(b, k, v, pos)
        ring = RingAttention(comm)
        steps, warm = 12, 3
        # GD_TABLE=1: device-resident step table; GD_GROUPED=1: one grouped All2All
        table = os.environ.get("GD_TABLE") == "1"
        gd = GraphedDecode(comm, caches[1], cfg, batch, max_steps=2 * (steps + warm) + 4,
                           first_positions={b: context for b in batch} if table else None,
                           grouped_a2a=os.environ.get("GD_GROUPED") == "1",
                           transport=os.environ.get("GD_TRANSPORT", "nccl"))
        gq = torch.Generator(device="cuda").manual_seed(7)  # same tokens on every rank
        max_err = 0.0
        t_e, t_g = [], []
        for it in range(steps + warm):
            own = plan_decode(batch, world, it).assignments[rank]
            q = torch.randn(B, hq, D, device="cuda", dtype=torch.bfloat16, generator=gq)
            k = torch.randn(B, hkv, D, device="cuda", dtype=torch.bfloat16, generator=gq)
            v = torch.randn(B, hkv, D, device="cuda", dtype=torch.bfloat16, generator=gq)
            idx = [b for _s, b in own]
            p = [context + it] * len(own)
            times = []
            for mode in ("eager", "graph"):
                dist.barrier()
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                if mode == "eager":
                    o1, l1 = ring.pass_q_decode(plan_decode(batch, world, it), caches[0], q[idx], k[idx], v[idx], p,
                                                cfg, gather=True)
                else:
                    o2, l2 = gd.step(q[idx], k[idx], v[idx], p)
                e.record()
                torch.cuda.synchronize()
                times.append(s.elapsed_time(e))
            if own:
                max_err = max(max_err, float((o1[: len(own)] - o2).abs().max()), float((l1[: len(own)] - l2).abs().max()))
            if it >= warm:
                t_e.append(times[0])
                t_g.append(times[1])
        stats = torch.tensor([max_err, statistics.median(t_e), statistics.median(t_g)], device="cuda")
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"world {world} B {B} ctx {context} kv={os.environ.get('GD_KV', 'bf16')} transport={os.environ.get('GD_TRANSPORT', 'nccl')} table={os.environ.get('GD_TABLE')} "
                  f"grouped={os.environ.get('GD_GROUPED')}: max |eager - graph| {stats[0].item():.2e}; step eager "
                  f"{stats[1].item():.3f} ms, graph {stats[2].item():.3f} ms", flush=True)
        res.append(stats[0].item())
        gd.check_transport()
        gd.close()
        del caches, gd
        torch.cuda.empty_cache()
    assert max(res) < 1e-3, res
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
