"""Where a graphed p2p decode step's time goes, per rank (debug stamps).

  RCP_DECODE_STAMPS=1 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/decode_stamps.py [context] [B]

%globaltimer stamps after each phase of GraphedDecode._launches_p2p (stamp
launches add ~2 us each); prints per-rank medians over the timed steps of:
put (Q stores + epoch signal), Q wait, decode + routed combine, partials wait,
merge, and the whole step from stamp 0 to the next step's stamp 0."""
import os
import sys

import numpy as np
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
    from paper_2411_01783_b200.ring import TorchRingComm
    from paper_2411_01783_b200.sharding import SequenceSpec, plan_decode, plan_full_prefill

    context = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    hq, hkv, D = 128, 8, 128
    cfg = GqaConfig(hq, hkv, D)
    comm = TorchRingComm()
    hplan = plan_full_prefill([SequenceSpec(0, 0, context)], world)
    loc = hplan.rank_local_indices(0, rank)
    pos = loc[loc >= 0]
    cache = RankKvCache(hkv, D, capacity_tokens=B * (len(pos) + 128))
    g = torch.Generator(device="cuda").manual_seed(rank)
    for b in range(B):
        cache._reserve(b, len(pos) + 64)
        x = torch.randn(len(pos), hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
        cache.append_rows(b, x, x, pos)
    steps = 40
    gd = GraphedDecode(comm, cache, cfg, list(range(B)), max_steps=steps + 2,
                       first_positions={b: context for b in range(B)}, transport="p2p")
    for t in gd.input_buffers():
        t.normal_()
    for it in range(steps):
        own = plan_decode(list(range(B)), world, it).assignments[rank]
        gd.step(None, None, None, [context + it] * len(own))
    st = gd.stamps()[5:]  # drop warm-up / capture steps
    d = np.diff(st, axis=1) / 1e3
    step = np.diff(st[:, 0]) / 1e3
    names = ["put", "Q wait", "decode+combine", "partials wait", "merge"]
    line = " | ".join(f"{n} {np.median(d[:, i]):.1f}" for i, n in enumerate(names))
    out = [None] * world
    dist.all_gather_object(out, f"rank {rank}: {line} | step {np.median(step):.1f} us")
    if rank == 0:
        print("\n".join(out), flush=True)
    gd.close()
    cache.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
