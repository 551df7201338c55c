"""run_turns over NCCL, one rank per GPU (torchrun), against the dense replay.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/turns_nccl_check.py

Runs the tests/test_turns_gloo.py conversation at D = 128 with pass-KV, pass-Q
and adaptive (ring and all-gather decode), checks every rank's turn outputs
against the single-rank replay (|dO| <= 2e-2, |dLSE| <= 1e-3) and pass-KV ==
pass-Q bitwise, and prints one line per strategy from rank 0.
"""

import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests.test_turns_gloo import check_transcript, dense_replay, make_scenario  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, TorchRingComm
    from paper_2411_01783_b200.turns import run_turns

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    turns = make_scenario(hq, hkv, D, seed=5)
    want = dense_replay(turns, hkv)
    comm = TorchRingComm()
    res = {}
    for strategy, gather in (("pass_kv", False), ("pass_q", False), ("adaptive", True)):
        cache = RankKvCache(hkv, D, capacity_tokens=32)
        recs = run_turns(RingAttention(comm), cache, cfg, turns, strategy=strategy, gather_decode=gather)
        torch.cuda.synchronize()
        n = torch.tensor([check_transcript(recs, want, 2e-2, 1e-3)], device="cuda")
        dist.all_reduce(n)
        res[strategy] = recs
        if rank == 0:
            print(f"world {world} {strategy:8s} gather_decode={gather}: {int(n.item())} rows match the replay; "
                  f"prefill strategies {[r.strategy for r in recs if r.kind != 'decode']}", flush=True)
    for a, b in zip(res["pass_kv"], res["pass_q"]):
        if a.kind != "decode":
            assert torch.equal(a.output.output.data, b.output.output.data) and torch.equal(a.output.lse, b.output.lse)
    if rank == 0:
        print(f"world {world}: pass-KV == pass-Q bitwise on every prefill turn", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
