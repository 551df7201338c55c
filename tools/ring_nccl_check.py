"""Multi-GPU check of the SPMD ring engine over NCCL (launch with torchrun).

For each protocol the per-rank result of RingAttention (real NCCL transport,
one process per GPU) must be bitwise identical to the simulated-rank driver
(same kernels on one GPU) and within bf16 tolerance of the CPU oracle.
Prints one line per check on rank 0 and exits non-zero on failure.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_01783_b200 as rc  # noqa: E402
from oracle import ringcp_oracle as orc  # noqa: E402
from paper_2411_01783_b200.kv_cache import RankKvCache  # noqa: E402
from paper_2411_01783_b200.ring import (RingAttention, TorchRingComm, ring_pass_kv_prefill,  # noqa: E402
                                        ring_pass_q_prefill)
from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block,  # noqa: E402
                                            plan_full_prefill)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    hq, hkv = 8, 2
    cfg = rc.GqaConfig(hq, hkv, 128)
    rng = np.random.default_rng(7)
    lens = [1536, 700]
    seqs = [SequenceSpec(3 + i, 0, t) for i, t in enumerate(lens)]
    plan = plan_full_prefill(seqs, world)

    def bf(shape):
        return torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).to(torch.bfloat16)

    q = [bf((t, hq, 128)) for t in lens]
    k = [bf((t, hkv, 128)) for t in lens]
    v = [bf((t, hkv, 128)) for t in lens]
    dev = lambda xs: [x.cuda() for x in xs]
    qd, kd, vd = dev(q), dev(k), dev(v)
    ok = True
    for proto in ("pass_kv", "pass_q"):
        ring = RingAttention(TorchRingComm())
        cache = RankKvCache(hkv, 128, capacity_tokens=4096)
        qb = materialize_rank_block(plan, rank, qd)
        kb = materialize_rank_block(plan, rank, kd)
        vb = materialize_rank_block(plan, rank, vd)
        fn = ring.pass_kv_prefill if proto == "pass_kv" else ring.pass_q_prefill
        got = fn(plan, cache, qb, kb, vb, cfg)
        torch.cuda.synchronize()
        # simulated ranks on this GPU, same kernels
        caches = [RankKvCache(hkv, 128, capacity_tokens=4096) for _ in range(world)]
        qbs = [materialize_rank_block(plan, r, qd) for r in range(world)]
        kbs = [materialize_rank_block(plan, r, kd) for r in range(world)]
        vbs = [materialize_rank_block(plan, r, vd) for r in range(world)]
        sim = (ring_pass_kv_prefill if proto == "pass_kv" else ring_pass_q_prefill)(
            plan, caches, qbs, kbs, vbs, cfg)[rank]
        bitwise = torch.equal(got.output.data, sim.output.data) and torch.equal(got.lse, sim.lse)
        # oracle
        oc = [orc.Cache(hkv, 128) for _ in range(world)]
        _, want = orc.ring_prefill([orc.Seq(s.seq_id, 0, s.new_len) for s in seqs], [[0] * world] * len(seqs),
                                   world, oc, [x.float().numpy() for x in q], [x.float().numpy() for x in k],
                                   [x.float().numpy() for x in v], hkv)
        eo = float(np.abs(got.output.data.cpu().numpy() - want[rank][0]).max())
        fin = np.isfinite(want[rank][1])
        el = float(np.abs(got.lse.cpu().numpy()[fin] - want[rank][1][fin]).max())
        good = bitwise and eo <= 2e-2 and el <= 1e-3
        ok &= good
        t = torch.tensor([1 if good else 0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"{proto} world={world}: nccl==simulated bitwise {bitwise}, |dO| {eo:.2e}, |dLSE| {el:.2e}, "
                  f"all ranks ok {bool(t.item())}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
