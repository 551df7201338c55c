"""pass-Q with the All2All fused into the attention stores (peer memory over
NVLink, RingAttention.fused_a2a) equals the NCCL All2All path bit for bit.

Two NCCL ranks (spawned here, one per GPU); skipped on boxes with fewer than
two GPUs.  Partial prefill on a cache from a full prefill, 405B-like GQA
(16 / 2 heads), D = 128, at three shapes (peer buffers allocated, re-slotted
for a smaller shape, re-allocated for a larger one), then RingAttention.close.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, errq):
    try:
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import paper_2411_01783_b200 as rc
        from paper_2411_01783_b200.kv_cache import RankKvCache
        from paper_2411_01783_b200.ring import RingAttention, TorchRingComm
        from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_full_prefill,
                                                    plan_partial_prefill)

        hq, hkv, D = 16, 2, 128
        cfg = rc.GqaConfig(hq, hkv, D)
        g = torch.Generator(device="cuda").manual_seed(3)
        rnd = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)
        ring = RingAttention(TorchRingComm())
        # (P, T): first shape allocates the peer buffers, the second is smaller
        # (re-slotted in place), the third larger (collective re-allocation)
        for P, T in ((3000, 700), (2000, 300), (3000, 1500)):
            hplan = plan_full_prefill([SequenceSpec(0, 0, P)], world)
            kh, vh = rnd(P, hkv, D), rnd(P, hkv, D)
            layout = [[hplan.new_token_count(0, r) for r in range(world)]]
            plan = plan_partial_prefill([SequenceSpec(0, P, T)], world, layout)
            qn, kn, vn = rnd(T, hq, D), rnd(T, hkv, D), rnd(T, hkv, D)
            outs = []
            for fused in (False, True, True):  # twice fused: buffer reuse across calls
                cache = RankKvCache(hkv, D, capacity_tokens=4096)
                kb = materialize_rank_block(hplan, rank, [kh])
                vb = materialize_rank_block(hplan, rank, [vh])
                loc = hplan.rank_local_indices(0, rank)
                sl = np.nonzero(loc >= 0)[0]
                cache.append_rows(0, kb.data[sl[0]:sl[-1] + 1], vb.data[sl[0]:sl[-1] + 1], loc[sl])
                ring.fused_a2a = fused
                part = ring.pass_q_prefill(plan, cache, materialize_rank_block(plan, rank, [qn]),
                                           materialize_rank_block(plan, rank, [kn]),
                                           materialize_rank_block(plan, rank, [vn]), cfg)
                torch.cuda.synchronize()
                outs.append((part.output.data.clone(), part.lse.clone()))
            for o, l in outs[1:]:
                assert torch.equal(o, outs[0][0]) and torch.equal(l, outs[0][1]), (P, T)
        ring.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_fused_a2a_equals_all2all():
    import torch.multiprocessing as mp

    from tests.test_ring_gloo import _free_port

    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
