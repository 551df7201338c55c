"""GraphedDecode(transport="p2p") — the decode step's Q all-gather and
partial All2All as kernel stores into CUDA-IPC peer buffers with device-side
epoch flags — equals the NCCL transport and the eager ring decode bit for bit.

Two NCCL ranks (spawned here, one per GPU); skipped on boxes with fewer than
two GPUs.  bf16 and e4m3 caches, 405B-like GQA (16 / 2 heads), 8 graphed
steps each, then close() on both ranks."""

import os

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
        from paper_2411_01783_b200.decode_graph import GraphedDecode
        from paper_2411_01783_b200.kv_cache import RankKvCache
        from paper_2411_01783_b200.ring import RingAttention, TorchRingComm
        from paper_2411_01783_b200.sharding import SequenceSpec, plan_decode, plan_full_prefill

        hq, hkv, D, ctx = 16, 2, 128, 3000
        cfg = rc.GqaConfig(hq, hkv, D)
        comm = TorchRingComm()
        batch = [0, 1, 2]
        hplan = plan_full_prefill([SequenceSpec(0, 0, ctx)], world)
        loc = hplan.rank_local_indices(0, rank)
        pos = loc[loc >= 0]
        for kv in ("bf16", "e4m3"):
            g = torch.Generator(device="cuda").manual_seed(100 + rank)
            caches = [RankKvCache(hkv, D, capacity_tokens=8192, kv_dtype=kv) for _ in range(3)]
            for b in batch:
                k = torch.randn(len(pos), hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
                v = torch.randn(len(pos), hkv, D, device="cuda", dtype=torch.bfloat16, generator=g)
                for c in caches:
                    c._reserve(b, len(pos) + 32)
                    c.append_rows(b, k, v, pos)
            steps = 8
            gds = [GraphedDecode(comm, caches[i], cfg, batch, max_steps=steps + 2,
                                 first_positions={b: ctx for b in batch}, transport=t)
                   for i, t in ((1, "nccl"), (2, "p2p"))]
            ring = RingAttention(comm)
            gq = torch.Generator(device="cuda").manual_seed(7)  # same tokens on every rank
            for it in range(steps):
                own = plan_decode(batch, world, it).assignments[rank]
                idx = [b for _s, b in own]
                q = torch.randn(len(batch), hq, D, device="cuda", dtype=torch.bfloat16, generator=gq)
                k = torch.randn(len(batch), hkv, D, device="cuda", dtype=torch.bfloat16, generator=gq)
                v = torch.randn(len(batch), hkv, D, device="cuda", dtype=torch.bfloat16, generator=gq)
                p = [ctx + it] * len(own)
                o0, l0 = ring.pass_q_decode(plan_decode(batch, world, it), caches[0], q[idx], k[idx], v[idx], p, cfg,
                                            gather=True)
                res = [gd.step(q[idx], k[idx], v[idx], p) for gd in gds]
                torch.cuda.synchronize()
                m = len(own)
                for o, l in res:
                    assert torch.equal(o, o0[:m]) and torch.equal(l, l0[:m]), (kv, it)
            for gd in gds:
                gd.check_transport()
                gd.close()
            for c in caches:
                c.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_p2p_decode_transport_equals_nccl():
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
