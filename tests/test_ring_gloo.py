"""World-size-2 (and 3) gloo test of the SPMD ring engine on CPU.

The transport (torch.distributed P2P ring exchange, All2All as pairwise
exchanges), the message layouts, the step schedule and the merge order are the
product code (paper_2411_01783_b200.ring.RingAttention); only the per-step
compute is injected — oracle attention / merge / decode on CPU tensors — since
there is no GPU here.  Results must equal the composed CPU oracle (SPEC Alg.
2-4), and pass-KV must equal pass-Q bitwise.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ringcp_oracle as orc

PAD_Q, PAD_K, POS_PAD_K = -(2 ** 31), -(2 ** 31) + 1, 2 ** 31 - 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _blk(data, pos, seq, pad):
    data = data.float().numpy()
    pos = pos.numpy().astype(np.int64)
    seq = seq.numpy().astype(np.int64)
    valid = seq != pad
    return orc.Blk(data, np.where(valid, pos, -1), valid, np.where(valid, seq, -1))


def oracle_attend(q, q_pos, q_seq, k, v, k_pos, k_seq, cfg, out, lse, mode, ws=None):
    qb = _blk(q, q_pos, q_seq, PAD_Q)
    kb = _blk(k, k_pos, k_seq, PAD_K)
    vb = _blk(v, k_pos, k_seq, PAD_K)
    o, l = orc.gqa(qb, kb, vb, cfg.n_kv_heads, cfg.scale)
    # round the partial to fp32 exactly where the kernels do (pass-Q stores it)
    o, l = o.astype(np.float32).astype(np.float64), l.astype(np.float32).astype(np.float64)
    if mode == 1:
        o, l = orc.merge_pair(out.double().numpy(), lse.double().numpy(), o, l)
    out.copy_(torch.from_numpy(o))
    lse.copy_(torch.from_numpy(l))


def oracle_merge(o_parts, l_parts, out, lse):
    """Left fold with an fp32 accumulator, as the running merge keeps it."""
    o, l = o_parts[0].double().numpy(), l_parts[0].double().numpy()
    for a, b in zip(o_parts[1:], l_parts[1:]):
        o, l = orc.merge_pair(o, l, a.double().numpy(), b.double().numpy())
        o, l = o.astype(np.float32).astype(np.float64), l.astype(np.float32).astype(np.float64)
    out.copy_(torch.from_numpy(o))
    lse.copy_(torch.from_numpy(l))


def oracle_decode(q, k_arena, v_arena, starts, lens, max_len, cfg, out, lse, ws=None):
    for b in range(q.shape[0]):
        s0, n = int(starts[b]), int(lens[b])
        qb = orc.blk_from_tokens(q[b:b + 1].float().numpy(), [0])
        kb = orc.blk_from_tokens(k_arena[s0:s0 + n].float().numpy(), np.zeros(n, np.int64))
        vb = orc.blk_from_tokens(v_arena[s0:s0 + n].float().numpy(), np.zeros(n, np.int64))
        o, l = orc.gqa(qb, kb, vb, cfg.n_kv_heads, cfg.scale)
        out[b] = torch.from_numpy(o[0])
        lse[b] = torch.from_numpy(l[0])


def _bf16(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16)


def _worker(rank, world, port, T, hq, hkv, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2411_01783_b200.attention import GqaConfig
        from paper_2411_01783_b200.kv_cache import RankKvCache
        from paper_2411_01783_b200.ring import KvLayout, QLayout, RingAttention, StepTrace, TorchRingComm
        from paper_2411_01783_b200.sharding import plan_decode

        D = 16
        cfg = GqaConfig(hq, hkv, D)
        rng = np.random.default_rng(123)  # same inputs on every rank
        qd = _bf16(rng.standard_normal((T, hq, D))).float().numpy()
        kd = _bf16(rng.standard_normal((T, hkv, D))).float().numpy()
        vd = _bf16(rng.standard_normal((T, hkv, D))).float().numpy()
        seqs = [orc.Seq(5, 0, T)]
        qb = orc.materialize(seqs, world, rank, [qd])
        kb = orc.materialize(seqs, world, rank, [kd])
        vb = orc.materialize(seqs, world, rank, [vd])
        S = qb.n
        q = _bf16(qb.data)
        q_pos = torch.from_numpy(np.where(qb.valid, qb.pos, -1).astype(np.int32))
        q_seq = torch.from_numpy(np.where(qb.valid, qb.seq, PAD_Q).astype(np.int32))
        lay = KvLayout(S, hkv, D)
        msg = torch.zeros(lay.nbytes, dtype=torch.uint8)
        k, v, kp, ks = lay.views(msg)
        k.copy_(_bf16(kb.data))
        v.copy_(_bf16(vb.data))
        kp.copy_(torch.from_numpy(np.where(kb.valid, kb.pos, POS_PAD_K).astype(np.int32)))
        ks.copy_(torch.from_numpy(np.where(kb.valid, kb.seq, PAD_K).astype(np.int32)))

        comm = TorchRingComm()
        ring = RingAttention(comm, attend=oracle_attend, merge=oracle_merge, decode=oracle_decode)
        ring.trace = StepTrace()
        out_kv = torch.empty((S, hq, D))
        lse_kv = torch.empty((S, hq))
        ring.pass_kv(q, q_pos, q_seq, lay, msg, cfg, out_kv, lse_kv)
        assert len(ring.trace.records) == world - 1  # N-1 sends per rank

        qlay = QLayout(S, hq, D)
        qmsg = torch.zeros(qlay.nbytes, dtype=torch.uint8)
        qq, qp, qs = qlay.views(qmsg)
        qq.copy_(q)
        qp.copy_(q_pos)
        qs.copy_(q_seq)
        out_q = torch.empty((S, hq, D))
        lse_q = torch.empty((S, hq))
        ring.pass_q(qlay, qmsg, k, v, kp, ks, cfg, out_q, lse_q)

        # composed oracle (ascending-source merge) and the ring's arrival-order merge
        caches = [orc.Cache(hkv, D) for _ in range(world)]
        _, want = orc.ring_prefill(seqs, [[0] * world], world, caches, [qd], [kd], [vd], hkv)
        sel = qb.valid
        assert np.abs(out_kv.numpy()[sel] - want[rank][0][sel]).max() < 1e-5
        assert np.abs(lse_kv.numpy()[sel] - want[rank][1][sel]).max() < 1e-5
        # pass-KV == pass-Q bitwise (same partials, same merge order)
        assert torch.equal(out_kv, out_q) and torch.equal(lse_kv, lse_q)

        # ---- decode: each rank's cache holds its prefill shard; 2 iterations
        cache = RankKvCache(hkv, D, capacity_tokens=64, device=torch.device("cpu"))
        kk = [i for i in range(S) if kb.valid[i]]
        cache.append_rows(5, _bf16(kb.data[kk]), _bf16(vb.data[kk]), kb.pos[kk])
        batch = [5]
        caches_o = [orc.Cache(hkv, D) for _ in range(world)]
        for r in range(world):
            b_r = orc.materialize(seqs, world, r, [kd])
            v_r = orc.materialize(seqs, world, r, [vd])
            caches_o[r].append(5, b_r, v_r)
        for it in range(4):
            dp = plan_decode(batch, world, it)
            tok_q = _bf16(rng.standard_normal((1, hq, D)))
            tok_k = _bf16(rng.standard_normal((1, hkv, D)))
            tok_v = _bf16(rng.standard_normal((1, hkv, D)))
            mine = dp.assignments[rank]
            o, l = ring.pass_q_decode(dp, cache, tok_q[: len(mine)] if mine else tok_q[:0],
                                      tok_k[: len(mine)], tok_v[: len(mine)], [T + it] * len(mine), cfg,
                                      gather=bool(it % 2))
            wo = orc.ring_decode(batch, world, it, caches_o, tok_q.float().numpy(), tok_k.float().numpy(),
                                 tok_v.float().numpy(), [T + it], hkv)
            if mine:
                assert np.abs(o[0].numpy() - wo[0][0][0]).max() < 1e-5
                assert np.abs(l[0].numpy() - wo[0][1][0]).max() < 1e-5
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,T,hq,hkv", [(2, 64, 4, 2), (3, 50, 4, 1), (8, 150, 4, 2)])
def test_ring_spmd_gloo(world, T, hq, hkv):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, hq, hkv, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
