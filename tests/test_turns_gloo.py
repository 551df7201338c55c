"""run_turns over world-size 2 and 3 gloo ranks on CPU.

A conversation of fused full prefill, decodes, partial prefills (one of them
adding a brand-new sequence next to a cached one) runs through
``paper_2411_01783_b200.turns.TurnRunner`` — product planning, cache layout
tracking, ring schedules and transport — with the per-step compute injected
from the CPU oracle (tests/test_ring_gloo.py).  Every turn's outputs must equal
the single-rank dense replay of the whole conversation (the SPEC's
post-condition), pass-KV and pass-Q transcripts must be bit-identical, and the
adaptive strategy must record Alg. 1's choice per prefill turn.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ringcp_oracle as orc
from tests.test_ring_gloo import _free_port, oracle_attend, oracle_decode, oracle_merge


def _bf16(x):
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16)


def make_scenario(hq, hkv, D, seed=7):
    """[prefill{7:40, 9:24}, decode[7,9], decode[7,9], prefill{7:8},
    prefill{9:5, 11:12}, decode[7,9,11], decode[11,7]] with bf16 data."""
    from paper_2411_01783_b200.turns import DecodeTurn, PrefillTurn

    rng = np.random.default_rng(seed)
    r = lambda *s: _bf16(rng.standard_normal(s))
    turns = []

    def pre(spec):
        ids = tuple(s for s, _ in spec)
        turns.append(PrefillTurn(ids, tuple(r(t, hq, D) for _, t in spec), tuple(r(t, hkv, D) for _, t in spec),
                                 tuple(r(t, hkv, D) for _, t in spec)))

    def dec(batch):
        b = len(batch)
        turns.append(DecodeTurn(tuple(batch), r(b, hq, D), r(b, hkv, D), r(b, hkv, D)))

    pre([(7, 40), (9, 24)])
    dec([7, 9])
    dec([7, 9])
    pre([(7, 8)])
    pre([(9, 5), (11, 12)])
    dec([7, 9, 11])
    dec([11, 7])
    return turns


def dense_replay(turns, hkv, scale=None):
    """Single-rank replay: per turn, {(seq_id, position): (o [Hq, D], lse [Hq])}."""
    from paper_2411_01783_b200.turns import PrefillTurn

    hist = {}  # seq id -> (k list, v list, positions list)
    want = []
    for turn in turns:
        if isinstance(turn, PrefillTurn):
            new = [(s, turn.q[i].float().numpy(), turn.k[i].float().numpy(), turn.v[i].float().numpy())
                   for i, s in enumerate(turn.seq_ids)]
        else:
            new = [(s, turn.q[b:b + 1].float().numpy(), turn.k[b:b + 1].float().numpy(),
                    turn.v[b:b + 1].float().numpy()) for b, s in enumerate(turn.batch)]
        qs = []
        for s, q, k, v in new:
            h = hist.setdefault(s, ([], [], []))
            p0 = len(h[2])
            pos = list(range(p0, p0 + q.shape[0]))
            h[0].append(k)
            h[1].append(v)
            h[2].extend(pos)
            qs.append((s, q, pos))
        res = {}
        for s, q, pos in qs:
            k, v, kp = np.concatenate(hist[s][0]), np.concatenate(hist[s][1]), hist[s][2]
            o, lse = orc.gqa(orc.blk_from_tokens(q, pos, s), orc.blk_from_tokens(k, kp, s),
                             orc.blk_from_tokens(v, kp, s), hkv, scale)
            for i, p in enumerate(pos):
                res[(s, p)] = (o[i], lse[i])
        want.append(res)
    return want


def check_transcript(records, want, otol, ltol):
    """Compare one rank's TurnRecords with the dense replay; returns #rows checked."""
    checked = 0
    for rec, exp in zip(records, want):
        if rec.kind == "decode":
            out, lse = rec.output
            last = {}
            for (s, p) in exp:
                last[s] = max(p, last.get(s, -1))
            for j, (sid, _b) in enumerate(rec.assignments):
                o_w, l_w = exp[(sid, last[sid])]
                assert np.abs(out[j].float().cpu().numpy() - o_w).max() < otol, (rec.index, sid)
                assert np.abs(lse[j].float().cpu().numpy() - l_w).max() < ltol, (rec.index, sid)
                checked += 1
        else:
            blk = rec.output.output
            data, lse = blk.data.float().cpu().numpy(), rec.output.lse.float().cpu().numpy()
            pos, valid, seq = (blk.positions.cpu().numpy(), blk.valid.cpu().numpy(), blk.seq_ids.cpu().numpy())
            for i in np.nonzero(valid)[0]:
                o_w, l_w = exp[(int(seq[i]), int(pos[i]))]
                assert np.abs(data[i] - o_w).max() < otol, (rec.index, int(seq[i]), int(pos[i]))
                assert np.abs(lse[i] - l_w).max() < ltol, (rec.index, int(seq[i]), int(pos[i]))
                checked += 1
    return checked


def _worker(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2411_01783_b200 import perf_model as pm
        from paper_2411_01783_b200.attention import GqaConfig
        from paper_2411_01783_b200.kv_cache import RankKvCache
        from paper_2411_01783_b200.ring import RingAttention, TorchRingComm
        from paper_2411_01783_b200.turns import TurnRunner

        hq, hkv, D = 4, 2, 16
        cfg = GqaConfig(hq, hkv, D)
        turns = make_scenario(hq, hkv, D)
        want = dense_replay(turns, hkv)
        comm = TorchRingComm()
        transcripts = {}
        for strategy in ("pass_kv", "pass_q", "adaptive"):
            ring = RingAttention(comm, attend=oracle_attend, merge=oracle_merge, decode=oracle_decode)
            cache = RankKvCache(hkv, D, capacity_tokens=16, device=torch.device("cpu"))  # forces arena growth
            runner = TurnRunner(ring, cache, cfg, strategy=strategy)
            recs = runner.run(turns)
            assert [r.kind for r in recs] == ["full_prefill", "decode", "decode", "partial_prefill",
                                              "partial_prefill", "decode", "decode"]
            n = check_transcript(recs, want, 1e-5, 1e-5)
            assert n > 0
            # cache state: per-rank cached counts add up to each sequence's length
            lens = torch.tensor([cache.cached_len(s) for s in (7, 9, 11)])
            dist.all_reduce(lens)
            assert lens.tolist() == [52, 32, 14], lens.tolist()
            for r in recs:
                if r.kind != "decode":
                    # N-1 ring sends per rank (+ one All2All for pass-Q)
                    kinds = [k for _s, _r, k, _b, _p in r.trace.records]
                    assert kinds.count("KV" if r.strategy == "pass_kv" else "Q") == world - 1
                    assert kinds.count("A2A") == (1 if r.strategy == "pass_q" else 0)
                    if strategy == "adaptive":
                        m = runner.cost_model
                        assert r.strategy == pm.choose_strategy(pm.PrefillShape(r.new_tokens, r.cached_tokens), m)
                    else:
                        assert r.strategy == strategy
            if strategy == "adaptive":  # P = 0 -> pass-KV; small partial turns -> pass-Q (Alg. 1)
                assert [r.strategy for r in recs if r.kind != "decode"] == ["pass_kv", "pass_q", "pass_q"]
            transcripts[strategy] = recs
        # protocol equivalence: pass-KV and pass-Q transcripts are bit-identical
        for a, b in zip(transcripts["pass_kv"], transcripts["pass_q"]):
            if a.kind == "decode":
                assert torch.equal(a.output[0], b.output[0]) and torch.equal(a.output[1], b.output[1])
            else:
                assert torch.equal(a.output.output.data, b.output.output.data)
                assert torch.equal(a.output.lse, b.output.lse)
        # unknown sequence in a decode turn is rejected before any work
        from paper_2411_01783_b200.turns import DecodeTurn
        bad = DecodeTurn((42,), turns[1].q[:1], turns[1].k[:1], turns[1].v[:1])
        with pytest.raises(ValueError, match="unknown sequence"):
            runner.decode(bad)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world", [2, 3, 8])
def test_run_turns_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
