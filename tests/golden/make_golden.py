"""Generate golden vectors by running the REAL reference package ``ringcp``.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``ringcp`` from /root/reference/pkg/src, evaluates the reference's
own functions on seeded inputs and writes ``tests/golden/*.npz``.  The fixtures
are committed; nothing on the GPU box reads /root/reference.

Cases:
  gqa_*      gqa_attention on the reference-test geometries (test_attention.py)
             plus D=128 bf16-exact cases sized for the CUDA kernel (ragged T,
             fused sequences, padding in the middle, cached offsets, peaky Q,
             zigzag rank blocks, empty K).
  merge_*    merge_attention folds (incl. all-masked partials).
  shard_*    plan_full_prefill / plan_partial_prefill / materialize_rank_block.
  decode_*   plan_decode assignments.
  ring_*     ring pass-KV composed from reference primitives (SPEC Alg. 2).
  sampled_*  the large-T recipe: a few query rows against 16K-24K keys, blocked
             gqa_attention + merge_attention and one unblocked call (inputs
             regenerated from the stored seed).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from ringcp.attention import (  # noqa: E402
    EmbeddingBlock,
    GqaConfig,
    PartialAttention,
    admitted_pair_count,
    gqa_attention,
    merge_attention,
)
from ringcp.sharding import (  # noqa: E402
    SequenceSpec,
    materialize_rank_block,
    plan_decode,
    plan_full_prefill,
    plan_partial_prefill,
)

OUT = os.path.dirname(os.path.abspath(__file__))


from make_golden_inputs import bf16_exact, sampled_inputs  # noqa: E402

def blk(data, pos, valid=None, seq=None):
    n = len(pos)
    valid = np.ones(n, bool) if valid is None else np.asarray(valid, bool)
    seq = np.zeros(n, np.int64) if seq is None else np.asarray(seq, np.int64)
    return EmbeddingBlock(data=np.asarray(data, np.float32), positions=np.asarray(pos, np.int64),
                          valid=valid, seq_ids=seq)


def put_block(store, key, b: EmbeddingBlock):
    store[f"{key}__data"] = np.asarray(b.data)
    store[f"{key}__pos"] = np.asarray(b.positions)
    store[f"{key}__valid"] = np.asarray(b.valid)
    store[f"{key}__seq"] = np.asarray(b.seq_ids)


def gqa_cases():
    store = {}
    names = []

    def add(name, q, k, v, cfg):
        part = gqa_attention(q, k, v, cfg)
        put_block(store, f"{name}__q", q)
        put_block(store, f"{name}__k", k)
        put_block(store, f"{name}__v", v)
        store[f"{name}__cfg"] = np.array([cfg.n_query_heads, cfg.n_kv_heads, cfg.head_dim])
        store[f"{name}__scale"] = np.array(cfg.scale, np.float64)
        store[f"{name}__out"] = np.asarray(part.output.data)
        store[f"{name}__lse"] = np.asarray(part.lse)
        store[f"{name}__pairs"] = np.array(admitted_pair_count(q, k))
        names.append(name)

    rng = np.random.default_rng(0)

    def mk(n, h, d, pos=None, seq=0, scale=1.0, exact=False):
        data = rng.standard_normal((n, h, d)).astype(np.float32) * scale
        if exact:
            data = bf16_exact(data)
        pos = np.arange(n) if pos is None else np.asarray(pos)
        return blk(data, pos, seq=np.full(n, seq))

    # --- reference-test geometries (test_attention.py:32-139)
    c = GqaConfig(2, 1, 4)
    add("single_key", mk(1, 2, 4, [5]), *(lambda b: (b, b))(mk(1, 1, 4, [3])), c)
    c = GqaConfig(1, 1, 4)
    kk = mk(1, 1, 4, [5])
    add("fully_masked", mk(1, 1, 4, [3]), kk, kk, c)
    c = GqaConfig(4, 2, 8)
    add("causal8", mk(8, 4, 8), mk(8, 2, 8), mk(8, 2, 8), c)
    c = GqaConfig(2, 2, 4)
    ko = mk(4, 2, 4, seq=2)
    add("cross_seq", mk(3, 2, 4, seq=1), ko, ko, c)

    # --- D=128 bf16-exact cases for the CUDA kernel
    c = GqaConfig(4, 1, 128)
    add("d128_ragged200", mk(200, 4, 128, exact=True), mk(200, 1, 128, exact=True),
        mk(200, 1, 128, exact=True), c)

    # fused two sequences with padding in the middle of the block (zigzag style)
    c = GqaConfig(8, 2, 128)
    T0, T1 = 150, 90
    qa, ka, va = (bf16_exact(rng.standard_normal((T0, h, 128)).astype(np.float32)) for h in (8, 2, 2))
    qb_, kb_, vb_ = (bf16_exact(rng.standard_normal((T1, h, 128)).astype(np.float32)) for h in (8, 2, 2))
    seqs = [SequenceSpec(7, 0, T0), SequenceSpec(9, 0, T1)]
    plan = plan_full_prefill(seqs, 2)
    q0 = materialize_rank_block(plan, 0, [qa, qb_])
    k1 = materialize_rank_block(plan, 1, [ka, kb_])
    v1 = materialize_rank_block(plan, 1, [va, vb_])
    k0 = materialize_rank_block(plan, 0, [ka, kb_])
    v0 = materialize_rank_block(plan, 0, [va, vb_])
    add("fused_r0_r0", q0, k0, v0, c)
    add("fused_r0_r1", q0, k1, v1, c)

    # cached offsets: queries at positions 300.., keys 0..299 (partial prefill shape)
    c = GqaConfig(8, 1, 128)
    add("cached_offset", mk(64, 8, 128, pos=np.arange(300, 364), exact=True),
        mk(300, 1, 128, exact=True), mk(300, 1, 128, exact=True), c)

    # peaky softmax (4x scaled Q) to stress tolerance
    c = GqaConfig(4, 1, 128)
    add("peaky", mk(256, 4, 128, scale=4.0, exact=True), mk(256, 1, 128, exact=True),
        mk(256, 1, 128, exact=True), c)

    # zigzag CP=2, T=512: rank-0 queries against rank-1 keys and own keys
    c = GqaConfig(4, 1, 128)
    T = 512
    qd, kd, vd = (bf16_exact(rng.standard_normal((T, h, 128)).astype(np.float32)) for h in (4, 1, 1))
    plan = plan_full_prefill([SequenceSpec(0, 0, T)], 2)
    for qr in range(2):
        for kr in range(2):
            add(f"zigzag_q{qr}_k{kr}", materialize_rank_block(plan, qr, [qd]),
                materialize_rank_block(plan, kr, [kd]), materialize_rank_block(plan, kr, [vd]), c)

    # empty key block
    c = GqaConfig(4, 1, 128)
    empty = EmbeddingBlock.padding(0, 1, 128)
    add("empty_k", mk(16, 4, 128, exact=True), empty, empty, c)
    # all-padding key block (no valid key anywhere)
    padk = EmbeddingBlock.padding(40, 1, 128)
    add("all_pad_k", mk(16, 4, 128, exact=True), padk, padk, c)
    return store, names


def merge_cases():
    store = {}
    rng = np.random.default_rng(1)
    names = []
    for idx, (n_parts, masked) in enumerate([(2, False), (3, False), (4, True), (1, False)]):
        parts = []
        for p in range(n_parts):
            out = rng.standard_normal((33, 4, 128))
            lse = rng.standard_normal((33, 4)) * 3
            if masked and p % 2 == 0:
                lse[::3] = -np.inf
                out[::3] = 0.0
            parts.append(PartialAttention(EmbeddingBlock.from_tokens(out, np.arange(33)), lse))
            store[f"m{idx}__p{p}__out"] = out
            store[f"m{idx}__p{p}__lse"] = lse
        if masked:  # a row that is -inf in every part
            for p in range(n_parts):
                store[f"m{idx}__p{p}__lse"][5] = -np.inf
                store[f"m{idx}__p{p}__out"][5] = 0.0
            parts = [PartialAttention(EmbeddingBlock.from_tokens(store[f"m{idx}__p{p}__out"], np.arange(33)),
                                      store[f"m{idx}__p{p}__lse"]) for p in range(n_parts)]
        merged = merge_attention(parts)
        store[f"m{idx}__n"] = np.array(n_parts)
        store[f"m{idx}__out"] = np.asarray(merged.output.data)
        store[f"m{idx}__lse"] = np.asarray(merged.lse)
        names.append(f"m{idx}")
    return store, names


def shard_cases():
    cases = []
    store = {}
    specs = [
        ("full", [(0, 0, 16)], 2, None),
        ("full", [(0, 0, 13)], 2, None),
        ("full", [(0, 0, 9)], 4, None),
        ("full", [(0, 0, 8)], 1, None),
        ("full", [(3, 0, 8), (5, 0, 4)], 2, None),
        ("full", [(1, 0, 37), (2, 0, 5), (4, 0, 64)], 3, None),
        ("full", [(0, 0, 4096)], 8, None),
        ("partial", [(0, 100, 8)], 2, [[50, 50]]),
        ("partial", [(0, 22, 8)], 2, [[10, 12]]),
        ("partial", [(1, 30, 11), (2, 7, 3)], 4, [[10, 5, 10, 5], [0, 7, 0, 0]]),
    ]
    rng = np.random.default_rng(2)
    for ci, (kind, seqs, n, layout) in enumerate(specs):
        ss = [SequenceSpec(*s) for s in seqs]
        plan = plan_full_prefill(ss, n) if kind == "full" else plan_partial_prefill(ss, n, layout)
        d = plan.to_json_dict()
        d["kind"] = kind
        d["total_query_slots"] = plan.total_query_slots()
        d["message_token_slots"] = plan.message_token_slots()
        d["local_indices"] = [[plan.rank_local_indices(i, r).tolist() for r in range(n)]
                              for i in range(len(ss))]
        d["to_json"] = plan.to_json()  # the plan wire format (--dump-plan), byte for byte
        cases.append(d)
        if max(s[2] for s in seqs) <= 128:
            data = [rng.standard_normal((s[2], 2, 4)).astype(np.float32) for s in seqs]
            for i, a in enumerate(data):
                store[f"s{ci}__in{i}"] = a
            for r in range(n):
                put_block(store, f"s{ci}__r{r}", materialize_rank_block(plan, r, data))
    return cases, store


def decode_cases():
    out = []
    for batch, n, it in [([0, 1, 2, 3], 2, 0), ([0, 1, 2, 3], 2, 1), ([5, 9, 2], 2, 3),
                         (list(range(32)), 8, 5), ([7], 8, 2), (list(range(10)), 4, 0)]:
        p = plan_decode(batch, n, it)
        out.append({"batch": batch, "n_ranks": n, "iteration": it,
                    "slots_per_rank": p.slots_per_rank,
                    "assignments": [[list(e) for e in a] for a in p.assignments]})
    return out


def ring_cases():
    """pass-KV composed from reference primitives."""
    store = {}
    rng = np.random.default_rng(3)
    names = []
    for name, n, seqs_t, hq, hkv in [("ring_n2_t256", 2, [256], 8, 1),
                                     ("ring_n3_fused", 3, [96, 60], 4, 2),
                                     ("ring_n4_t512", 4, [512], 4, 1)]:
        ss = [SequenceSpec(i, 0, t) for i, t in enumerate(seqs_t)]
        plan = plan_full_prefill(ss, n)
        cfg = GqaConfig(hq, hkv, 128)
        qd = [bf16_exact(rng.standard_normal((t, hq, 128)).astype(np.float32)) for t in seqs_t]
        kd = [bf16_exact(rng.standard_normal((t, hkv, 128)).astype(np.float32)) for t in seqs_t]
        vd = [bf16_exact(rng.standard_normal((t, hkv, 128)).astype(np.float32)) for t in seqs_t]
        for i in range(len(ss)):
            store[f"{name}__q{i}"] = qd[i]
            store[f"{name}__k{i}"] = kd[i]
            store[f"{name}__v{i}"] = vd[i]
        store[f"{name}__meta"] = np.array([n, hq, hkv] + seqs_t)
        # KV message of rank s: per sequence, new valid tokens (position-sorted) padded to L^i
        msgs = []
        for s in range(n):
            kb = materialize_rank_block(plan, s, kd)
            vb = materialize_rank_block(plan, s, vd)
            kp, vp = [], []
            for i, sp in enumerate(ss):
                sel = kb.valid & (kb.seq_ids == sp.seq_id)
                order = np.argsort(kb.positions[sel], kind="stable")
                kk = EmbeddingBlock(kb.data[sel][order], kb.positions[sel][order],
                                    kb.valid[sel][order], kb.seq_ids[sel][order])
                vv = EmbeddingBlock(vb.data[sel][order], vb.positions[sel][order],
                                    vb.valid[sel][order], vb.seq_ids[sel][order])
                L = plan.padded_len(i)
                kp.append(kk.pad_to(L))
                vp.append(vv.pad_to(L))
            msgs.append((EmbeddingBlock.concat(kp), EmbeddingBlock.concat(vp)))
        for r in range(n):
            qb = materialize_rank_block(plan, r, qd)
            merged = merge_attention([gqa_attention(qb, msgs[s][0], msgs[s][1], cfg) for s in range(n)])
            put_block(store, f"{name}__r{r}__q", qb)
            store[f"{name}__r{r}__out"] = np.asarray(merged.output.data)
            store[f"{name}__r{r}__lse"] = np.asarray(merged.lse)
        names.append(name)
    return store, names


def sampled_cases():
    """Large-T recipe: a few query rows against a long key
    sequence, as gqa_attention over consecutive key blocks folded with
    merge_attention (ascending), and as ONE gqa_attention call over all keys."""
    store = {}
    names = []
    for name, seed, T, hq, hkv, block, rows in [
        ("s24k_8x2", 5, 24576, 8, 2, 4096, [0, 1, 4095, 4096, 12287, 12288, 20000, 24575]),
        ("s16k_16x1", 6, 16384, 16, 1, 5000, [0, 127, 128, 8191, 8192, 16383]),
    ]:
        rows = np.array(rows, np.int64)
        q, k, v = sampled_inputs(seed, T, hq, hkv, rows)
        cfg = GqaConfig(hq, hkv, 128)
        qb = blk(q, rows)
        parts = []
        for a in range(0, T, block):
            b = min(T, a + block)
            parts.append(gqa_attention(qb, blk(k[a:b], np.arange(a, b)), blk(v[a:b], np.arange(a, b)), cfg))
        merged = merge_attention(parts)
        single = gqa_attention(qb, blk(k, np.arange(T)), blk(v, np.arange(T)), cfg)
        store[f"{name}__meta"] = np.array([seed, T, hq, hkv, block])
        store[f"{name}__rows"] = rows
        store[f"{name}__out_blocked"] = np.asarray(merged.output.data)
        store[f"{name}__lse_blocked"] = np.asarray(merged.lse)
        store[f"{name}__out_single"] = np.asarray(single.output.data)
        store[f"{name}__lse_single"] = np.asarray(single.lse)
        names.append(name)
    return store, names


def main():
    g, gn = gqa_cases()
    np.savez_compressed(os.path.join(OUT, "gqa.npz"), names=np.array(gn), **g)
    m, mn = merge_cases()
    np.savez_compressed(os.path.join(OUT, "merge.npz"), names=np.array(mn), **m)
    sc, ss = shard_cases()
    np.savez_compressed(os.path.join(OUT, "shard.npz"), **ss)
    with open(os.path.join(OUT, "shard.json"), "w") as f:
        json.dump(sc, f, indent=1, sort_keys=True)
    with open(os.path.join(OUT, "decode.json"), "w") as f:
        json.dump(decode_cases(), f, indent=1)
    r, rn = ring_cases()
    np.savez_compressed(os.path.join(OUT, "ring.npz"), names=np.array(rn), **r)
    sm, smn = sampled_cases()
    np.savez_compressed(os.path.join(OUT, "sampled.npz"), names=np.array(smn), **sm)
    print("wrote golden fixtures:", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
