"""Property tests (hypothesis) of the host-side planning against the oracle.

Random batches of sequences (1..4 sequences, 1..3000 new tokens, random
cached layouts over 1..8 ranks) and decode batches: the product planners
(`paper_2411_01783_b200.sharding`) must agree with the oracle restatement of
sharding.py (`oracle/ringcp_oracle.py`, itself pinned to the reference's
golden vectors) on every per-rank index map, token count, padded length and
query-slot count, and keep the load-balance invariants the paper relies on.
Pure host integer work: bit-exact equality.
"""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import ringcp_oracle as orc
from paper_2411_01783_b200.sharding import SequenceSpec, plan_decode, plan_full_prefill, plan_partial_prefill


@st.composite
def batches(draw, partial):
    n = draw(st.integers(1, 8))
    k = draw(st.integers(1, 4))
    ids = draw(st.lists(st.integers(0, 10 ** 6), min_size=k, max_size=k, unique=True))
    seqs, layout = [], []
    for sid in ids:
        T = draw(st.integers(1, 3000))
        if partial:
            row = draw(st.lists(st.integers(0, 500), min_size=n, max_size=n))
        else:
            row = [0] * n
        seqs.append(SequenceSpec(sid, sum(row), T))
        layout.append(row)
    return n, seqs, layout


def _check_plan(plan, n, seqs, layout):
    for i, s in enumerate(seqs):
        owned = []
        for r in range(n):
            loc = plan.rank_local_indices(i, r)
            want = orc.local_indices(s.new_len, n, r)
            assert np.array_equal(np.asarray(loc), want), (i, r)
            assert plan.new_token_count(i, r) == orc.new_count(s.new_len, n, r)
            owned.append(loc[loc >= 0])
        # every new token is owned by exactly one rank
        allv = np.sort(np.concatenate(owned))
        assert np.array_equal(allv, np.arange(s.new_len))
        assert plan.padded_len(i) == orc.padded_len(s.new_len, layout[i], n)
        c, _ = orc.chunk_table(s.new_len, n)
        assert plan.query_slots(i) == 2 * c
    assert plan.total_query_slots() == sum(2 * orc.chunk_table(s.new_len, n)[0] for s in seqs)


@settings(max_examples=150, deadline=None)
@given(batches(partial=False))
def test_full_prefill_plans_match_oracle(b):
    n, seqs, layout = b
    plan = plan_full_prefill(seqs, n)
    _check_plan(plan, n, seqs, layout)
    # load balance (SURVEY finding 2): new-token counts per rank differ by at
    # most 2 * (chunk remainder effects) -- exactly: max - min <= 2 * chunk_len
    for i, s in enumerate(seqs):
        counts = [plan.new_token_count(i, r) for r in range(n)]
        c, _ = orc.chunk_table(s.new_len, n)
        assert max(counts) - min(counts) <= 2 * c


@settings(max_examples=150, deadline=None)
@given(batches(partial=True))
def test_partial_prefill_plans_match_oracle(b):
    n, seqs, layout = b
    plan = plan_partial_prefill(seqs, n, layout)
    _check_plan(plan, n, seqs, layout)
    assert [list(r) for r in plan.cached_layout] == layout


@settings(max_examples=100, deadline=None)
@given(st.integers(1, 8), st.lists(st.integers(0, 10 ** 6), min_size=1, max_size=40, unique=True),
       st.integers(0, 1000))
def test_decode_plans_match_oracle(n, batch, it):
    plan = plan_decode(batch, n, it)
    want = orc.decode_assignments(batch, n, it)
    assert [list(a) for a in plan.assignments] == [list(map(tuple, a)) for a in want]
    sizes = [len(a) for a in plan.assignments]
    assert max(sizes) - min(sizes) <= 1  # round-robin balance
    assert max(sizes) <= plan.slots_per_rank
    for b, sid in enumerate(batch):
        assert (sid, b) in plan.assignments[plan.owner(b)]


@settings(deadline=None, max_examples=60)
@given(n=st.integers(1, 8), B=st.integers(1, 33), k=st.integers(1, 4), it0=st.integers(0, 50))
def test_decode_capacity_balance_invariant(n, B, k, it0):
    """running Alg. 4 for k·N iterations on a B-sequence batch
    leaves max - min over ranks of the cached decode tokens <= B (the plan's
    round-robin owner rotation), and every token is owned exactly once."""
    from paper_2411_01783_b200.sharding import plan_decode

    batch = list(range(100, 100 + B))
    per_rank = [0] * n
    per_seq = {s: 0 for s in batch}
    for it in range(it0, it0 + k * n):
        plan = plan_decode(batch, n, it)
        for r, a in enumerate(plan.assignments):
            per_rank[r] += len(a)
            for sid, _b in a:
                per_seq[sid] += 1
    assert max(per_rank) - min(per_rank) <= B
    assert all(v == k * n for v in per_seq.values())
