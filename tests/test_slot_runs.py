"""Host-buffer staging: the vectorised run split of a slot range's source-row
map (ring._slot_runs) equals the per-element definition — maximal runs of
consecutive rows of one sequence, and of padding slots."""

import numpy as np

from paper_2411_01783_b200.ring import _slot_runs


def _runs_by_element(seg, seq_off):
    out, j = [], 0
    while j < seg.size:
        if seg[j] < 0:
            e = j
            while e < seg.size and seg[e] < 0:
                e += 1
            out.append((j, e, -1, 0))
        else:
            g = int(seg[j])
            si = int(np.searchsorted(seq_off, g, side="right")) - 1
            e = j + 1
            while e < seg.size and seg[e] == seg[e - 1] + 1 and seg[e] < seq_off[si + 1]:
                e += 1
            out.append((j, e, si, g - int(seq_off[si])))
        j = e
    return out


def test_slot_runs_random_maps():
    rng = np.random.default_rng(0)
    for _ in range(2000):
        lens = rng.integers(1, 40, size=rng.integers(1, 5))
        seq_off = np.cumsum([0, *lens])
        n = int(rng.integers(0, 80))
        seg = np.where(rng.random(n) < 0.2, -1, rng.integers(0, seq_off[-1], size=n))
        if n > 5 and rng.random() < 0.7:  # long consecutive stretches, possibly across sequences
            a = int(rng.integers(0, n - 3))
            b = int(rng.integers(a + 1, n))
            st = int(rng.integers(0, seq_off[-1]))
            seg[a:b] = np.clip(np.arange(st, st + b - a), 0, seq_off[-1] - 1)
        assert _slot_runs(seg, seq_off) == _runs_by_element(seg, seq_off)


def test_slot_runs_plan_layout():
    from paper_2411_01783_b200.sharding import SequenceSpec, _host_index_map, plan_full_prefill

    plan = plan_full_prefill([SequenceSpec(0, 0, 1000), SequenceSpec(1, 0, 37)], 4)
    seq_off = np.array([0, 1000, 1037])
    for r in range(4):
        idx, _, _ = _host_index_map(plan, r)
        runs = _slot_runs(idx, seq_off)
        assert runs == _runs_by_element(idx, seq_off)
        # every valid slot is covered exactly once, in order
        assert runs[0][0] == 0 and runs[-1][1] == idx.size
        assert all(x[1] == y[0] for x, y in zip(runs, runs[1:]))
