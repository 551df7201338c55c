"""Pin the large-T sampled-row oracle (oracle.gqa_grouped / sampled_rows_attention)
to the real reference: tests/golden/sampled.npz holds the reference's own
blocked gqa_attention + merge_attention and single-call results for a few query
rows against 16K-24K keys (make_golden.py::sampled_cases).  CPU only."""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from tests import _golden as G
from tests.golden.make_golden_inputs import sampled_inputs


@pytest.mark.parametrize("name", ["s24k_8x2", "s16k_16x1"])
def test_sampled_oracle_matches_reference(name):
    z = G.npz("sampled.npz")
    seed, T, hq, hkv, block = (int(x) for x in z[f"{name}__meta"])
    rows = z[f"{name}__rows"]
    q, k, v = sampled_inputs(seed, T, hq, hkv, rows)
    qb = orc.blk_from_tokens(q, rows)
    kb = orc.blk_from_tokens(k, np.arange(T))
    vb = orc.blk_from_tokens(v, np.arange(T))
    # same blocking as the reference run: agrees to fp64 rounding (BLAS order)
    o, l = orc.sampled_rows_attention(qb, kb, vb, hkv, block=block)
    assert np.abs(o - z[f"{name}__out_blocked"]).max() < 1e-12
    assert np.abs(l - z[f"{name}__lse_blocked"]).max() < 1e-12
    # and the reference's blocked fold equals its single call to fp64 rounding
    assert np.abs(z[f"{name}__out_blocked"] - z[f"{name}__out_single"]).max() < 1e-12
    # another blocking gives the same answer
    o2, l2 = orc.sampled_rows_attention(qb, kb, vb, hkv, block=3000)
    assert np.abs(o2 - z[f"{name}__out_single"]).max() < 1e-12
    assert np.abs(l2 - z[f"{name}__lse_single"]).max() < 1e-12


def test_grouped_gqa_matches_reference_golden():
    """gqa_grouped on every golden gqa case (padding, fused sequences, empty K, GQA ratios)."""
    z = G.npz("gqa.npz")
    for name in z["names"]:
        c = G.gqa_case(z, name)
        out, lse = orc.gqa_grouped(c["q"], c["k"], c["v"], c["hkv"], c["scale"])
        assert np.abs(out - c["out"]).max() < 1e-12, name
        assert np.array_equal(np.isneginf(lse), np.isneginf(c["lse"])), name
        fin = np.isfinite(c["lse"])
        if fin.any():
            assert np.abs(lse[fin] - c["lse"][fin]).max() < 1e-12, name


def test_sample_rows_cover_chunk_boundaries():
    rows = orc.sample_rows(131072, 8, 32)
    c = 131072 // 16
    for m in range(1, 16):
        assert m * c - 1 in rows and m * c in rows
    assert rows[0] == 0 and rows[-1] == 131071 and len(rows) >= 32
    assert np.all(np.diff(rows) > 0)
