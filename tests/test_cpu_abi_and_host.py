"""CPU-only: the C-ABI library loads and exports every symbol include/*.h
declares; host-side plan logic matches the reference's golden plans; message
layouts and the ring topology.  No kernel is launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from tests import _golden as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ringcp_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(rcp_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2411_01783_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2411_01783_b200 import _build

        _build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    # every declared symbol is typed by the binding, and vice versa
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_product_and_ab_library_forms():
    """The product library runs only the v4 attention kernel (the selector is
    compiled out); the A/B library exports the same ABI and honours it."""
    import subprocess
    import sys

    from paper_2411_01783_b200 import _build, _lib

    if not os.path.exists(_build.LIB_AB):
        _build.build()
    ab = ctypes.CDLL(_build.LIB_AB)
    for s in declared_symbols():
        assert hasattr(ab, s), s
    code = ("import ctypes,sys; l=ctypes.CDLL(sys.argv[1]); l.rcp_attn_version.restype=ctypes.c_int; "
            "print(l.rcp_attn_version())")
    env = dict(os.environ, RCP_ATTN_VERSION="12")
    prod = subprocess.run([sys.executable, "-c", code, _lib.LIB_PATH], env=env, capture_output=True, text=True)
    abv = subprocess.run([sys.executable, "-c", code, _build.LIB_AB], env=env, capture_output=True, text=True)
    assert prod.stdout.strip() == "4" and abv.stdout.strip() == "12", (prod.stdout, prod.stderr, abv.stderr)


def test_library_host_only_calls():
    """Calls that never touch a GPU: version, workspace sizes, argument errors."""
    from paper_2411_01783_b200 import _lib

    lib = _lib.load()
    assert b"sm_100a" in lib.rcp_version()
    assert lib.rcp_attn_workspace_bytes(256, 512) >= 32 * (2 + 8)
    assert lib.rcp_decode_workspace_bytes(4, 32, 1024) >= 4 * 32 * 129 * 4
    # argument validation happens before any CUDA call
    rc = lib.rcp_attn_fwd(None, 0, None, 0, None, 0, None, None, None, None, 4, 4, 3, 2, 128,
                          1.0, None, None, 0, None, 0, None)
    assert rc == _lib.RCP_ERR_INVALID and b"divisible" in lib.rcp_last_error()
    rc = lib.rcp_attn_fwd(None, 0, None, 0, None, 0, None, None, None, None, 4, 4, 2, 1, 64,
                          1.0, None, None, 0, None, 0, None)
    assert rc == _lib.RCP_ERR_INVALID and b"head_dim" in lib.rcp_last_error()
    with pytest.raises(ValueError, match="empty"):
        _lib.check(lib.rcp_merge_attn(None, None, 0, 1, 128, None, None, None))


def test_plans_match_reference_golden():
    from paper_2411_01783_b200.sharding import SequenceSpec, plan_full_prefill, plan_partial_prefill

    for c in G.js("shard.json"):
        n = c["n_ranks"]
        seqs = [SequenceSpec(s["seq_id"], s["cached_len"], s["new_len"]) for s in c["sequences"]]
        plan = (plan_full_prefill(seqs, n) if c["kind"] == "full" else
                plan_partial_prefill(seqs, n, [s["rank_cached_counts"] for s in c["sequences"]]))
        d = plan.to_json_dict()
        for key in ("n_ranks", "assignment"):
            assert d[key] == c[key]
        for got, want in zip(d["sequences"], c["sequences"]):
            assert got == want
        assert plan.total_query_slots() == c["total_query_slots"]
        assert plan.message_token_slots() == c["message_token_slots"]
        for i in range(len(seqs)):
            for r in range(n):
                assert plan.rank_local_indices(i, r).tolist() == c["local_indices"][i][r]


def test_plan_errors_match_reference_messages():
    from paper_2411_01783_b200.sharding import (SequenceSpec, plan_decode, plan_full_prefill,
                                                plan_partial_prefill)

    with pytest.raises(ValueError, match="empty sequence list"):
        plan_full_prefill([], 2)
    with pytest.raises(ValueError, match="duplicate seq_id"):
        plan_full_prefill([SequenceSpec(1, 0, 4), SequenceSpec(1, 0, 4)], 2)
    with pytest.raises(ValueError, match="use plan_partial_prefill"):
        plan_full_prefill([SequenceSpec(1, 3, 4)], 2)
    with pytest.raises(ValueError, match="decode turns use plan_decode"):
        plan_full_prefill([SequenceSpec(1, 0, 0)], 2)
    with pytest.raises(ValueError, match="cached_layout"):
        plan_partial_prefill([SequenceSpec(1, 10, 4)], 2, [[3, 3]])
    with pytest.raises(ValueError, match="n_ranks"):
        plan_full_prefill([SequenceSpec(1, 0, 4)], 0)
    with pytest.raises(ValueError, match="duplicate"):
        plan_decode([1, 1], 2, 0)
    with pytest.raises(ValueError):
        SequenceSpec(1, -1, 3)


def test_decode_plans_match_reference_golden():
    from paper_2411_01783_b200.sharding import plan_decode

    for c in G.js("decode.json"):
        p = plan_decode(c["batch"], c["n_ranks"], c["iteration"])
        assert [[list(e) for e in a] for a in p.assignments] == c["assignments"]
        assert p.slots_per_rank == c["slots_per_rank"]


def test_decode_round_robin_balance():
    """after t iterations, per-sequence per-rank appended counts differ by <= 1."""
    from paper_2411_01783_b200.sharding import plan_decode

    for B in range(1, 9):
        for n in (1, 2, 3, 4, 8):
            counts = np.zeros((B, n), int)
            for it in range(32):
                p = plan_decode(list(range(B)), n, it)
                for b in range(B):
                    counts[b, p.owner(b)] += 1
                assert (counts.max(1) - counts.min(1)).max() <= 1


def test_load_balance_pair_counts():
    """SPEC.md:145 (code semantics, SURVEY finding 4): equal admitted pairs per
    rank for T divisible by 2N, T(T+1)/(2N) each."""
    from oracle import ringcp_oracle as orc

    for n in (1, 2, 4):
        for T in (16, 64, 256):
            pos = [orc.local_indices(T, n, r) for r in range(n)]
            cnt = [int(sum(p + 1 for p in ps if p >= 0)) for ps in pos]
            assert len(set(cnt)) == 1 and cnt[0] == T * (T + 1) // (2 * n)


def test_message_layouts_and_topology():
    from paper_2411_01783_b200.ring import KvLayout, QLayout, RingTopology

    lay = KvLayout(1000, 8, 128)
    assert lay.v_off % 256 == 0 and lay.pos_off % 256 == 0 and lay.seq_off % 256 == 0
    assert lay.nbytes >= 2 * 1000 * 8 * 128 * 2 + 8 * 1000
    q = QLayout(77, 32, 128)
    assert q.nbytes >= 77 * 32 * 128 * 2 + 8 * 77
    t = RingTopology(4)
    assert [t.next(k) for k in range(4)] == [1, 2, 3, 0]
    assert [t.source_at(1, s) for s in range(4)] == [1, 0, 3, 2]


def test_shard_plan_json_wire_format_matches_reference_bytes():
    """ShardPlan.to_json (sharding.py:117-141, the --dump-plan wire format,
    SPEC.md:158/497) is byte-identical to the reference's for every golden
    plan, and round-trips through json."""
    import json

    from paper_2411_01783_b200.sharding import SequenceSpec, plan_full_prefill, plan_partial_prefill

    for c in G.js("shard.json"):
        seqs = [SequenceSpec(s["seq_id"], s["cached_len"], s["new_len"]) for s in c["sequences"]]
        n = c["n_ranks"]
        plan = (plan_full_prefill(seqs, n) if c["kind"] == "full" else
                plan_partial_prefill(seqs, n, [s["rank_cached_counts"] for s in c["sequences"]]))
        assert plan.to_json() == c["to_json"]
        d = json.loads(plan.to_json())
        assert d["assignment"] == [[r, 2 * n - 1 - r] for r in range(n)]
