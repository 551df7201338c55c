"""Heuristic / cost model (Eq. 1-3, Alg. 1, Tables 4-5). CPU only."""

import pytest

from paper_2411_01783_b200 import perf_model as pm

# (P, T, pass-KV ms, pass-Q ms) on CP4, P+T = 128000
TABLE4 = [(126720, 1280, 1023.39, 898.71), (124800, 3200, 1110.18, 1046.43),
          (123840, 4160, 1298.92, 1280.1), (121600, 6400, 1305.56, 1302.01),
          (115200, 12800, 2080.67, 2205.27), (102400, 25600, 3353.02, 3617.02),
          (89600, 38400, 4629.23, 4922.52), (76800, 51200, 5745.08, 6217.83),
          (64000, 64000, 6845.21, 7367.99), (51200, 76800, 7890.35, 8468.66),
          (38400, 89600, 8697.27, 9666.62), (25600, 102400, 10105.78, 10652.39),
          (12800, 115200, 11136.4, 11571.62), (0, 128000, 11462.15, 12360.57)]


def test_eq1_llama3_405b():
    assert pm.size_threshold(pm.profile("gtt-h100")) == 0.125
    m = pm.CostModel(128, 128, 128, 1e15, 1e11)
    assert pm.size_threshold(m) == 2.0  # MHA: ratio cap
    assert pm.size_threshold(pm.CostModel(32, 1, 128, 1e15, 1e11)) == 0.0625


def test_eq2_eq3_examples():
    m = pm.CostModel(128, 8, 128, 8e14, 5e10, n_ranks=1)
    assert pm.pass_kv_overlap_min_T(m) == pytest.approx(1000)
    assert pm.pass_q_overlap_min_ctx(m) == pytest.approx(8000)
    m4 = pm.with_ranks(m, 4)
    assert pm.pass_kv_overlap_min_T(m4) == pytest.approx(4000)  # linear in N
    assert pm.pass_q_overlap_min_ctx(pm.CostModel(64, 1, 256, 8e14, 5e10)) == pytest.approx(8000)


def test_comm_bytes_and_flops():
    m = pm.profile("gtt-h100")
    s = pm.PrefillShape(128000, 0)
    assert pm.comm_bytes(s, m, "KV") == pytest.approx(pm.comm_bytes(s, m, "Q") / 8)
    assert pm.comm_bytes(pm.PrefillShape(0, 10), m, "Q") == 0
    assert pm.comm_bytes(pm.PrefillShape(1, 4095), m, "Q") < pm.comm_bytes(pm.PrefillShape(1, 4095), m, "KV")
    a = pm.attention_flops(pm.PrefillShape(1024, 0), m)
    assert pm.attention_flops(pm.PrefillShape(2048, 0), m) == pytest.approx(4 * a)


@pytest.mark.parametrize("refined,name", [(False, "gtt-h100"), (True, "gtt-h100-calibrated")])
def test_table4_decisions(refined, name):
    """Every Table 4 row gets the measured winner except the 3.25 % and 5 % rows,
    which the SPEC exempts ("either option")."""
    m = pm.profile(name)
    hits = 0
    for P, T, kv, q in TABLE4:
        want = "pass_kv" if kv <= q else "pass_q"
        got = pm.choose_strategy(pm.PrefillShape(T, P), m, refined=refined)
        if T not in (4160, 6400):
            assert got == want, (P, T, got)
        hits += got == want
    assert hits >= 12


def test_table5_orderings():
    m = pm.profile("gtt-h100-calibrated")
    kv, q, attn, a2a = pm.predict_step_times(pm.PrefillShape(3200, 124800), m)
    assert kv > attn                     # 2.5 %: 627 > 414 us, exposed pass-KV comm
    assert a2a == pytest.approx(424e-6, rel=0.05)
    kv, q, attn, a2a = pm.predict_step_times(pm.PrefillShape(12800, 115200), m)
    assert attn > kv and attn > q        # 10 %: 1608 > 631, 544
    assert a2a == pytest.approx(1023e-6, rel=0.05)


def test_full_prefill_and_ties_pick_pass_kv():
    m = pm.profile("b200-nvl", n_ranks=8)
    assert pm.choose_strategy(pm.PrefillShape(131072, 0), m) == "pass_kv"
    assert pm.choose_strategy(pm.PrefillShape(16384, 114688), m) == "pass_kv"  # miss = 0.125 tie
    assert pm.choose_strategy(pm.PrefillShape(1, 1 << 20), m) == "pass_q"      # decode-like
    assert pm.choose_strategy(pm.PrefillShape(5, 5), pm.with_ranks(m, 1)) == "pass_kv"


def test_b200_thresholds_match_baseline_md():
    """Eq. 2 ≈ 228/456/911 tokens at N = 2/4/8 with C = 1640.6 TF/s, BW = 900 GB/s."""
    for n, want in [(2, 228), (4, 456), (8, 911)]:
        m = pm.CostModel(128, 8, 128, 1640.6e12, 900e9, n_ranks=n)
        assert pm.pass_kv_overlap_min_T(m) == pytest.approx(want, rel=0.01)
        assert pm.pass_q_overlap_min_ctx(m) == pytest.approx(want * 8, rel=0.01)
