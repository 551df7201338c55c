"""On-box calibration of the pass-KV / pass-Q cost model (perf_model.calibrate_b200;
SPEC.md:372-390, 422): the attention rate is measured from the kernel in this
run, and Alg. 1 with the calibrated constants still picks pass-KV for full
prefill (P = 0) and for high miss rates."""

import pytest

pytestmark = pytest.mark.gpu


def test_calibrate_world1_is_sane_and_drives_alg1():
    from paper_2411_01783_b200 import perf_model as pm
    from paper_2411_01783_b200.ring import _LocalComm

    m, meas = pm.calibrate_b200(_LocalComm(0, 1), pm.LLAMA3_8B, n_ranks=1, step_tokens=4096, reps=3)
    assert 300.0 < meas["attn_tflops"] < 2500.0, meas
    assert m.peak_compute == pytest.approx(meas["attn_tflops"] * 1e12)
    m4 = pm.with_ranks(m, 4)
    assert pm.choose_strategy(pm.PrefillShape(131072, 0), m4) == "pass_kv"
    assert pm.choose_strategy(pm.PrefillShape(65536, 65536), m4) == "pass_kv"
    for refined in (False, True):
        assert pm.choose_strategy(pm.PrefillShape(128, 131072), pm.with_ranks(m, 8), refined=refined) in (
            "pass_kv", "pass_q")
