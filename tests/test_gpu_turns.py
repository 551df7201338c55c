"""run_turns on one B200 through the sm_100a kernels (world 1).

The conversation of tests/test_turns_gloo.py (fused full prefill, decodes,
partial prefills, a new sequence joining a cached one) at D = 128, run with
pass-KV, pass-Q and adaptive, against the single-rank dense replay of the
whole conversation; tolerances are the bf16 ones of the other GPU tests
(|dO| <= 2e-2, |dLSE| <= 1e-3).
"""

import pytest
import torch

from tests.test_turns_gloo import check_transcript, dense_replay, make_scenario

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["pass_kv", "pass_q", "adaptive"])
@pytest.mark.parametrize("gather", [False, True])
def test_run_turns_cuda(strategy, gather):
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.turns import run_turns

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    turns = make_scenario(hq, hkv, D, seed=11)
    want = dense_replay(turns, hkv)
    ring = RingAttention(_LocalComm(0, 1))
    cache = RankKvCache(hkv, D, capacity_tokens=32)  # grows during the conversation
    recs = run_turns(ring, cache, cfg, turns, strategy=strategy, gather_decode=gather)
    torch.cuda.synchronize()
    assert check_transcript(recs, want, 2e-2, 1e-3) == 40 + 24 + 2 + 2 + 8 + 5 + 12 + 3 + 2
    assert [cache.cached_len(s) for s in (7, 9, 11)] == [52, 32, 14]


@pytest.mark.parametrize("strategy", ["pass_kv", "pass_q"])
def test_run_turns_cuda_e4m3_cache(strategy):
    """The same conversation on an FP8 (e4m3) cache with power-of-two scales:
    every cached K/V row is quantised on append and read back by the prefill
    messages (dequantised to bf16, exact for these scales) and by the decode
    kernel; the dense replay sees the same quantised rows."""
    import dataclasses

    import numpy as np

    from oracle import ringcp_oracle as orc
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.turns import run_turns

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    turns = make_scenario(hq, hkv, D, seed=11)
    sc = np.full(hkv, 2.0 ** -5, np.float32)

    def deq(t):
        return torch.from_numpy(orc.dequantize_e4m3(orc.quantize_e4m3(t.float().numpy(), sc), sc).astype(np.float32))

    def quantised(turn):
        if isinstance(turn.k, tuple):
            return dataclasses.replace(turn, k=tuple(deq(x) for x in turn.k), v=tuple(deq(x) for x in turn.v))
        return dataclasses.replace(turn, k=deq(turn.k), v=deq(turn.v))

    want = dense_replay([quantised(t) for t in turns], hkv)
    ring = RingAttention(_LocalComm(0, 1))
    cache = RankKvCache(hkv, D, capacity_tokens=32, kv_dtype="e4m3", k_scale=sc, v_scale=sc)
    recs = run_turns(ring, cache, cfg, turns, strategy=strategy)
    torch.cuda.synchronize()
    assert check_transcript(recs, want, 2e-2, 1e-3) == 40 + 24 + 2 + 2 + 8 + 5 + 12 + 3 + 2
    cache.close()
