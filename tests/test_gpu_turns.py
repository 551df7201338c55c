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
