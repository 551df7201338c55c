"""GraphedDecode (CUDA-graph replay of the decode step) on one B200.

Two sequences with cached histories; every decode step is replayed from the
captured graph and checked against the dense oracle over the full history
(bf16 tolerances), and the cache must hold exactly the appended tokens.
"""

import numpy as np
import pytest
import torch

from oracle import ringcp_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("hist,table", [((3000, 1500), False), ((700, 2), False), ((3000, 1500), True),
                                        ((700, 2), True)])
def test_graphed_decode_matches_oracle(hist, table):
    """table=True: the step metadata of all future steps is precomputed on the
    device (first_positions given) and selected by the graph itself."""
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.decode_graph import GraphedDecode
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import _LocalComm

    hq, hkv, D = 16, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    rng = np.random.default_rng(3)
    bf = lambda *s: torch.from_numpy(rng.standard_normal(s).astype(np.float32)).to(torch.bfloat16)
    batch = [4, 9]
    cache = RankKvCache(hkv, D, capacity_tokens=64)
    host = {}
    for sid, L in zip(batch, hist):
        k, v = bf(L, hkv, D), bf(L, hkv, D)
        cache.append_rows(sid, k.cuda(), v.cuda(), np.arange(L))
        host[sid] = [k.float().numpy(), v.float().numpy()]
    first = {sid: L for sid, L in zip(batch, hist)} if table else None
    g = GraphedDecode(_LocalComm(0, 1), cache, cfg, batch, max_steps=8, first_positions=first)
    assert (g._table is not None) == table
    for step in range(6):
        q, k, v = bf(2, hq, D), bf(2, hkv, D), bf(2, hkv, D)
        pos = [cache.cached_len(s) for s in batch]
        out, lse = g.step(q.cuda(), k.cuda(), v.cuda(), pos)
        out, lse = out.cpu().numpy(), lse.cpu().numpy()
        for j, sid in enumerate(batch):
            host[sid][0] = np.concatenate([host[sid][0], k[j:j + 1].float().numpy()])
            host[sid][1] = np.concatenate([host[sid][1], v[j:j + 1].float().numpy()])
            n = host[sid][0].shape[0]
            o_w, l_w = orc.gqa(orc.blk_from_tokens(q[j:j + 1].float().numpy(), [pos[j]], sid),
                               orc.blk_from_tokens(host[sid][0], np.arange(n), sid),
                               orc.blk_from_tokens(host[sid][1], np.arange(n), sid), hkv)
            assert np.abs(out[j] - o_w[0]).max() < 2e-2, (step, sid)
            assert np.abs(lse[j] - l_w[0]).max() < 1e-3, (step, sid)
        assert g.graph is not None  # captured on the first step, replayed afterwards
        assert (g._table is not None) == table  # consecutive positions keep the device table
    assert [cache.cached_len(s) for s in batch] == [hist[0] + 6, hist[1] + 6]
    # the cached rows are the appended tokens, in position order
    for sid in batch:
        st, ln = cache.segment(sid)
        assert torch.equal(cache.k[st:st + ln].float().cpu(), torch.from_numpy(host[sid][0]))
        assert cache.pos[st:st + ln].cpu().tolist() == list(range(ln))
