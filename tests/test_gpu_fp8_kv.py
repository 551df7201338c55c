"""GPU: the FP8 (e4m3) KV-cache mode.

Quantise / dequantise / calibrate kernels bit-exact against the oracle's e4m3
restatement (itself pinned to torch.float8_e4m3fn in test_oracle_fp8.py); the
e4m3 decode kernel against the fp64 decode oracle on the DEQUANTISED K/V at
the bf16 decode tolerance; RankKvCache(kv_dtype="e4m3") through snapshots,
the simulated ring decode, the SPMD decode and the CUDA-graph decode."""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc
from tests import _golden as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rc():
    import paper_2411_01783_b200 as rc

    return rc


def _bf16(x):
    return orc.f32_to_bf16_values(np.asarray(x, np.float32))


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rows(rng, n, hkv, spread=True):
    x = rng.standard_normal((n, hkv, 128)) * (rng.uniform(0.05, 20, (1, hkv, 1)) if spread else 1.0)
    return _bf16(x)


def test_quantize_dequantize_calibrate_bit_exact(rc):
    import torch

    from paper_2411_01783_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(1)
    for n, hkv in ((1, 1), (37, 8), (4096, 2)):
        x = _rows(rng, n, hkv)
        x[0, 0, :4] = [1e4, -1e4, 1e-30, 0.0]  # saturation after a user scale, tiny, zero
        x = _bf16(x)
        xd = _dev(x).to(torch.bfloat16)
        row = hkv * 128
        scale = torch.empty(hkv, dtype=torch.float32, device="cuda")
        ws = torch.empty(hkv, dtype=torch.int32, device="cuda")
        _lib.check(lib.rcp_kv_calibrate_e4m3(_lib.ptr(xd), row, n, hkv, 128, _lib.ptr(scale), _lib.ptr(ws),
                                             _lib.stream_handle()))
        s = scale.cpu().numpy()
        np.testing.assert_array_equal(s, orc.e4m3_scale(x, hkv))
        for sc in (s, s * np.float32(0.25)):  # the second scale forces saturation
            sd = _dev(sc.astype(np.float32))
            q = torch.zeros((n, hkv, 128), dtype=torch.uint8, device="cuda")
            _lib.check(lib.rcp_kv_quantize_e4m3(_lib.ptr(q), row, 0, _lib.ptr(xd), row, n, hkv, 128, _lib.ptr(sd),
                                                _lib.stream_handle()))
            want = orc.quantize_e4m3(x, sc)
            np.testing.assert_array_equal(q.cpu().numpy(), want)
            back = torch.empty((n, hkv, 128), dtype=torch.bfloat16, device="cuda")
            _lib.check(lib.rcp_kv_dequantize_e4m3(_lib.ptr(back), row, _lib.ptr(q), row, n, hkv, 128, _lib.ptr(sd),
                                                  _lib.stream_handle()))
            np.testing.assert_array_equal(back.float().cpu().numpy(), orc.dequantize_e4m3_bf16(want, sc))
        # scatter form: row j -> dst_rows[j]
        dst_rows = rng.permutation(n + 5)[:n].astype(np.int64)
        q2 = torch.zeros((n + 5, hkv, 128), dtype=torch.uint8, device="cuda")
        rows_d, s_d = _dev(dst_rows), _dev(s)  # keep both alive across the launch
        _lib.check(lib.rcp_kv_quantize_e4m3(_lib.ptr(q2), row, _lib.ptr(rows_d), _lib.ptr(xd), row, n, hkv,
                                            128, _lib.ptr(s_d), _lib.stream_handle()))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(q2.cpu().numpy()[dst_rows], orc.quantize_e4m3(x, s))


def _decode_fp8(rc, q, kq, vq, ks, vs, starts, lens, hq, hkv):
    import torch

    from paper_2411_01783_b200.ring import _cuda_decode

    cfg = rc.GqaConfig(hq, hkv, 128)
    out = torch.empty((len(lens), hq, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((len(lens), hq), dtype=torch.float32, device="cuda")
    _cuda_decode(_dev(q).to(torch.bfloat16), _dev(kq), _dev(vq), _dev(np.asarray(starts, np.int64)),
                 _dev(np.asarray(lens, np.int64)), max(lens), cfg, out, lse, scales=(_dev(ks), _dev(vs)))
    return out.cpu().numpy(), lse.cpu().numpy()


@pytest.mark.parametrize("hq,hkv,lens", [(128, 8, [5000, 70, 0, 1]), (32, 8, [4099, 64]), (16, 1, [20000]),
                                         (8, 8, [63, 65, 129]), (64, 8, [100000]), (40, 1, [3000, 17])])
def test_decode_fp8_kernel_vs_oracle(rc, hq, hkv, lens):
    """rcp_decode_attn_fp8: ragged lengths, empty segment, tail blocks, many
    splits, GQA groups 1..16; per-head scales spanning 400x."""
    rng = np.random.default_rng(sum(lens) + hq)
    cap = sum(lens) + 256
    k = _rows(rng, cap, hkv)
    v = _rows(rng, cap, hkv)
    q = _bf16(rng.standard_normal((len(lens), hq, 128)) * 0.2)
    ks, vs = orc.e4m3_scale(k, hkv), orc.e4m3_scale(v, hkv)
    kq, vq = orc.quantize_e4m3(k, ks), orc.quantize_e4m3(v, vs)
    kd, vd = orc.dequantize_e4m3(kq, ks), orc.dequantize_e4m3(vq, vs)
    starts = np.cumsum([0] + lens[:-1]) + 3
    out, lse = _decode_fp8(rc, q, kq, vq, ks, vs, starts, lens, hq, hkv)
    vmax = np.abs(vd).max()
    for b, n in enumerate(lens):
        s0 = starts[b]
        qb = orc.blk_from_tokens(q[b:b + 1], [n])
        wo, wl = orc.gqa(qb, orc.blk_from_tokens(kd[s0:s0 + n], np.arange(n)),
                         orc.blk_from_tokens(vd[s0:s0 + n], np.arange(n)), hkv)
        # V spans up to 20x: the output tolerance scales with the V range (O is a convex combination)
        assert np.abs(out[b] - wo[0]).max() <= G.O_TOL * max(1.0, vmax / 4), (b, np.abs(out[b] - wo[0]).max())
        assert G.lse_err(lse[b], wl[0]) <= G.LSE_TOL


def test_decode_fp8_close_to_bf16(rc):
    """Quantisation error of the mode itself (informative bound): e4m3 K/V
    against the bf16 decode of the same rows, unit-variance data."""
    import torch

    from paper_2411_01783_b200.ring import _cuda_decode

    rng = np.random.default_rng(7)
    hq, hkv, n = 32, 8, 8192
    k, v = _rows(rng, n, hkv, spread=False), _rows(rng, n, hkv, spread=False)
    q = _bf16(rng.standard_normal((1, hq, 128)) * 0.2)
    ks, vs = orc.e4m3_scale(k, hkv), orc.e4m3_scale(v, hkv)
    out8, lse8 = _decode_fp8(rc, q, orc.quantize_e4m3(k, ks), orc.quantize_e4m3(v, vs), ks, vs, [0], [n], hq, hkv)
    cfg = rc.GqaConfig(hq, hkv, 128)
    o16 = torch.empty((1, hq, 128), dtype=torch.float32, device="cuda")
    l16 = torch.empty((1, hq), dtype=torch.float32, device="cuda")
    _cuda_decode(_dev(q).to(torch.bfloat16), _dev(k).to(torch.bfloat16), _dev(v).to(torch.bfloat16),
                 _dev(np.array([0], np.int64)), _dev(np.array([n], np.int64)), n, cfg, o16, l16)
    assert np.abs(out8 - o16.cpu().numpy()).max() <= 2e-2
    assert np.abs(lse8 - l16.cpu().numpy()).max() <= 5e-2


def test_fp8_cache_append_snapshot_and_growth(rc):
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache

    rng = np.random.default_rng(3)
    hkv = 2
    c = RankKvCache(hkv, 128, capacity_tokens=64, kv_dtype="e4m3", max_tokens=1 << 20)
    assert c.k.dtype == torch.uint8 and c.dtype == torch.bfloat16
    k0, v0 = _rows(rng, 100, hkv), _rows(rng, 100, hkv)
    mk = lambda a, p: rc.EmbeddingBlock(_dev(a).to(torch.bfloat16), np.asarray(p), np.ones(len(p), bool),
                                        np.zeros(len(p), np.int64))
    c.append(0, mk(k0, np.arange(100)), mk(v0, np.arange(100)))
    ks, vs = c.k_scale.cpu().numpy(), c.v_scale.cpu().numpy()
    np.testing.assert_array_equal(ks, orc.e4m3_scale(k0, hkv))
    np.testing.assert_array_equal(vs, orc.e4m3_scale(v0, hkv))
    # a later, out-of-order append (re-sorted) and growth far beyond the first mapping
    k1, v1 = _rows(rng, 50000, hkv), _rows(rng, 50000, hkv)
    p1 = np.arange(200, 50200)
    c.append(0, mk(k1, p1), mk(v1, p1))
    k2, v2 = _rows(rng, 50, hkv), _rows(rng, 50, hkv)
    c.append(0, mk(k2, np.arange(100, 150)), mk(v2, np.arange(100, 150)))
    kb, vb = c.snapshot_padded(0, 50200)
    allk = np.concatenate([k0, k2, k1])
    allv = np.concatenate([v0, v2, v1])
    np.testing.assert_array_equal(kb.data.float().cpu().numpy()[:50150],
                                  orc.dequantize_e4m3_bf16(orc.quantize_e4m3(allk, ks), ks))
    np.testing.assert_array_equal(vb.data.float().cpu().numpy()[:50150],
                                  orc.dequantize_e4m3_bf16(orc.quantize_e4m3(allv, vs), vs))
    assert kb.positions.cpu().tolist()[:151] == list(range(150)) + [200]
    c.close()


def test_fp8_ring_decode_vs_oracle(rc):
    """Alg. 4 over 4 simulated ranks with e4m3 caches (given scales), against
    the oracle ring decode on the dequantised rows."""
    import torch

    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import ring_pass_q_decode
    from paper_2411_01783_b200.sharding import plan_decode

    rng = np.random.default_rng(11)
    n, hq, hkv, B = 4, 16, 4, 3
    cfg = rc.GqaConfig(hq, hkv, 128)
    ks = np.float32(rng.uniform(0.002, 0.01, hkv))
    vs = np.float32(rng.uniform(0.002, 0.01, hkv))
    caches = [RankKvCache(hkv, 128, capacity_tokens=256, kv_dtype="e4m3", k_scale=ks, v_scale=vs)
              for _ in range(n)]
    # history: 700 tokens per sequence spread round-robin over ranks in 2N chunks (plain appends)
    hist = {}
    for b in range(B):
        T = 700 + 37 * b
        kk, vv = _rows(rng, T, hkv, spread=False), _rows(rng, T, hkv, spread=False)
        hist[b] = (kk, vv)
        for r in range(n):
            idx = orc.local_indices(T, n, r)
            idx = idx[idx >= 0]  # drop the padding slots
            caches[r].append_rows(b, _dev(kk[idx]).to(torch.bfloat16), _dev(vv[idx]).to(torch.bfloat16), idx)
    pos = {b: 700 + 37 * b for b in range(B)}
    for it in range(2 * n):
        plan = plan_decode(list(range(B)), n, it)
        q = _bf16(rng.standard_normal((B, hq, 128)) * 0.2)
        kt, vt = _rows(rng, B, hkv, spread=False), _rows(rng, B, hkv, spread=False)
        out, lse = ring_pass_q_decode(plan, caches, _dev(q).to(torch.bfloat16), _dev(kt).to(torch.bfloat16),
                                      _dev(vt).to(torch.bfloat16), [pos[b] for b in range(B)], cfg)
        for b in range(B):
            hk, hv = hist[b]
            hist[b] = (np.concatenate([hk, kt[b:b + 1]]), np.concatenate([hv, vt[b:b + 1]]))
            kd = orc.dequantize_e4m3(orc.quantize_e4m3(hist[b][0], ks), ks)
            vd = orc.dequantize_e4m3(orc.quantize_e4m3(hist[b][1], vs), vs)
            L = kd.shape[0]
            wo, wl = orc.gqa(orc.blk_from_tokens(q[b:b + 1], [pos[b]]), orc.blk_from_tokens(kd, np.arange(L)),
                             orc.blk_from_tokens(vd, np.arange(L)), hkv)
            assert np.abs(out[b].cpu().numpy() - wo[0]).max() <= G.O_TOL
            assert G.lse_err(lse[b].cpu().numpy(), wl[0]) <= G.LSE_TOL
            pos[b] += 1
    for c in caches:
        c.close()


def test_fp8_graphed_decode_vs_oracle(rc):
    """GraphedDecode over an e4m3 cache (the quantising appends are captured
    in the graph) against the oracle on the dequantised history."""
    import torch

    from paper_2411_01783_b200.decode_graph import GraphedDecode
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import _LocalComm

    rng = np.random.default_rng(5)
    hq, hkv = 32, 8
    cfg = rc.GqaConfig(hq, hkv, 128)
    batch = [4, 9]
    cache = RankKvCache(hkv, 128, capacity_tokens=64, kv_dtype="e4m3")
    with pytest.raises(ValueError):
        GraphedDecode(_LocalComm(0, 1), cache, cfg, batch, max_steps=8)  # no scales yet
    host = {}
    for sid, L in zip(batch, (3000, 700)):
        k, v = _rows(rng, L, hkv, spread=False), _rows(rng, L, hkv, spread=False)
        cache.append_rows(sid, _dev(k).to(torch.bfloat16), _dev(v).to(torch.bfloat16), np.arange(L))
        host[sid] = [k, v]
    ks, vs = cache.k_scale.cpu().numpy(), cache.v_scale.cpu().numpy()
    np.testing.assert_array_equal(ks, orc.e4m3_scale(host[4][0], hkv))  # calibrated on the first append
    g = GraphedDecode(_LocalComm(0, 1), cache, cfg, batch, max_steps=8)
    for step in range(6):
        q = _bf16(rng.standard_normal((2, hq, 128)) * 0.2)
        k, v = _rows(rng, 2, hkv, spread=False), _rows(rng, 2, hkv, spread=False)
        pos = [cache.cached_len(s) for s in batch]
        out, lse = g.step(_dev(q).to(torch.bfloat16), _dev(k).to(torch.bfloat16), _dev(v).to(torch.bfloat16), pos)
        out, lse = out.cpu().numpy(), lse.cpu().numpy()
        for j, sid in enumerate(batch):
            host[sid][0] = np.concatenate([host[sid][0], k[j:j + 1]])
            host[sid][1] = np.concatenate([host[sid][1], v[j:j + 1]])
            n = host[sid][0].shape[0]
            kd = orc.dequantize_e4m3(orc.quantize_e4m3(host[sid][0], ks), ks)
            vd = orc.dequantize_e4m3(orc.quantize_e4m3(host[sid][1], vs), vs)
            o_w, l_w = orc.gqa(orc.blk_from_tokens(q[j:j + 1], [pos[j]], sid), orc.blk_from_tokens(kd, np.arange(n), sid),
                               orc.blk_from_tokens(vd, np.arange(n), sid), hkv)
            assert np.abs(out[j] - o_w[0]).max() <= G.O_TOL, (step, sid)
            assert G.lse_err(lse[j], l_w[0]) <= G.LSE_TOL, (step, sid)
        assert g.graph is not None
    # the appended rows were quantised in the graph exactly as the oracle does
    for sid in batch:
        st, ln = cache.segment(sid)
        np.testing.assert_array_equal(cache.k[st:st + ln].cpu().numpy(), orc.quantize_e4m3(host[sid][0], ks))
    cache.close()
