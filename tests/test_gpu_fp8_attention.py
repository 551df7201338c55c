"""GPU: the FP8-QK attention kernel (rcp_attn_fwd_qk8: e4m3 Q / K with
per-head scales, S on tcgen05 kind::f8f6f4, P / V bf16) — an opt-in FP8 mode
(SURVEY §8f rank 4).  Parity is against the fp32 torch reference (and the
fp64 oracle at scale) on the DEQUANTISED Q / K, at the bf16 tolerances:
segmented / padded / GQA / merge-mode cases, the reference's causal mask at
a CP-step shape, and gqa_attention_fp8 through the public blocks."""

import math

import numpy as np
import pytest
import torch

from oracle import ringcp_oracle as orc
from tests import _golden as G
from tests.test_gpu_attention_soak import PAD_K, PAD_Q, POS_PAD_K, _block, _reference

pytestmark = pytest.mark.gpu


def _deq(x8: torch.Tensor, scale: torch.Tensor) -> torch.Tensor:
    """e4m3 bytes [T, H, D] -> the exact float32 values scale[h] * e4m3."""
    return torch.from_numpy(orc.dequantize_e4m3(x8.cpu().numpy(), scale.cpu().numpy()).astype(np.float32)).cuda()


@pytest.mark.parametrize("case", range(8))
def test_qk8_kernel_vs_reference(case):
    from paper_2411_01783_b200 import _lib
    from paper_2411_01783_b200.attention import attend_into_qk8, quantize_heads_e4m3

    rng = np.random.default_rng(900 + case)
    hkv = int(rng.choice([1, 2, 8]))
    hq = hkv * int(rng.choice([1, 4, 8]))
    tq, tk = int(rng.integers(200, 2100)), int(rng.integers(200, 2600))
    qp, qs = _block(rng, tq, 2, [3, 9], PAD_Q, -1)
    kp, ks = _block(rng, tk, 2, [3, 9], PAD_K, POS_PAD_K)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(case)
    q = torch.randn(tq, hq, 128, device=dev, dtype=torch.bfloat16, generator=g) * (0.5 + case)
    k = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(tk, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    q8, qsc = quantize_heads_e4m3(q)
    k8, ksc = quantize_heads_e4m3(k)
    qp_d, qs_d = torch.from_numpy(qp).to(dev), torch.from_numpy(qs).to(dev)
    kp_d, ks_d = torch.from_numpy(kp).to(dev), torch.from_numpy(ks).to(dev)
    scale = 1.0 / math.sqrt(128)
    merge = case % 2 == 1
    out = torch.randn(tq, hq, 128, device=dev) if merge else torch.empty(tq, hq, 128, device=dev)
    lse = torch.randn(tq, hq, device=dev) if merge else torch.empty(tq, hq, device=dev)
    o0, l0 = out.clone(), lse.clone()
    attend_into_qk8(q8, qsc, (qp_d, qs_d), k8, ksc, v, (kp_d, ks_d), hq, hkv, scale, out, lse,
                    _lib.MODE_MERGE if merge else _lib.MODE_OVERWRITE)
    ro, rl = _reference(_deq(q8, qsc), _deq(k8, ksc), v, qp_d.long(), qs_d.long(), kp_d.long(), ks_d.long(),
                        hq, hkv, scale)
    if merge:
        m = torch.maximum(l0, rl)
        m = torch.where(torch.isfinite(m), m, torch.zeros_like(m))
        wa, wb = torch.exp(l0 - m), torch.exp(rl - m)
        tot = wa + wb
        rl = torch.log(tot) + m
        ro = (o0 * wa[..., None] + ro * wb[..., None]) / tot[..., None]
    torch.cuda.synchronize()
    valid = torch.from_numpy(qs != PAD_Q).to(dev)
    assert float((out[valid] - ro[valid]).abs().max()) <= G.O_TOL
    fin = torch.isfinite(rl) & valid[:, None]
    assert torch.equal(torch.isfinite(lse) & valid[:, None], fin)
    if fin.any():
        assert float((lse[fin] - rl[fin]).abs().max()) <= G.LSE_TOL


def test_gqa_attention_fp8_cp_step_shape_vs_oracle():
    """A CP8 step of the 8B-shape 128K run (16384 x 16384 causal, 32 / 8 heads)
    through gqa_attention_fp8, sampled rows against the fp64 oracle on the
    dequantised Q / K; and the quantisation error against the bf16 kernel."""
    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.attention import gqa_attention_fp8, quantize_heads_e4m3

    T, hq, hkv = 16384, 32, 8
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(5)
    q = torch.randn(T, hq, 128, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(T, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(T, hkv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    pos = np.arange(T)
    cfg = rc.GqaConfig(hq, hkv, 128)
    mk = lambda x: rc.EmbeddingBlock(x, pos, np.ones(T, bool), np.zeros(T, np.int64))
    got = gqa_attention_fp8(mk(q), mk(k), mk(v), cfg)
    q8, qs = quantize_heads_e4m3(q)
    k8, ks = quantize_heads_e4m3(k)
    qd, kd = _deq(q8, qs).cpu().numpy(), _deq(k8, ks).cpu().numpy()
    vf = v.float().cpu().numpy()
    rows = np.array([0, 1, 127, 128, 8191, 8192, 16000, T - 1])
    wo, wl = orc.gqa(orc.blk_from_tokens(qd[rows], rows), orc.blk_from_tokens(kd, pos), orc.blk_from_tokens(vf, pos),
                     hkv, cfg.scale)
    o = got.output.data[rows].cpu().numpy()
    l = got.lse[rows].cpu().numpy()
    assert np.abs(o - wo).max() <= G.O_TOL
    assert G.lse_err(l, wl) <= G.LSE_TOL
    # informative: the quantisation error itself, e4m3 Q / K against the bf16
    # kernel on the same inputs (largest on the first rows, which attend to a
    # handful of keys; small on average)
    ref = rc.gqa_attention(mk(q), mk(k), mk(v), cfg)
    d_o = (got.output.data - ref.output.data).abs()
    assert float(d_o.max()) <= 0.25 and float(d_o.mean()) <= 5e-3, (float(d_o.max()), float(d_o.mean()))
    d_l = (got.lse - ref.lse).abs()
    assert float(d_l.max()) <= 0.25 and float(d_l.mean()) <= 1e-2, (float(d_l.max()), float(d_l.mean()))


def test_ring_with_fp8_qk_attend_vs_oracle():
    """RingAttention(attend=Fp8QkAttend()) — the CP prefill's opt-in FP8 mode —
    on one rank: the pass-KV prefill of a fused two-sequence batch against the
    oracle on the per-call quantised-then-dequantised Q / K."""
    import paper_2411_01783_b200 as rc
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import Fp8QkAttend, RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    rng = np.random.default_rng(17)
    hq, hkv = 16, 2
    cfg = rc.GqaConfig(hq, hkv, 128)
    lens = [700, 333]
    bf = lambda a: orc.f32_to_bf16_values(np.asarray(a, np.float32))
    q = [bf(rng.standard_normal((t, hq, 128))) for t in lens]
    k = [bf(rng.standard_normal((t, hkv, 128))) for t in lens]
    v = [bf(rng.standard_normal((t, hkv, 128))) for t in lens]
    plan = plan_full_prefill([SequenceSpec(i, 0, t) for i, t in enumerate(lens)], 1)
    dev = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)
    qb = materialize_rank_block(plan, 0, [dev(x) for x in q])
    kb = materialize_rank_block(plan, 0, [dev(x) for x in k])
    vb = materialize_rank_block(plan, 0, [dev(x) for x in v])
    ring = RingAttention(_LocalComm(0, 1), attend=Fp8QkAttend())
    cache = RankKvCache(hkv, 128, capacity_tokens=4096)
    got = ring.pass_kv_prefill(plan, cache, qb, kb, vb, cfg)
    torch.cuda.synchronize()
    # the oracle: Q block and the KV message's K quantised per call exactly as the kernel saw them
    qd = qb.data.float().cpu().numpy()
    kd = kb.data.float().cpu().numpy()  # one rank: the message holds the same rows as the block
    q_deq = orc.dequantize_e4m3(orc.quantize_e4m3(qd, orc.e4m3_scale(qd, hq)), orc.e4m3_scale(qd, hq))
    k_deq = orc.dequantize_e4m3(orc.quantize_e4m3(kd, orc.e4m3_scale(kd, hkv)), orc.e4m3_scale(kd, hkv))
    qpos, qseq = qb.positions.cpu().numpy(), qb.seq_ids.cpu().numpy()
    kv = kb.valid.cpu().numpy()
    wo, wl = orc.gqa(orc.Blk(q_deq, qpos, qb.valid.cpu().numpy(), qseq),
                     orc.Blk(k_deq, kb.positions.cpu().numpy(), kv, kb.seq_ids.cpu().numpy()),
                     orc.Blk(vb.data.float().cpu().numpy(), kb.positions.cpu().numpy(), kv, kb.seq_ids.cpu().numpy()),
                     hkv)
    valid = qb.valid.cpu().numpy()
    assert np.abs(got.output.data.cpu().numpy()[valid] - wo[valid]).max() <= G.O_TOL
    assert G.lse_err(got.lse.cpu().numpy()[valid], wl[valid]) <= G.LSE_TOL
    cache.close()
