"""pass_kv_prefill_host (host inputs/outputs, PCIe copies overlapped with the
attention) must equal pass_kv_prefill on device inputs bit for bit: the query
slot ranges are multiples of 256 rows, so every CTA sees the same query tile
pair and the same key blocks."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_sub", [1, 3, 8])
@pytest.mark.parametrize("partial", [False, True])
def test_host_stream_equals_device_path(n_sub, partial):
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_full_prefill,
                                                plan_partial_prefill)

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    g = torch.Generator().manual_seed(1)
    lens = [1700, 900]
    cached = [600, 0] if partial else [0, 0]
    seqs = [SequenceSpec(3, cached[0], lens[0]), SequenceSpec(8, cached[1], lens[1])]
    plan = plan_partial_prefill(seqs, 1, [[c] for c in cached]) if partial else plan_full_prefill(seqs, 1)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).pin_memory()
    qh = [mk(n, hq, D) for n in lens]
    kh = [mk(n, hkv, D) for n in lens]
    vh = [mk(n, hkv, D) for n in lens]
    hist = (mk(cached[0], hkv, D), mk(cached[0], hkv, D)) if partial else None

    def fresh_cache():
        c = RankKvCache(hkv, D, capacity_tokens=256)
        if partial:
            c.append_rows(3, hist[0].cuda(), hist[1].cuda(), np.arange(cached[0]))
        return c

    ring = RingAttention(_LocalComm(0, 1))
    ref = ring.pass_kv_prefill(plan, fresh_cache(), materialize_rank_block(plan, 0, [t.cuda() for t in qh]),
                               materialize_rank_block(plan, 0, [t.cuda() for t in kh]),
                               materialize_rank_block(plan, 0, [t.cuda() for t in vh]), cfg)
    S = ref.output.n_tokens
    out_h = torch.full((S, hq, D), float("nan")).pin_memory()
    lse_h = torch.full((S, hq), float("nan")).pin_memory()
    ring.pass_kv_prefill_host(plan, fresh_cache(), qh, kh, vh, cfg, out_h, lse_h, n_sub=n_sub)
    torch.cuda.synchronize()
    assert torch.equal(out_h, ref.output.data.cpu())
    assert torch.equal(lse_h, ref.lse.cpu())


def test_staged_pipeline_two_requests():
    """Serving-loop use: request 2 is staged while request 1 computes, the
    D2H stream is joined once at the end; both results equal the device path."""
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    g = torch.Generator().manual_seed(5)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).pin_memory()
    reqs = []
    for T in (2048, 1300):
        plan = plan_full_prefill([SequenceSpec(1, 0, T)], 1)
        reqs.append((plan, [mk(T, hq, D)], [mk(T, hkv, D)], [mk(T, hkv, D)]))
    ring = RingAttention(_LocalComm(0, 1))
    refs = []
    for plan, qh, kh, vh in reqs:
        r = ring.pass_kv_prefill(plan, RankKvCache(hkv, D, capacity_tokens=256),
                                 materialize_rank_block(plan, 0, [qh[0].cuda()]),
                                 materialize_rank_block(plan, 0, [kh[0].cuda()]),
                                 materialize_rank_block(plan, 0, [vh[0].cuda()]), cfg)
        refs.append((r.output.data.cpu(), r.lse.cpu()))
    torch.cuda.synchronize()
    outs = []
    dev = torch.device("cuda")
    st = ring.stage_host_inputs(reqs[0][0], reqs[0][1], reqs[0][2], reqs[0][3], cfg, dev)
    for i, (plan, qh, kh, vh) in enumerate(reqs):
        nxt = ring.stage_host_inputs(*reqs[i + 1], cfg, dev) if i + 1 < len(reqs) else None
        S = plan.total_query_slots()
        oh = torch.empty((S, hq, D)).pin_memory()
        lh = torch.empty((S, hq)).pin_memory()
        ring.pass_kv_prefill_host(plan, RankKvCache(hkv, D, capacity_tokens=256), qh, kh, vh, cfg, oh, lh,
                                  staged=st, join=False)
        outs.append((oh, lh))
        st = nxt
    ring.join_host_copies()
    torch.cuda.synchronize()
    for (oh, lh), (ro, rl) in zip(outs, refs):
        assert torch.equal(oh, ro) and torch.equal(lh, rl)


@pytest.mark.parametrize("ahead", [1, 3, 6])
def test_staged_pipeline_slot_reuse(ahead):
    """Six requests with distinct data and alternating shapes (the rotating
    staging / output slots are re-used and re-allocated), staged ``ahead``
    requests before their compute (more than the two steady-state slots:
    pending slots are never overwritten); every result equals the device path."""
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    g = torch.Generator().manual_seed(11)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).pin_memory()
    reqs = []
    for i in range(6):
        T = (3000, 1100)[(i // 2) % 2]
        plan = plan_full_prefill([SequenceSpec(1, 0, T)], 1)
        reqs.append((plan, [mk(T, hq, D)], [mk(T, hkv, D)], [mk(T, hkv, D)]))
    ring = RingAttention(_LocalComm(0, 1))
    refs = []
    for plan, qh, kh, vh in reqs:
        r = ring.pass_kv_prefill(plan, RankKvCache(hkv, D, capacity_tokens=256),
                                 materialize_rank_block(plan, 0, [qh[0].cuda()]),
                                 materialize_rank_block(plan, 0, [kh[0].cuda()]),
                                 materialize_rank_block(plan, 0, [vh[0].cuda()]), cfg)
        refs.append((r.output.data.cpu(), r.lse.cpu()))
    torch.cuda.synchronize()
    dev = torch.device("cuda")
    staged = [ring.stage_host_inputs(*reqs[j], cfg, dev) for j in range(min(ahead, len(reqs)))]
    outs = []
    for i, (plan, qh, kh, vh) in enumerate(reqs):
        S = plan.total_query_slots()
        oh = torch.full((S, hq, D), float("nan")).pin_memory()
        lh = torch.full((S, hq), float("nan")).pin_memory()
        ring.pass_kv_prefill_host(plan, RankKvCache(hkv, D, capacity_tokens=256), qh, kh, vh, cfg, oh, lh,
                                  staged=staged[i], join=False)
        outs.append((oh, lh))
        if i + ahead < len(reqs):
            staged.append(ring.stage_host_inputs(*reqs[i + ahead], cfg, dev))
    ring.join_host_copies()
    torch.cuda.synchronize()
    for i, ((oh, lh), (ro, rl)) in enumerate(zip(outs, refs)):
        assert torch.equal(oh, ro) and torch.equal(lh, rl), i


@pytest.mark.parametrize("n_sub", [1, 3])
def test_host_stream_token_order_outputs(n_sub):
    """Token-ordered host outputs (per-sequence lists): equal to the device
    path's slot-ordered result scattered to token order
    (sharding.scatter_rank_block), bitwise, with ragged fused sequences whose
    chunks end in padding slots."""
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import (SequenceSpec, materialize_rank_block, plan_full_prefill,
                                                scatter_rank_block)

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    g = torch.Generator().manual_seed(2)
    lens = [1501, 699]
    plan = plan_full_prefill([SequenceSpec(3, 0, lens[0]), SequenceSpec(8, 0, lens[1])], 1)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).pin_memory()
    qh, kh, vh = ([mk(n, h, D) for n in lens] for h in (hq, hkv, hkv))
    ring = RingAttention(_LocalComm(0, 1))
    ref = ring.pass_kv_prefill(plan, RankKvCache(hkv, D, capacity_tokens=256),
                               materialize_rank_block(plan, 0, [t.cuda() for t in qh]),
                               materialize_rank_block(plan, 0, [t.cuda() for t in kh]),
                               materialize_rank_block(plan, 0, [t.cuda() for t in vh]), cfg)
    want_o = [torch.empty(n, hq, D, device="cuda") for n in lens]
    want_l = [torch.empty(n, hq, device="cuda") for n in lens]
    scatter_rank_block(plan, 0, ref.output.data, want_o)
    scatter_rank_block(plan, 0, ref.lse, want_l)
    out_h = [torch.full((n, hq, D), float("nan")).pin_memory() for n in lens]
    lse_h = [torch.full((n, hq), float("nan")).pin_memory() for n in lens]
    ring.pass_kv_prefill_host(plan, RankKvCache(hkv, D, capacity_tokens=256), qh, kh, vh, cfg, out_h, lse_h,
                              n_sub=n_sub)
    torch.cuda.synchronize()
    for i in range(2):
        assert torch.equal(out_h[i], want_o[i].cpu())
        assert torch.equal(lse_h[i], want_l[i].cpu())


def test_host_stream_bf16_outputs():
    """bf16 host outputs: O is the device fp32 result cast round-to-nearest-even
    (rcp_cast_f32_bf16), bitwise equal to torch's cast; LSE stays fp32."""
    from paper_2411_01783_b200.attention import GqaConfig
    from paper_2411_01783_b200.kv_cache import RankKvCache
    from paper_2411_01783_b200.ring import RingAttention, _LocalComm
    from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill

    hq, hkv, D = 8, 2, 128
    cfg = GqaConfig(hq, hkv, D)
    g = torch.Generator().manual_seed(3)
    lens = [1300]
    plan = plan_full_prefill([SequenceSpec(0, 0, lens[0])], 1)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).pin_memory()
    qh, kh, vh = ([mk(n, h, D) for n in lens] for h in (hq, hkv, hkv))
    ring = RingAttention(_LocalComm(0, 1))
    ref = ring.pass_kv_prefill(plan, RankKvCache(hkv, D, capacity_tokens=256),
                               *(materialize_rank_block(plan, 0, [t.cuda() for t in x]) for x in (qh, kh, vh)), cfg)
    S = ref.output.n_tokens
    out_h = torch.empty((S, hq, D), dtype=torch.bfloat16).pin_memory()
    lse_h = torch.empty((S, hq), dtype=torch.float32).pin_memory()
    ring.pass_kv_prefill_host(plan, RankKvCache(hkv, D, capacity_tokens=256), qh, kh, vh, cfg, out_h, lse_h, n_sub=2)
    torch.cuda.synchronize()
    assert torch.equal(out_h, ref.output.data.to(torch.bfloat16).cpu())
    assert torch.equal(lse_h, ref.lse.cpu())
