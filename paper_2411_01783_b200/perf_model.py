"""pass-KV / pass-Q selection heuristic and the cost formulas behind it.

Reference: SPEC.md:305-437 (module ``perf_model``, not shipped in pkg/) and
PAPER.md §3.3 — Eq. 1 (:155-158), Eq. 2 (:203-206), Eq. 3 (:216-219), Alg. 1
(:225-237), Table 2 (comm bytes / FLOPs), Table 4-5 (:500-587, calibration
data for the refined, All2All-aware rule of Appendix C as restated by
SPEC.md:375).  Host-only arithmetic; the B200 profile takes its compute and
link constants from MEASURED_PEAKS.json / the measured NVLink copy bandwidth.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, replace

__all__ = [
    "CostModel",
    "PrefillShape",
    "attention_flops",
    "b200_profile",
    "calibrate_b200",
    "choose_strategy",
    "comm_bytes",
    "pass_kv_overlap_min_T",
    "pass_q_overlap_min_ctx",
    "predict_step_times",
    "profile",
    "size_threshold",
]


@dataclass(frozen=True)
class CostModel:
    """Model + hardware constants.  ``peak_compute`` C is
    FLOP/s per CP rank, ``bandwidth`` BW bytes/s per rank link, ``elem_size`` e
    bytes, ``n_ranks`` N; All2All time is affine in bytes."""

    n_query_heads: int
    n_kv_heads: int
    head_dim: int
    peak_compute: float
    bandwidth: float
    elem_size: int = 2
    n_ranks: int = 1
    sendrecv_latency_s: float = 0.0
    a2a_base_s: float = 0.0
    a2a_per_byte_s: float | None = None  # None -> 1 / bandwidth

    def __post_init__(self):
        for name in ("n_query_heads", "n_kv_heads", "head_dim", "peak_compute", "bandwidth",
                     "elem_size", "n_ranks"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @property
    def model_dim(self) -> int:
        """D = N_H * D_H (Table 2's D)."""
        return self.n_query_heads * self.head_dim


@dataclass(frozen=True)
class PrefillShape:
    """New tokens T and cached tokens P of one prefill."""

    new_len: int
    cached_len: int = 0

    def __post_init__(self):
        if self.new_len < 0 or self.cached_len < 0 or self.new_len + self.cached_len < 1:
            raise ValueError("need T >= 0, P >= 0 and T + P >= 1")

    @property
    def miss_rate(self) -> float:
        return self.new_len / (self.new_len + self.cached_len)


def comm_bytes(shape: PrefillShape, m: CostModel, kind: str) -> float:
    """Table 2: Q -> T·D·e; KV -> 2·(T+P)·D·(N_KV/N_H)·e."""
    T, P, D, e = shape.new_len, shape.cached_len, m.model_dim, m.elem_size
    if kind == "Q":
        return float(T * D * e)
    if kind == "KV":
        return 2.0 * (T + P) * D * (m.n_kv_heads / m.n_query_heads) * e
    raise ValueError(f"unknown message kind {kind!r}")


def attention_flops(shape: PrefillShape, m: CostModel) -> float:
    """Table 2: 4·T·D·(T + P)."""
    return 4.0 * shape.new_len * m.model_dim * (shape.new_len + shape.cached_len)


def size_threshold(m: CostModel) -> float:
    """Eq. 1: pass-Q moves fewer bytes iff miss rate <= 2·N_KV/N_H."""
    return 2.0 * m.n_kv_heads / m.n_query_heads


def pass_kv_overlap_min_T(m: CostModel) -> float:
    """Eq. 2: ring pass-KV hides its traffic iff T >= N·C·N_KV·e / (2·N_H·BW)."""
    return m.n_ranks * m.peak_compute * m.n_kv_heads * m.elem_size / (
        2.0 * m.n_query_heads * m.bandwidth)


def pass_q_overlap_min_ctx(m: CostModel) -> float:
    """Eq. 3: ring pass-Q hides its traffic iff T + P >= N·e·C / (4·BW)."""
    return m.n_ranks * m.elem_size * m.peak_compute / (4.0 * m.bandwidth)


def predict_step_times(shape: PrefillShape, m: CostModel):
    """Per ring step: (sendrecv_kv_s, sendrecv_q_s, attn_s, a2a_s).

    A rank's KV message carries 1/N of the K/V bytes, the Q message 1/N of the
    Q bytes; each step computes 1/N² of the attention FLOPs; the All2All moves
    (N-1)/N of a rank's partial outputs (T/N rows of D values + LSE)."""
    n = m.n_ranks
    kv = comm_bytes(shape, m, "KV") / n
    q = comm_bytes(shape, m, "Q") / n
    sendrecv_kv = kv / m.bandwidth + m.sendrecv_latency_s
    sendrecv_q = q / m.bandwidth + m.sendrecv_latency_s
    attn = attention_flops(shape, m) / (n * n) / m.peak_compute
    a2a_bytes = (n - 1) / n * (shape.new_len / n) * (m.model_dim * m.elem_size + 4 * m.n_query_heads)
    per_byte = m.a2a_per_byte_s if m.a2a_per_byte_s is not None else 1.0 / m.bandwidth
    a2a = (m.a2a_base_s + a2a_bytes * per_byte) if n > 1 else 0.0
    return sendrecv_kv, sendrecv_q, attn, a2a


def choose_strategy(shape: PrefillShape, m: CostModel, refined: bool = False) -> str:
    """Alg. 1: pass-KV iff T >= Eq. 2 or miss >= Eq. 1
    (ties -> pass-KV); else pass-Q.  ``refined`` (Appendix C as restated in
    SPEC.md:375) instead compares the exposed pass-KV ring time
    (N-1)·max(0, SendRecv_KV - Attn) with pass-Q's exposed ring time plus its
    All2All and picks the smaller (ties -> pass-KV)."""
    if m.n_ranks == 1:
        return "pass_kv"
    if refined:
        kv_s, q_s, attn, a2a = predict_step_times(shape, m)
        n1 = m.n_ranks - 1
        exposed_kv = n1 * max(0.0, kv_s - attn)
        exposed_q = n1 * max(0.0, q_s - attn) + a2a
        return "pass_kv" if exposed_kv <= exposed_q else "pass_q"
    if shape.new_len >= pass_kv_overlap_min_T(m) or shape.miss_rate >= size_threshold(m):
        return "pass_kv"
    return "pass_q"


# ---------------------------------------------------------------------- profiles
# Llama3-405B attention geometry (§4.1: 128 Q heads, 8 KV heads, D_H 128).
LLAMA3_405B = dict(n_query_heads=128, n_kv_heads=8, head_dim=128)
LLAMA3_8B = dict(n_query_heads=32, n_kv_heads=8, head_dim=128)

# Paper hardware (per CP rank = one 8xH100 node, TP8).  "gtt": 400 Gb/s RDMA per
# GPU; "gti": 100 Gb/s TCP per GPU.  The simple profile uses the
# constants under which Alg. 1 is analysed (C = 8e14, BW = 5e10);
# the calibrated one fits Table 5: effective per-node
# compute from the Attn column, link from SendRecv, affine All2All from the two
# All2All rows (424 us at 2.5 %, 1023 us at 10 % miss).
_PROFILES = {
    "gtt-h100": dict(peak_compute=8e14, bandwidth=5e10),
    "gti-h100": dict(peak_compute=8e14, bandwidth=1.25e10),
    "gtt-h100-calibrated": dict(peak_compute=4.05e15, bandwidth=2.09e11, a2a_base_s=224e-6,
                                a2a_per_byte_s=1.0e-11),
}


def profile(name: str, model=LLAMA3_405B, n_ranks: int = 4) -> CostModel:
    if name == "b200-nvl":
        return b200_profile(model, n_ranks)
    if name not in _PROFILES:
        raise ValueError(f"unknown profile {name!r}; known: {sorted(_PROFILES) + ['b200-nvl']}")
    return CostModel(**model, n_ranks=n_ranks, **_PROFILES[name])


def b200_profile(model=LLAMA3_405B, n_ranks: int = 8, attn_efficiency: float | None = None,
                 link_gbs: float = 770.0) -> CostModel:
    """B200 / NVLink-5 constants without a measurement in this run: C =
    measured bf16 peak x attention efficiency (default 0.74: K1's measured
    fraction of the burst peak, profiles/r02_*), BW = measured NVLink copy per
    direction (B200_PROFILING.md: 770 GB/s).  ``calibrate_b200`` measures all
    of them on the box instead (what TurnRunner(calibrate=True) and
    tools/bench_configs.py --calibrate use)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    peak = 1590e12
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["bf16_tflops"]) * 1e12
    except Exception:
        pass
    eff = 0.74 if attn_efficiency is None else attn_efficiency
    return CostModel(**model, n_ranks=n_ranks, peak_compute=peak * eff, bandwidth=link_gbs * 1e9,
                     sendrecv_latency_s=15e-6, a2a_base_s=30e-6)


def with_ranks(m: CostModel, n_ranks: int) -> CostModel:
    return replace(m, n_ranks=n_ranks)


def calibrate_b200(comm, model=LLAMA3_405B, n_ranks: int | None = None, device=None, step_tokens: int = 8192,
                   link_bytes: int = 256 << 20, reps: int = 5):
    """On-box calibration of the B200 cost model (
    PAPER.md:556-564): measure, in THIS run, the constants Alg. 1 and the
    refined rule need instead of assuming them.

    * C: TF/s of one attention launch at a ring-step shape (``step_tokens``
      queries x keys, causal, the model's heads) — the kernel's sustained rate;
    * BW and SendRecv latency: one ring exchange (``comm.exchange``) of
      ``link_bytes`` and of 4 KB, per direction;
    * All2All: affine fit of ``comm.all_to_all`` at two sizes.

    Collective over the ring (every rank calls it).  With one rank the link
    terms keep the measured NVLink copy figure (770 GB/s).  Returns
    (CostModel, dict of the measurements)."""
    import statistics

    import torch

    from . import _lib
    from .attention import attend_into

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = n_ranks if n_ranks is not None else getattr(comm, "world", 1)
    hq, hkv, d = model["n_query_heads"], model["n_kv_heads"], model["head_dim"]

    def timed(fn, inner=1):
        """Seconds per call: median over ``reps`` of ``inner`` back-to-back calls
        (transfers are issued in a row, as a ring issues them, so per-call host
        launch cost is not counted as link time)."""
        for _ in range(2):
            fn()
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(inner):
                fn()
            e.record()
            torch.cuda.synchronize(dev)
            ts.append(s.elapsed_time(e) * 1e-3 / inner)
        return statistics.median(ts)

    T = step_tokens
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((T, hq, d), generator=g, device=dev, dtype=torch.bfloat16)
    k = torch.randn((T, hkv, d), generator=g, device=dev, dtype=torch.bfloat16)
    v = torch.randn((T, hkv, d), generator=g, device=dev, dtype=torch.bfloat16)
    pos = torch.arange(T, device=dev, dtype=torch.int32)
    seq = torch.zeros(T, device=dev, dtype=torch.int32)
    out = torch.empty((T, hq, d), device=dev, dtype=torch.float32)
    lse = torch.empty((T, hq), device=dev, dtype=torch.float32)
    ws = torch.empty(_lib.load().rcp_attn_workspace_bytes(T, T), dtype=torch.uint8, device=dev)
    t_attn = timed(lambda: attend_into(q, (pos, seq), k, v, (pos, seq), hq, hkv, d ** -0.5, out, lse,
                                       _lib.MODE_OVERWRITE, workspace=ws))
    flops = 4.0 * d * hq * T * (T + 1) / 2
    meas = {"attn_tflops": flops / t_attn / 1e12, "attn_shape": f"{T}x{T} causal, {hq}/{hkv} heads"}
    bw, lat, a2a_base, a2a_per_byte = 770e9, 15e-6, 30e-6, None
    if n > 1:
        big = torch.empty(link_bytes, dtype=torch.uint8, device=dev)
        big_r = torch.empty_like(big)
        small = torch.empty(4096, dtype=torch.uint8, device=dev)
        small_r = torch.empty_like(small)
        t_big = timed(lambda: comm.wait(comm.exchange(big, big_r)), inner=8)
        t_small = timed(lambda: comm.wait(comm.exchange(small, small_r)), inner=8)
        lat = t_small
        bw = link_bytes / max(t_big - t_small, 1e-9)
        sizes = (1 << 20, 16 << 20)
        ts = []
        for sz in sizes:
            sends = [torch.empty(sz // n, dtype=torch.uint8, device=dev) for _ in range(n)]
            recvs = [torch.empty_like(x) for x in sends]
            ts.append(timed(lambda: comm.wait(comm.all_to_all(sends, recvs)), inner=4))
        per_rank_bytes = [(n - 1) * sz // n for sz in sizes]
        a2a_per_byte = max((ts[1] - ts[0]) / (per_rank_bytes[1] - per_rank_bytes[0]), 0.0)
        a2a_base = max(ts[0] - a2a_per_byte * per_rank_bytes[0], 0.0)
        # one consistent set of constants on every rank: the slowest rank's
        vals = torch.tensor([meas["attn_tflops"], bw, lat, a2a_base, a2a_per_byte], dtype=torch.float64, device=dev)
        lo = vals.clone()
        comm.dist.all_reduce(lo, op=comm.dist.ReduceOp.MIN, group=comm.group)
        hi = vals.clone()
        comm.dist.all_reduce(hi, op=comm.dist.ReduceOp.MAX, group=comm.group)
        meas["attn_tflops"], bw = float(lo[0]), float(lo[1])
        lat, a2a_base, a2a_per_byte = float(hi[2]), float(hi[3]), float(hi[4])
    meas.update({"link_gbs": bw / 1e9, "sendrecv_latency_us": lat * 1e6, "a2a_base_us": a2a_base * 1e6,
                 "a2a_per_byte_ns": None if a2a_per_byte is None else a2a_per_byte * 1e9})
    m = CostModel(**model, n_ranks=n, peak_compute=meas["attn_tflops"] * 1e12, bandwidth=bw,
                  sendrecv_latency_s=lat, a2a_base_s=a2a_base, a2a_per_byte_s=a2a_per_byte)
    return m, meas
