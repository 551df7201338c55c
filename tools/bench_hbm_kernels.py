"""Achieved HBM bandwidth of the byte-moving kernels (K0 shard gather / scatter,
K2 merge, the e4m3 KV quantise / dequantise rows).

  python tools/bench_hbm_kernels.py

K2 rcp_merge_attn: fold N fp32 partials [T, Hq, 128] + LSE [T, Hq] (the pass-Q
All2All merge), sized as SURVEY §8(a5): 405B shape, 128K CP8 -> T = 16384
query slots per rank, Hq = 128, N = 8 partials.  Algorithmic bytes =
N·T·Hq·(4·128 + 4) read + T·Hq·(4·128 + 4) written.
K0 rcp_shard_gather (materialize_rank_block on device): this rank's two
chunks of a 1M-token sequence at CP8 -> 262144 slots x 128 heads x 128 dims
bf16 (8.6 GB read + 8.6 GB written... per SURVEY a7's cfg3 Q shard).
CUDA events around each launch, median of 10 after 3 warm-ups; peak =
MEASURED_PEAKS.json HBM copy bandwidth.
"""

import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2411_01783_b200.attention import merge_rows_into  # noqa: E402
from paper_2411_01783_b200.sharding import SequenceSpec, materialize_rank_block, plan_full_prefill  # noqa: E402


def timed(fn, n=10, w=3):
    for _ in range(w):
        fn()
    ts = []
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return statistics.median(ts)


def main():
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6466.1
    out = {}
    # K2 merge
    T, H, D, N = 16384, 128, 128, 8
    o_parts = [torch.randn(T, H, D, device="cuda") for _ in range(N)]
    l_parts = [torch.randn(T, H, device="cuda") for _ in range(N)]
    o = torch.empty(T, H, D, device="cuda")
    lse = torch.empty(T, H, device="cuda")
    ms = timed(lambda: merge_rows_into(o_parts, l_parts, o, lse))
    nbytes = (N + 1) * T * H * (4 * D + 4)
    out["K2_merge"] = dict(shape=f"{N} partials x [{T},{H},{D}] fp32", ms=ms, bytes=nbytes,
                           gbs=nbytes / ms / 1e6, frac=nbytes / ms / 1e6 / peak)
    del o_parts, l_parts, o, lse
    torch.cuda.empty_cache()
    # K0 shard gather: CP8 rank block of a 1M-token sequence, 405B Q shape
    Tseq, n_ranks = 1 << 20, 8
    plan = plan_full_prefill([SequenceSpec(0, 0, Tseq)], n_ranks)
    q = torch.randn(Tseq, H, D, device="cuda", dtype=torch.bfloat16)
    ms = timed(lambda: materialize_rank_block(plan, 3, [q]))
    slots = plan.total_query_slots()
    nbytes = 2 * slots * H * D * 2 + slots * 8
    out["K0_shard_gather"] = dict(shape=f"rank 3 of CP8, 1M tokens, [{slots},{H},{D}] bf16", ms=ms, bytes=nbytes,
                                  gbs=nbytes / ms / 1e6, frac=nbytes / ms / 1e6 / peak)
    # K0 shard scatter (the inverse): the same rank block back to token order
    from paper_2411_01783_b200.sharding import scatter_rank_block

    blk = materialize_rank_block(plan, 3, [q]).data
    dst = torch.empty_like(q)
    ms = timed(lambda: scatter_rank_block(plan, 3, blk, [dst]))
    valid = plan.new_token_count(0, 3)
    nbytes = 2 * valid * H * D * 2
    out["K0_shard_scatter"] = dict(shape=f"rank 3 of CP8, 1M tokens, {valid} valid slots x [{H},{D}] bf16", ms=ms,
                                   bytes=nbytes, gbs=nbytes / ms / 1e6, frac=nbytes / ms / 1e6 / peak)
    del q, blk, dst
    torch.cuda.empty_cache()
    # e4m3 KV rows: quantise (bf16 -> e4m3) and dequantise (e4m3 -> bf16), 1M rows x 8 heads x 128
    from paper_2411_01783_b200 import _lib

    lib = _lib.load()
    R, HK = 1 << 20, 8
    x = torch.randn(R, HK, D, device="cuda", dtype=torch.bfloat16)
    e8 = torch.empty(R, HK, D, device="cuda", dtype=torch.uint8)
    back = torch.empty_like(x)
    sc = torch.full((HK,), 0.01, device="cuda")
    row = HK * D
    ms = timed(lambda: _lib.check(lib.rcp_kv_quantize_e4m3(e8.data_ptr(), row, 0, x.data_ptr(), row, R, HK, D,
                                                           sc.data_ptr(), _lib.stream_handle())))
    nbytes = R * row * 3
    out["kv_quantize_e4m3"] = dict(shape=f"[{R},{HK},{D}] bf16 -> e4m3", ms=ms, bytes=nbytes,
                                   gbs=nbytes / ms / 1e6, frac=nbytes / ms / 1e6 / peak)
    ms = timed(lambda: _lib.check(lib.rcp_kv_dequantize_e4m3(back.data_ptr(), row, e8.data_ptr(), row, R, HK, D,
                                                             sc.data_ptr(), _lib.stream_handle())))
    out["kv_dequantize_e4m3"] = dict(shape=f"[{R},{HK},{D}] e4m3 -> bf16", ms=ms, bytes=nbytes,
                                     gbs=nbytes / ms / 1e6, frac=nbytes / ms / 1e6 / peak)
    out["peak_gbs"] = peak
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
