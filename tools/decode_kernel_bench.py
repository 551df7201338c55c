"""Decode kernel alone (rcp_decode_attn / rcp_decode_attn_fp8: split-KV +
combine), CUDA-event timed over back-to-back launches; K/V larger than L2 at
the default sizes.  One JSON line per (kv dtype, batch):

    python tools/decode_kernel_bench.py --context 262144 --batch 1 4 16 --hq 128 --hkv 8

hbm_gbs = algorithmic bytes (K + V rows read once, q, fp32 o/lse) / time.
Tuning: RCP_DEC_CTA_TARGET / RCP_DEC_CTA_TARGET_FP8 in the environment."""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_01783_b200 import _lib  # noqa: E402
from paper_2411_01783_b200.attention import GqaConfig  # noqa: E402
from paper_2411_01783_b200.ring import _cuda_decode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=262144)
    ap.add_argument("--batch", type=int, nargs="*", default=[1, 4, 16])
    ap.add_argument("--hq", type=int, default=128)
    ap.add_argument("--hkv", type=int, default=8)
    ap.add_argument("--dtypes", nargs="*", default=["bf16", "e4m3"])
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda")
    cfg = GqaConfig(args.hq, args.hkv, 128)
    g = torch.Generator(device=dev).manual_seed(0)
    for B in args.batch:
        rows = B * args.context
        for dt in args.dtypes:
            if dt == "e4m3":
                k = torch.randint(0, 0x7E, (rows, args.hkv, 128), dtype=torch.uint8, device=dev, generator=g)
                v = torch.randint(0, 0x7E, (rows, args.hkv, 128), dtype=torch.uint8, device=dev, generator=g)
                sc = (torch.full((args.hkv,), 0.01, device=dev), torch.full((args.hkv,), 0.01, device=dev))
                kw = {"scales": sc}
                elem = 1
            else:
                k = torch.randn(rows, args.hkv, 128, dtype=torch.bfloat16, device=dev, generator=g)
                v = torch.randn(rows, args.hkv, 128, dtype=torch.bfloat16, device=dev, generator=g)
                kw = {}
                elem = 2
            q = torch.randn(B, args.hq, 128, dtype=torch.bfloat16, device=dev, generator=g)
            starts = torch.arange(B, dtype=torch.int64, device=dev) * args.context
            lens = torch.full((B,), args.context, dtype=torch.int64, device=dev)
            out = torch.empty(B, args.hq, 128, dtype=torch.float32, device=dev)
            lse = torch.empty(B, args.hq, dtype=torch.float32, device=dev)
            need = _lib.load().rcp_decode_workspace_bytes(B, args.hq, args.context)
            ws = torch.empty(need, dtype=torch.uint8, device=dev)
            run = lambda: _cuda_decode(q, k, v, starts, lens, args.context, cfg, out, lse, ws, **kw)  # noqa: E731
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.iters):
                run()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / args.iters
            nbytes = 2 * rows * args.hkv * 128 * elem + B * args.hq * 128 * (2 + 4) + B * args.hq * 4
            print(json.dumps({"kernel": "decode", "kv_dtype": dt, "batch": B, "context": args.context,
                              "n_q_heads": args.hq, "n_kv_heads": args.hkv, "ms": ms,
                              "keys_per_s": rows / (ms * 1e-3), "hbm_gbs": nbytes / (ms * 1e-3) / 1e9,
                              "cta_target": os.environ.get("RCP_DEC_CTA_TARGET_FP8" if dt == "e4m3"
                                                           else "RCP_DEC_CTA_TARGET", "default")}), flush=True)
            del k, v
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
