"""Loaders for the committed golden fixtures (tests/golden/*.npz, *.json)."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import ringcp_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def npz(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def js(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def block(z, key) -> orc.Blk:
    return orc.Blk(z[f"{key}__data"], z[f"{key}__pos"], z[f"{key}__valid"], z[f"{key}__seq"])


def gqa_case(z, name):
    hq, hkv, d = (int(x) for x in z[f"{name}__cfg"])
    return dict(
        q=block(z, f"{name}__q"), k=block(z, f"{name}__k"), v=block(z, f"{name}__v"),
        hq=hq, hkv=hkv, d=d, scale=float(z[f"{name}__scale"]),
        out=z[f"{name}__out"], lse=z[f"{name}__lse"], pairs=int(z[f"{name}__pairs"]))


# bf16 tolerances from the north star: |dO| <= 2e-2, |dLSE| <= 1e-3
O_TOL = 2e-2
LSE_TOL = 1e-3


def lse_err(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    ninf_g, ninf_w = np.isneginf(got), np.isneginf(want)
    if not np.array_equal(ninf_g, ninf_w):
        return float("inf")
    fin = ~ninf_w
    return float(np.abs(got[fin] - want[fin]).max()) if fin.any() else 0.0
