"""Seeded inputs shared by make_golden.py and the tests (no reference import,
so the tests can regenerate a fixture's inputs on the GPU box)."""

from __future__ import annotations

import numpy as np


def bf16_exact(x: np.ndarray) -> np.ndarray:
    """Round float32 to bf16 (round-to-nearest-even) and back to float32."""
    x = np.asarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def sampled_inputs(seed, T, hq, hkv, rows):
    """Inputs of a sampled-row case, regenerated from the seed by the tests
    (numpy PCG64 streams are stable), so the fixture stores outputs only."""
    rng = np.random.default_rng(seed)
    k = bf16_exact(rng.standard_normal((T, hkv, 128)).astype(np.float32))
    v = bf16_exact(rng.standard_normal((T, hkv, 128)).astype(np.float32))
    q = bf16_exact(rng.standard_normal((len(rows), hq, 128)).astype(np.float32))
    return q, k, v
