"""CPU: the e4m3 restatement in the oracle (encode / decode / calibration /
quantise / dequantise) pinned against torch.float8_e4m3fn, the one
independent e4m3 implementation in this image (the reference itself has no
FP8 path: this mode is SURVEY §8f rank 4)."""

import numpy as np
import pytest

from oracle import ringcp_oracle as orc


def _torch_e4m3(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()


def test_encode_every_bf16_value_in_range():
    x = (np.arange(1 << 16, dtype=np.uint32) << 16).view(np.float32)
    x = x[np.isfinite(x) & (np.abs(x) <= 448)]
    np.testing.assert_array_equal(orc.e4m3_encode(x), _torch_e4m3(x))


def test_encode_random_float32_and_ties():
    rng = np.random.default_rng(0)
    y = (rng.standard_normal(400_000) * np.exp(rng.uniform(-14, 6, 400_000))).astype(np.float32)
    y = y[np.abs(y) <= 448]
    np.testing.assert_array_equal(orc.e4m3_encode(y), _torch_e4m3(y))
    # exact midpoints between neighbours round to the even mantissa
    grid = orc.e4m3_decode(np.arange(0x7E, dtype=np.uint8))
    mids = ((grid[:-1] + grid[1:]) / 2).astype(np.float32)
    np.testing.assert_array_equal(orc.e4m3_encode(mids), _torch_e4m3(mids))
    assert np.all(orc.e4m3_encode(mids) % 2 == 0)


def test_saturation_nan_and_signed_zero():
    big = np.array([448.0, 449.0, 463.9, 464.0, 1e6, np.inf, -1e6, -np.inf], np.float32)
    np.testing.assert_array_equal(orc.e4m3_encode(big), [0x7E] * 6 + [0xFE] * 2)
    assert orc.e4m3_encode(np.array([np.nan], np.float32))[0] == 0x7F
    np.testing.assert_array_equal(orc.e4m3_encode(np.array([0.0, -0.0, -1e-9], np.float32)), [0x00, 0x80, 0x80])


def test_decode_every_byte():
    import torch

    b = np.arange(256, dtype=np.uint8)
    want = torch.from_numpy(b).view(torch.float8_e4m3fn).float().numpy().astype(np.float64)
    got = orc.e4m3_decode(b)
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    np.testing.assert_array_equal(got[ok], want[ok])
    # encode(decode(b)) is the identity on every non-NaN byte (except -0 -> 0x80 kept)
    np.testing.assert_array_equal(orc.e4m3_encode(got[ok].astype(np.float32)), b[ok])


@pytest.mark.parametrize("H", [1, 8])
def test_quantize_round_trip_error_bound(H):
    rng = np.random.default_rng(H)
    x = (rng.standard_normal((300, H, 128)) * rng.uniform(0.1, 30, (1, H, 1))).astype(np.float32)
    s = orc.e4m3_scale(x, H)
    assert s.dtype == np.float32 and s.shape == (H,)
    amax = np.abs(x).max(axis=(0, 2))
    ideal = (amax / np.float32(448)).astype(np.float32)
    assert np.all(np.log2(s) == np.round(np.log2(s)))  # powers of two
    assert np.all((s >= ideal) & (s < 2 * ideal))       # the smallest ones covering absmax
    q = orc.quantize_e4m3(x, s)
    back = orc.dequantize_e4m3(q, s)
    # relative error <= 2^-4 for normals; absolute <= 2^-10 * scale in the subnormal range
    tol = np.maximum(np.abs(x) * 2.0 ** -4, 2.0 ** -10 * s.reshape(1, -1, 1))
    assert np.all(np.abs(back - x) <= tol)
    # nothing saturates: the absmax element keeps its value within e4m3 rounding
    for h in range(H):
        assert np.abs(back[:, h]).max() == pytest.approx(float(amax[h]), rel=2.0 ** -4)
    # with a power-of-two scale the dequantised values are exact in bf16
    np.testing.assert_array_equal(orc.dequantize_e4m3_bf16(q, s), back.astype(np.float32))
    # bf16 dequantisation equals rounding the fp32 product (any scale)
    s3 = (s * np.float32(1.37)).astype(np.float32)
    np.testing.assert_array_equal(orc.dequantize_e4m3_bf16(q, s3),
                                  orc.f32_to_bf16_values((orc.e4m3_decode(q).astype(np.float32)
                                                          * s3.reshape(1, -1, 1)).astype(np.float32)))
