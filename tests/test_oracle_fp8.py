"""Oracle pins for the fp8 e4m3 Q-token format (NEXT-2; "FP8").

The e4m3 code table and its round-to-nearest-even / satfinite encoder are checked
against the format's definition (OCP FP8 E4M3: bias 7, 3 mantissa bits, no infinities,
S.1111.111 = NaN), hand-computed ties, and torch's independent float8_e4m3fn cast."""
import numpy as np
import pytest
import torch

import oracle as O


def test_e4m3_table_definition():
    t = O.E4M3
    assert len(t) == 127 and np.all(np.diff(t) > 0)
    assert t[0x00] == 0.0 and t[0x01] == 2.0 ** -9 and t[0x07] == 7 * 2.0 ** -9
    assert t[0x08] == 2.0 ** -6                 # smallest normal
    assert t[0x38] == 1.0 and t[0x30] == 0.5 and t[0x40] == 2.0
    assert t[0x7E] == 448.0 == O.E4M3_MAX       # 0x7F is NaN


@pytest.mark.parametrize("x,code", [
    (1.0, 0x38), (0.5, 0x30), (-2.0, 0xC0), (448.0, 0x7E), (1000.0, 0x7E), (-1e9, 0xFE),
    (1.0625, 0x38),            # tie between 1.0 (0x38) and 1.125 (0x39): even code
    (1.1875, 0x3A),            # tie between 1.125 (0x39) and 1.25 (0x3A): even code
    (2.0 ** -10, 0x00),        # tie between 0 and the smallest subnormal
    (3 * 2.0 ** -10, 0x02),    # tie between 2^-9 (0x01) and 2^-8 (0x02)
    (-0.0, 0x80), (0.0, 0x00),
    (1.07, 0x39), (240.0, 0x77), (464.0, 0x7E),
])
def test_e4m3_encode_hand_cases(x, code):
    assert int(O.e4m3_encode(np.float32(x))) == code


def test_e4m3_matches_torch_cast():
    g = torch.Generator().manual_seed(5)
    x = torch.cat([torch.randn(20000, generator=g) * s for s in (1e-3, 0.1, 1.0, 30.0, 200.0)])
    x = x.clamp(-448, 448)
    ref = x.to(torch.float8_e4m3fn).view(torch.uint8).numpy().astype(np.int64)
    got = O.e4m3_encode(x.numpy().astype(np.float32))
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(O.e4m3_decode(got), x.to(torch.float8_e4m3fn).to(torch.float64).numpy())


@pytest.mark.parametrize("g", [128, 32, 16])
def test_fp8_quantize_error_bound(g):
    """|x - x̃| <= half an e4m3 step at |x/s|: 2^-4 |x| in the normal range, s·2^-10 below."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        x = (rng.standard_normal(128) * rng.uniform(0.01, 20)).astype(np.float32)
        x[:2] *= 8
        c, s, z = O.quantize(x, 8, g, "fp8")
        assert np.all(z == 0)
        xt = O.dequantize(c, s, z, g, "fp8")
        sv = np.repeat(s.astype(np.float64), g)
        bound = np.maximum(np.abs(x) * 2.0 ** -4, sv * 2.0 ** -10) * (1 + 1e-6)
        assert np.all(np.abs(xt - x) <= bound)
        # the group maximum lands exactly on 448 (or within fp32 rounding of s)
        amax = np.abs(x.reshape(-1, g)).max(axis=1)
        np.testing.assert_allclose(amax / s, 448.0, rtol=1e-6)


def test_fp8_zero_group_and_promotion():
    x = np.zeros(16, dtype=np.float32)
    c, s, z = O.quantize(x, 8, 16, "fp8")
    assert np.all(c == 0) and s[0] == 1.0
    # promotion: bf16_rne(f32(e4m3(code) * s)): exact for these values
    y = np.array([1.0, -0.5, 448.0, 3.0] * 4, dtype=np.float32)
    c, s, z = O.quantize(y, 8, 16, "fp8")
    np.testing.assert_array_equal(O.promote(c, s, z, 16, "fp8"), y.astype(np.float64))
