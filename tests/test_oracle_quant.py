"""Pins for the oracle's group quantizer, dequantizer and promotion (R23, R24)."""
import json
import os

import numpy as np
import pytest
import torch
from hypothesis import given, settings, strategies as st

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def bf16_vals(rng, n, scale=1.0):
    return torch.tensor(rng.normal(size=n) * scale, dtype=torch.float32).to(torch.bfloat16).double().numpy()


def test_spec_symmetric_int8_example():
    g = GOLD["quantize_sym_int8"]
    codes, s, z = O.quantize(np.array(g["x"]), 8, 3, "sym")
    assert codes.tolist() == g["codes"]
    assert s[0] == np.float32(1.0) / np.float32(127.0) and z[0] == 0.0
    np.testing.assert_allclose(O.dequantize(codes, s, z, 3), g["dequant"], rtol=1e-6)


def test_zero_and_constant_groups():
    c, s, z = O.quantize(np.zeros(16), 4, 16, "sym")
    assert (c == 0).all() and s[0] == 1.0
    np.testing.assert_array_equal(O.dequantize(c, s, z, 16), 0.0)
    c, s, z = O.quantize(np.full(16, -0.375), 4, 8, "asym")
    assert (c == 0).all() and (s == 1.0).all() and (z == np.float32(-0.375)).all()
    np.testing.assert_array_equal(O.dequantize(c, s, z, 8), -0.375)      # constant group is exact


@pytest.mark.parametrize("bits", [2, 4, 8])
@pytest.mark.parametrize("g", [8, 32, 128])
def test_asym_endpoints_and_bound(bits, g):
    rng = np.random.default_rng(bits * 1000 + g)
    for trial in range(20):
        x = bf16_vals(rng, 128, scale=10 ** rng.uniform(-3, 2))
        c, s, z = O.quantize(x, bits, g, "asym")
        xt = O.dequantize(c, s, z, g)
        for gi in range(128 // g):
            xs = x[gi * g:(gi + 1) * g]
            cs = c[gi * g:(gi + 1) * g]
            assert cs[np.argmin(xs)] == 0                     # min -> code 0
            assert cs[np.argmax(xs)] == 2 ** bits - 1         # max -> top code
            assert z[gi] == np.float32(xs.min())
            # |x - x̃| <= s/2 (+ fp32 slack)
            err = np.abs(xs - xt[gi * g:(gi + 1) * g])
            assert err.max() <= float(s[gi]) * (0.5 + 1e-5) + abs(xs).max() * 1e-6


@settings(max_examples=100, deadline=None)
@given(st.integers(0, 2 ** 31), st.sampled_from([2, 4, 8]), st.sampled_from(["asym", "sym"]))
def test_code_is_nearest_level(seed, bits, mode):
    """Independent check with Python floats: each code is within 1/2 (+fp32 slack) of
    the exact quotient, i.e. the nearest representable level."""
    rng = np.random.default_rng(seed)
    x = bf16_vals(rng, 32)
    c, s, z = O.quantize(x, bits, 32, mode)
    q = [(float(v) - float(z[0])) / float(s[0]) for v in x]
    lo, hi = (0, 2 ** bits - 1) if mode == "asym" else (-(2 ** (bits - 1) - 1), 2 ** (bits - 1) - 1)
    for ci, qi in zip(c.tolist(), q):
        assert lo <= ci <= hi
        assert abs(ci - min(max(qi, lo), hi)) <= 0.5 + 1e-4


def test_fp32_emulation_matches_torch_float32():
    """The op-by-op float32 emulation equals torch's float32 kernels (an independent
    IEEE implementation): sub, div, round-half-even."""
    rng = np.random.default_rng(5)
    for bits in (2, 4, 8):
        x = bf16_vals(rng, 64, 3.0)
        c, s, z = O.quantize(x, bits, 64, "asym")
        t = torch.tensor(x, dtype=torch.float32)
        mn, mx = t.min(), t.max()
        ts = (mx - mn) / torch.tensor(float(2 ** bits - 1), dtype=torch.float32)
        tc = torch.clamp(torch.round((t - mn) / ts), 0, 2 ** bits - 1).to(torch.int64)
        assert ts.item() == float(s[0])
        assert tc.tolist() == c.tolist()


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(6)
    x = (rng.normal(size=4096) * 10 ** rng.uniform(-4, 4, size=4096)).astype(np.float32)
    ref = torch.tensor(x).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(O.f32_to_bf16_rne(x), ref)


def test_promote_by_hand():
    codes = np.array([0, 3, 15, 7])
    s = np.array([np.float32(0.1)], dtype=np.float32)
    z = np.array([np.float32(-0.75)], dtype=np.float32)
    got = O.promote(codes, s, z, 4)
    exp = [torch.tensor(float(np.float32(np.float32(c) * s[0]) + z[0]), dtype=torch.float32).to(torch.bfloat16).item()
           for c in codes]
    np.testing.assert_array_equal(got, exp)
