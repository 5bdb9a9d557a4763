"""Pins for the oracle's prefill statistics (Eqs. 2-7).

Every check ties the oracle to something other than itself: SPEC's printed
examples (tests/golden/spec_examples.json), closed forms, and brute-force loops.
"""
import json
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _cfg(**kw):
    base = dict(n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=8, window=2, budget_tokens=8)
    base.update(kw)
    return O.Cfg(**base)


# --- Eq. 2 windowed attention ------------------------------------------------

@pytest.mark.parametrize("case", GOLD["slice_window_shapes"]["cases"])
def test_slice_window_shapes(case):
    H, K, W = case["H"], case["K"], case["W"]
    rng = np.random.default_rng(0)
    cfg = _cfg(n_q_heads=H, n_kv_heads=1, head_dim=4, window=W)
    a = O.windowed_attention(rng.normal(size=(H, W, 4)), rng.normal(size=(1, K, 4)), cfg)
    assert list(a.shape) == case["shape"]


def _brute_windowed(q_win, k, sm):
    """Pure-Python loops: softmax over causally visible keys, then slice (R1)."""
    H, W, d = q_win.shape
    P = k.shape[1]
    G = H // k.shape[0]
    out = np.zeros((H, W, P - W))
    for h in range(H):
        for i in range(W):
            qp = P - W + i
            logits = [sum(float(q_win[h, i, x]) * float(k[h // G, j, x]) for x in range(d)) * sm
                      for j in range(qp + 1)]
            m = max(logits)
            e = [math.exp(s - m) for s in logits]
            Z = sum(e)
            for j in range(P - W):
                out[h, i, j] = e[j] / Z
    return out


def test_windowed_attention_brute_force():
    rng = np.random.default_rng(1)
    H, Hkv, W, P, d = 4, 2, 3, 9, 5
    cfg = _cfg(n_q_heads=H, n_kv_heads=Hkv, head_dim=d, window=W)
    qw, k = rng.normal(size=(H, W, d)), rng.normal(size=(Hkv, P, d))
    np.testing.assert_allclose(O.windowed_attention(qw, k, cfg), _brute_windowed(qw, k, cfg.sm_scale), rtol=1e-12, atol=1e-15)


def test_windowed_attention_identical_keys_closed_form():
    """All keys equal -> each row is uniform over its visible keys: Ã[h,i,j] = 1/(P-W+i+1)."""
    H, W, P, d = 2, 4, 12, 6
    cfg = _cfg(n_q_heads=H, n_kv_heads=1, head_dim=d, window=W)
    rng = np.random.default_rng(2)
    k = np.repeat(rng.normal(size=(1, 1, d)), P, axis=1)
    a = O.windowed_attention(rng.normal(size=(H, W, d)), k, cfg)
    for i in range(W):
        np.testing.assert_allclose(a[:, i, :], 1.0 / (P - W + i + 1), rtol=1e-13)
    assert np.all(a.sum(axis=2) < 1.0)          # sliced rows sum to < 1


# --- Eq. 3 key mass ----------------------------------------------------------

def test_key_mass_spec_examples():
    g = GOLD["key_mass"]
    a = np.array(g["per_head_key_sums"], dtype=float)[:, None, :]        # [H][1][K]
    np.testing.assert_allclose(O.key_mass(a), g["p"], rtol=1e-15)
    np.testing.assert_allclose(O.key_mass(np.ones((1, 1, 4))), [0.25] * 4)
    oh = np.zeros((1, 1, 4)); oh[0, 0, 2] = 0.7
    np.testing.assert_allclose(O.key_mass(oh), [0, 0, 1, 0])
    with pytest.raises(ValueError):
        O.key_mass(np.zeros((1, 1, 4)))


# --- Eqs. 3-5 statistics --------------------------------------------------------

@pytest.mark.parametrize("case", GOLD["compute_stats"]["cases"])
def test_stats_spec_examples(case):
    H, V, K = O.compute_stats(np.array(case["p"]))
    assert H == pytest.approx(max(case["entropy"], 1e-30), abs=5e-7)
    if "variance" in case:
        assert V == pytest.approx(max(case["variance"], 1e-30), abs=1e-15)


@pytest.mark.parametrize("n", [2, 3, 4, 7, 100, 32736])
def test_stats_uniform_closed_form(n):
    H, V, K = O.compute_stats(np.full(n, 1.0 / n))
    assert H == pytest.approx(math.log(n), rel=1e-12)
    assert V <= 1e-30 and K == 1.0           # R6: K := 1 for a flat distribution


@pytest.mark.parametrize("n", [2, 4, 5, 64, 1000])
def test_stats_one_hot_closed_form(n):
    p = np.zeros(n); p[n // 2] = 1.0
    H, V, K = O.compute_stats(p)
    assert H == 1e-30                         # 𝓗 = 0, clamped (R6)
    assert V == pytest.approx((n - 1) / n ** 2, rel=1e-12)
    assert K == pytest.approx((n * n - 3 * n + 3) / (n - 1), rel=1e-10)


def test_stats_dyadic_closed_form():
    H, V, K = O.compute_stats(np.array([0.5, 0.25, 0.125, 0.125]))
    assert H == pytest.approx(1.75 * math.log(2), rel=1e-14)
    assert V == pytest.approx(0.0234375, rel=1e-14)
    assert K == pytest.approx(2.0, rel=1e-13)


@settings(max_examples=200, deadline=None)
@given(st.lists(st.floats(0.0, 10.0), min_size=2, max_size=40).filter(lambda x: sum(x) > 1e-3))
def test_stats_properties(xs):
    p = np.array(xs) / np.sum(xs)
    n = len(p)
    H, V, K = O.compute_stats(p)
    assert H <= math.log(n) + 1e-9            # entropy bounded by ln n
    # brute-force moments with Python floats
    m2 = sum((x - 1.0 / n) ** 2 for x in p) / n
    assert V == pytest.approx(max(m2, 1e-30), rel=1e-9, abs=1e-30)
    if m2 > 1e-20:
        m4 = sum((x - 1.0 / n) ** 4 for x in p) / n
        assert K == pytest.approx(m4 / m2 ** 2, rel=1e-7)
        assert K >= 1.0 - 1e-9                # Pearson kurtosis >= 1 (R5)


# --- Eqs. 6-7 OQ score and ratio ------------------------------------------------

@pytest.mark.parametrize("case", GOLD["oq_score"]["cases"])
def test_oq_score_spec(case):
    q = O.oq_score(case["H"], case["V"], case["K"], tuple(case["tau"]))
    assert q == pytest.approx(case["q"], abs=5e-7)


@pytest.mark.parametrize("case", GOLD["oq_ratios"]["cases"])
def test_oq_ratios_spec(case):
    np.testing.assert_allclose(O.oq_ratios(case["q"]), case["rho"], rtol=1e-15)


@settings(max_examples=100, deadline=None)
@given(st.lists(st.floats(1e-6, 1e3), min_size=1, max_size=40), st.floats(1e-3, 1e3))
def test_oq_ratio_scale_invariance(q, c):
    r = O.oq_ratios(q)
    assert r.max() == 1.0
    np.testing.assert_allclose(O.oq_ratios(np.array(q) * c), r, rtol=1e-12)


def test_prefill_stats_end_to_end_brute():
    """prefill_stats() = brute windowed attention -> hand key mass -> closed-form moments."""
    rng = np.random.default_rng(3)
    B, L, Hq, Hkv, W, P, d = 1, 3, 4, 2, 3, 10, 4
    cfg = _cfg(n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, window=W, budget_tokens=7)
    qw = rng.normal(size=(B, L, Hq, W, d)); k = rng.normal(size=(B, L, Hkv, P, d)) * (1 + np.arange(L))[None, :, None, None, None]
    stats, oq, rho, _ = O.prefill_stats(qw, k, cfg)
    for l in range(L):
        a = _brute_windowed(qw[0, l], k[0, l], cfg.sm_scale)
        col = [sum(a[h, i, j] for h in range(Hq) for i in range(W)) for j in range(P - W)]
        Z = sum(col)
        p = [c / Z for c in col]
        n = P - W
        H = -sum(x * math.log(x) for x in p)
        m2 = sum((x - 1 / n) ** 2 for x in p) / n
        m4 = sum((x - 1 / n) ** 4 for x in p) / n
        np.testing.assert_allclose(stats[0, l], [H, m2, m4 / m2 ** 2], rtol=1e-10)
        t = cfg.tau
        assert oq[0, l] == pytest.approx(H ** (1 / t[0]) * m2 ** (1 / t[1]) * (m4 / m2 ** 2) ** (1 / t[2]), rel=1e-10)
    assert rho.max() == 1.0 and rho[0, int(np.argmax(oq[0]))] == 1.0
