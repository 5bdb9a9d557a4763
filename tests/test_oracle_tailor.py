"""Pins for the oracle's counts, heavy-hitter scores, ranking and tailor (Eqs. 1, 8-10)."""
import json
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def toy_cfg(**kw):
    # BASELINE configs[0] with reading R29 (W = 8 so that B > 2W)
    base = dict(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, window=8,
                budget_tokens=32, quant_bits=4, group_size=16)
    base.update(kw)
    return O.Cfg(**base)


# --- Eq. 1 costs -------------------------------------------------------------------

def test_costs_by_hand():
    c = O.Cfg(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, budget_tokens=8192)
    assert O.cost_orig(c) == 512                      # 128 bf16 K + 128 bf16 V
    assert O.cost_quant(c) == 2 * (64 + 8)            # 4-bit codes + fp32 scale & zero, K and V
    c8 = O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=128, quant_bits=8, group_size=32)
    assert O.cost_quant(c8) == 2 * (128 + 4 * 8)
    assert O.budget_bytes(c) == 8192 * 512


# --- Alg. 1 budget split ----------------------------------------------------

@pytest.mark.parametrize("case", GOLD["origin_quota"]["cases"])
def test_origin_quota_spec(case):
    cfg = O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=16, window=case["W"], budget_tokens=case["B"])
    assert case["W"] + O.origin_quota(case["rho"], cfg) == case["original_quota"]


def test_keep_size_spec():
    g = GOLD["build_plan"]
    n_e = g["K"] - g["W"]
    assert n_e == g["eligible"]
    assert math.floor(g["alpha"] * n_e) == g["b"]


def _brute_counts(K, rho, cfg):
    """Independent formulation of R14: walk the ranked keep list of b tokens; give
    Original to the first min(⌊ρ(B−W)⌋, B−2W) of them, then add Quantized tokens one
    at a time while the unit (window included) stays within B_bytes − W·C_o."""
    W, B = cfg.window, cfg.budget_tokens
    n_e = K - W
    b = (3 * n_e) // 4 if cfg.alpha == 0.75 else int(cfg.alpha * n_e)
    quota = int(rho * (B - W))
    n_oe = 0
    for _ in range(b):
        if n_oe < quota and n_oe < B - 2 * W:
            n_oe += 1
    n_q = 0
    limit = cfg.budget_tokens * 4 * cfg.head_dim - W * 4 * cfg.head_dim
    while n_oe + n_q < b and (n_oe + W) * 4 * cfg.head_dim + (n_q + 1) * O.cost_quant(cfg) <= limit:
        n_q += 1
    return n_oe, n_q


@settings(max_examples=300, deadline=None)
@given(st.integers(40, 3000), st.floats(0.01, 1.0), st.sampled_from([(16, 4, 16), (128, 4, 128), (128, 2, 32), (64, 8, 64)]),
       st.integers(2, 40))
def test_tailor_counts_vs_brute(K, rho, dbg, W):
    d, bits, g = dbg
    B = 2 * W + 1 + K // 3
    cfg = O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=d, window=W, budget_tokens=B, quant_bits=bits, group_size=g)
    if K <= W:
        return
    assert O.tailor_counts(K, rho, cfg) == _brute_counts(K, rho, cfg)


@settings(max_examples=150, deadline=None)
@given(st.integers(10, 600), st.integers(0, 400), st.floats(0.02, 1.0), st.integers(2, 16),
       st.sampled_from([(16, 4, 16), (128, 4, 128), (32, 2, 16), (64, 8, 32)]))
def test_schedule_invariants(P, steps, rho, W, dbg):
    """Budget is never exceeded at any attention step (Eq. 1); every tailor leaves
    at least W tokens of headroom (R14), so tailors are > W steps apart; counts
    are non-negative and partition the eligible tokens."""
    d, bits, g = dbg
    B = 2 * W + 1 + (P // 2)
    cfg = O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=d, window=W, budget_tokens=B, quant_bits=bits, group_size=g)
    ev = O.schedule(P, steps, rho, cfg)
    Bb, Co = O.budget_bytes(cfg), O.cost_orig(cfg)
    last = None
    for (s, n_o, n_q, n_ev) in ev:
        assert n_o >= W and n_q >= 0 and n_ev >= 0
        assert O.usage_bytes(cfg, n_o, n_q) <= Bb - W * Co
        if last is not None:
            assert s - last >= W      # U_after <= B_bytes - W*C_o (R14) and U >= B_bytes fires (R12)
        last = s
    # replay: usage <= budget at every attention
    n_o, n_q = (ev[0][1], ev[0][2]) if ev and ev[0][0] == -1 else (P, 0)
    assert O.usage_bytes(cfg, n_o, n_q) <= Bb
    evd = {e[0]: e for e in ev}
    for s in range(steps):
        n_o += 1
        if s in evd:
            n_o, n_q = evd[s][1], evd[s][2]
        assert O.usage_bytes(cfg, n_o, n_q) <= Bb


def test_schedule_toy_hand_derived():
    """Toy (BASELINE configs[0], R29): P=64, B=32, W=8, d=16, 4-bit g=16.
    C_o = 64 B, C_q = 32 B, B_bytes = 2048.  Hand derivation (DESIGN.md §3 R12/R14):
    prefill K=64 -> n_e=56, b=42; rho=1: n_oe=min(24,42,16)=16, n_q=min(26,(2048-32*64)//32=0)
    -> (24, 0, 40).  rho=0.5: n_oe=12, n_q=min(30, 256//32=8)=8 -> (20, 8, 36).
    rho=0.25: n_oe=6, n_q=min(36, 640//32=20)=20 -> (14, 20, 30).  Decode: rho=1, usage
    24*64 = 1536 reaches 2048 after 8 appends (0-based step index 7): K=32, n_e=24, b=18,
    n_oe=16 -> (24, 0, 8) (tests/test_schedule_appendix.py)."""
    cfg = toy_cfg()
    assert O.schedule(64, 16, 1.0, cfg) == [(-1, 24, 0, 40), (7, 24, 0, 8), (15, 24, 0, 8)]
    assert O.schedule(64, 0, 0.5, cfg) == [(-1, 20, 8, 36)]
    assert O.schedule(64, 0, 0.25, cfg) == [(-1, 14, 20, 30)]


# --- Eq. 9 heavy-hitter score ---------------------------------------------------------

def test_hh_spec_example():
    g = GOLD["hh_scores"]
    S = O.hh_scores(np.array(g["weights"])[:, None], g["gamma"])
    assert S[0] == pytest.approx(g["S"], rel=1e-12)
    assert S[0] == pytest.approx(g["mu"] + g["gamma"] * g["var"], rel=1e-12)


def test_hh_constant_and_gamma0():
    rng = np.random.default_rng(0)
    s = np.full((12, 5), 0.07)
    np.testing.assert_allclose(O.hh_scores(s, 263.81), 0.07, rtol=1e-14)
    x = rng.random((8, 30))
    np.testing.assert_allclose(O.hh_scores(x, 0.0), x.mean(axis=0), rtol=1e-14)


def test_hh_brute_and_equivariance():
    rng = np.random.default_rng(1)
    x = rng.random((16, 20)) * 1e-2
    S = O.hh_scores(x, 263.81)
    for j in range(20):
        col = [float(v) for v in x[:, j]]
        mu = sum(col) / len(col)
        var = sum((c - mu) ** 2 for c in col) / len(col)
        assert S[j] == pytest.approx(mu + 263.81 * var, rel=1e-12)
    perm = rng.permutation(20)
    np.testing.assert_allclose(O.hh_scores(x[:, perm], 263.81), S[perm], rtol=1e-15)


# --- Eq. 10 ranking / plan ------------------------------------------------------------

def test_top_b_spec():
    g = GOLD["top_b"]
    order = O.rank_order(np.array(g["scores"]), np.arange(3))
    assert set(order[:g["b"]].tolist()) == set(g["set"])
    assert len(order[:0]) == 0
    eq = O.rank_order(np.ones(5), np.arange(5))
    assert list(eq[:3]) == [0, 1, 2]         # all equal -> lowest positions


@settings(max_examples=300, deadline=None)
@given(st.lists(st.integers(0, 6), min_size=1, max_size=60), st.data())
def test_plan_vs_full_sort(levels, data):
    """Heavy ties: plan_states equals a brute-force Python sort on (-S, pos)."""
    n = len(levels)
    S = np.array(levels, dtype=float) * 0.1
    pos = np.array(data.draw(st.permutations(list(range(n)))), dtype=np.int64) * 3 + 5
    n_oe = data.draw(st.integers(0, n))
    n_q = data.draw(st.integers(0, n - n_oe))
    stt = O.plan_states(S, pos, n_oe, n_q)
    ranked = sorted(range(n), key=lambda i: (-S[i], pos[i]))
    exp = np.full(n, 3)
    for r, i in enumerate(ranked):
        exp[i] = 1 if r < n_oe else (2 if r < n_oe + n_q else 3)
    assert stt.tolist() == exp.tolist()
    # score monotonicity
    if (stt == 1).any() and (stt == 2).any():
        assert S[stt == 1].min() >= S[stt == 2].max()
    if (stt == 2).any() and (stt == 3).any():
        assert S[stt == 2].min() >= S[stt == 3].max()
