"""Pins for the "smoothed" heavy-hitter scores (Alg. 1; reading R34, NEXT-4).

The paper names smoothing but gives no formula; R34 reads it as an exponential moving
average across tailors.  The pins check what any correct implementation of that reading
must satisfy, not the formula itself:
  * λ = 0 leaves every tailor exactly as the unsmoothed path (R21);
  * stationarity: when every token's Eq. 9 score is the same at each tailor, the average
    equals the score, so any λ gives the unsmoothed states (a dropped (1 − λ), a λ on the
    wrong term or a previous score taken from another token breaks this);
  * memory: a token that was the top heavy hitter at the previous tailor survives one bad
    window with λ = 0.9 and is evicted without smoothing;
  * only tokens the previous tailor scored and kept carry a previous score.
"""
import numpy as np
import pytest

import oracle as O

W = 2


def unit_cfg(lam):
    return O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=16, window=W, budget_tokens=12,
                 quant_bits=4, group_size=16, smooth=lam)


def two_tailors(lam, p1, p2, seed=0):
    """Prefill of 16 tokens, tailor 1 on the 14 eligible ones with per-token scores p1,
    three appends, tailor 2 on the 13 eligible ones with scores p2 (positions ascending).
    Identical samples in both window rows make the Eq. 9 score the sample itself
    (variance 0)."""
    rng = np.random.default_rng(seed)
    u = O.UnitCache(unit_cfg(lam))
    u.ingest(rng.standard_normal((16, 16)), rng.standard_normal((16, 16)))
    e1, _ = u.eligible()
    assert len(e1) == 14
    u.tailor(0.5, [(e1, np.stack([p1, p1]))], 16)
    s1 = u.export()["state"].copy()
    for t in range(16, 19):
        u.append(t, rng.standard_normal(16), rng.standard_normal(16))
    e2, _ = u.eligible()
    assert len(e2) == 13
    u.tailor(0.5, [(e2, np.stack([p2, p2]))], 19)
    return u, s1, e1, e2


def p_first():
    p = 0.01 * (1.0 + np.arange(14) / 13.0)
    p[0] = 0.5                   # token 0: the top heavy hitter at tailor 1
    return p


def test_counts_of_the_scenario():
    u, s1, e1, e2 = two_tailors(0.0, p_first(), np.linspace(0.02, 0.04, 13))
    assert (s1[:14] == 1).sum() == 5 + 0 and (s1 == 2).sum() == 5 and (s1 == 3).sum() == 4
    assert u.n_o == 5 + W and u.n_q == 4


def test_lambda_zero_is_unsmoothed():
    rng = np.random.default_rng(3)
    p1, p2 = rng.uniform(0.001, 0.1, 14), rng.uniform(0.001, 0.1, 13)
    a = two_tailors(0.0, p1, p2)[0].export()
    b = O.UnitCache(unit_cfg(0.0))
    assert O.smooth_scores(p2, np.arange(13), {0: 5.0}, 0.0) is not None
    np.testing.assert_array_equal(O.smooth_scores(p2, np.arange(13), {0: 5.0, 3: 1.0}, 0.0), p2)
    # a run with smoothing configured but λ = 0 equals one that never heard of it
    c = two_tailors(0.0, p1, p2)[0].export()
    for k in a:
        np.testing.assert_array_equal(np.asarray(a[k]), np.asarray(c[k]))
    assert b.prev_score == {}


@pytest.mark.parametrize("lam", [0.25, 0.5, 0.9])
def test_stationary_scores_are_left_unchanged(lam):
    rng = np.random.default_rng(7)
    p1 = rng.uniform(0.001, 0.1, 14)
    u0, _, e1, e2 = two_tailors(0.0, p1, np.zeros(13))
    # tailor 2 sees every surviving token with its tailor-1 score; tokens new since
    # tailor 1 (the old window and the append) get fresh distinct scores
    by_pos = dict(zip(e1.tolist(), p1.tolist()))
    fresh = iter(rng.uniform(0.001, 0.1, 13))
    p2 = np.array([by_pos[p] if p in by_pos else next(fresh) for p in e2.tolist()])
    ref = two_tailors(0.0, p1, p2)[0].export()
    got = two_tailors(lam, p1, p2)[0].export()
    for k in ("state", "q_k", "q_v", "k_scale", "v_scale"):
        np.testing.assert_array_equal(np.asarray(ref[k]), np.asarray(got[k]), err_msg=k)


def test_memory_keeps_a_past_heavy_hitter():
    p2 = np.linspace(0.02, 0.04, 13)
    p2[0] = 1e-4                 # token 0 (still position 0, eligible) has one bad window
    _, s1, _, e2 = two_tailors(0.0, p_first(), p2)
    assert s1[0] == 1 and e2[0] == 0
    no = two_tailors(0.0, p_first(), p2)[0].export()["state"]
    yes = two_tailors(0.9, p_first(), p2)[0].export()["state"]
    assert no[0] == 3            # unsmoothed: the lowest score of the window -> evicted
    assert yes[0] == 1           # λ = 0.9: 0.9·0.5 + 0.1·1e-4 still ranks first -> Original


def test_previous_scores_only_for_scored_and_kept_tokens():
    u, s1, e1, e2 = two_tailors(0.5, p_first(), np.linspace(0.02, 0.04, 13))
    kept_after_2 = {int(p) for p in e2.tolist() if u.export()["state"][p] in (1, 2)}
    assert set(u.prev_score) == kept_after_2
    # tailor 2's eligible set: kept tokens of tailor 1 (with a previous score), the two
    # old window tokens (14, 15) and the first append (16) (without one)
    assert {14, 15, 16} <= set(e2.tolist())
    with pytest.raises(ValueError):
        O.validate(unit_cfg(1.0))
