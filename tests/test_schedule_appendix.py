"""Count-schedule pins (CPU): SURVEY Appendix A's tuples verbatim and SPEC's needs_tailor
boundary examples, checked against the oracle (oracle.schedule) and the host C++ schedule
(arkv_schedule through the C ABI; host-only, no GPU).  Reading R12: the decode tailor
fires after the append iff U >= B_bytes ("triggered when the KV cache reaches the
limit"; "true iff usage >= budget.total")."""
import json
import os

import pytest

import oracle as O
from paper_2603_08727_b200 import arkv as A

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a_schedule.json")))


def _cfg(g):
    return O.Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=g["d"], window=g["W"], budget_tokens=g["B"],
                 quant_bits=g["bits"], group_size=g["g"])


def _one_based(ev):
    """oracle.schedule steps are 0-based decode-call indices (-1 = prefill tailor)."""
    pre = [e[1:] for e in ev if e[0] == -1]
    dec = [[e[0] + 1, *e[1:]] for e in ev if e[0] >= 0]
    return pre, dec


@pytest.mark.parametrize("case", GOLD["toy"]["cases"], ids=lambda c: f"rho{c['rho']}")
def test_appendix_a_toy(case):
    g = GOLD["toy"]
    cfg = _cfg(g)
    pre, dec = _one_based(O.schedule(g["P"], g["steps"], case["rho"], cfg))
    assert pre == [tuple(case["prefill"])]
    assert [list(x) for x in dec] == case["decode"]


@pytest.mark.parametrize("case", GOLD["config2"]["cases"], ids=lambda c: f"rho{c['rho']}")
def test_appendix_a_config2(case):
    g = GOLD["config2"]
    cfg = _cfg(g)
    last = case["decode"][-1][0]
    pre, dec = _one_based(O.schedule(g["P"], last + 4096, case["rho"], cfg))
    assert pre == [tuple(case["prefill"])]
    assert [list(x) for x in dec[:len(case["decode"])]] == case["decode"]
    if "then_every" in case:
        steps = [x[0] for x in dec]
        assert all(b - a == case["then_every"] for a, b in zip(steps, steps[1:]))
        assert all(list(x[1:]) == case["decode"][0][1:] for x in dec)


@pytest.mark.parametrize("which", ["toy", "config2"])
def test_appendix_a_host_schedule(which):
    """The host C++ schedule (drives every kernel launch) reproduces the same tuples."""
    g = GOLD[which]
    for case in g["cases"]:
        steps = case["decode"][-1][0] + (4096 if which == "config2" else 0)
        if which == "toy":
            steps = g["steps"]
        c = A.make_config(1, 4, 2, g["d"], window=g["W"], budget_tokens=g["B"], quant_bits=g["bits"],
                          group_size=g["g"], max_positions=g["P"] + steps + 1, max_prompt=g["P"])
        pre, dec = _one_based(A.arkv_schedule(c, g["P"], case["rho"], steps))
        assert pre == [tuple(case["prefill"])]
        assert [list(x) for x in dec[:len(case["decode"])]] == case["decode"]


@pytest.mark.parametrize("case", GOLD["needs_tailor"]["cases"])
def test_needs_tailor_boundary(case):
    """usage equal to the budget triggers (the boundary case)."""
    cfg = O.Cfg(n_layers=1, n_q_heads=1, n_kv_heads=1, head_dim=64, window=32,
                budget_tokens=GOLD["needs_tailor"]["B"])
    assert O.decode_needs_tailor(case["n_o"], case["n_q"], cfg) is case["tailor"]


def test_host_trigger_step_at_boundary():
    """The host fires on the append that makes U == B_bytes exactly: an untailored prompt of
    B - W tokens (U = B_bytes - W*C_o) tailors on its W-th decode call."""
    W, B = 8, 40
    c = A.make_config(1, 2, 1, 16, window=W, budget_tokens=B, quant_bits=4, group_size=16,
                      max_positions=200, max_prompt=B - W)
    ev = A.arkv_schedule(c, B - W, 1.0, 3 * W)
    assert ev[0][0] == W - 1            # 0-based: the W-th call
