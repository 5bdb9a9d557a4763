"""Oracle pins for layer-shared token states (NEXT-3; scores "computed over the
query heads of each group then averaged across groups into one vector").

Special cases that reduce to the per-KV-head path (already pinned): one KV head per layer,
and identical KV heads (the average of equal score vectors is that vector).  Plus the
defining invariant — every KV head of a layer ends with the same token states — and the
selection equal to a brute-force sort of the averaged scores."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from synth import Shape, prefill_inputs, decode_inputs


def _np(t):
    return t.double().numpy()


def _run(cfg, sh, steps, seed, rho, dup_heads=False):
    qw, k, v = prefill_inputs(sh, seed=seed, recipe="margin")
    if dup_heads:   # every KV head (and its query group) a copy of head 0
        G = sh.n_q_heads // sh.n_kv_heads
        k[:, :, 1:] = k[:, :, :1]
        v[:, :, 1:] = v[:, :, :1]
        qw[:, :, G:] = qw[:, :, :G].repeat(1, 1, sh.n_kv_heads - 1, 1, 1)
    ora = O.OracleARKV(cfg)
    ora.prefill(_np(qw), _np(k), _np(v), rho_override=rho)
    outs = []
    for s in range(steps):
        q, kn, vn = decode_inputs(sh, s, seed=seed, recipe="margin")
        if dup_heads:
            G = sh.n_q_heads // sh.n_kv_heads
            kn[:, :, 1:] = kn[:, :, :1]
            vn[:, :, 1:] = vn[:, :, :1]
            q[:, :, G:] = q[:, :, :G].repeat(1, 1, sh.n_kv_heads - 1, 1)
        outs.append(ora.decode_step(_np(q), _np(kn), _np(vn)))
    return ora, np.stack(outs)


def _cfg(sh, B, sharing):
    return O.Cfg(n_layers=sh.n_layers, n_q_heads=sh.n_q_heads, n_kv_heads=sh.n_kv_heads, head_dim=sh.head_dim,
                 batch=sh.batch, window=sh.window, budget_tokens=B, quant_bits=4, group_size=sh.head_dim // 2,
                 state_sharing=sharing)


def _exports_equal(a, b, sh):
    for bb in range(sh.batch):
        for l in range(sh.n_layers):
            for h in range(sh.n_kv_heads):
                ea, eb = a.export(bb, l, h), b.export(bb, l, h)
                for key in ("state", "q_k", "k_scale", "o_v"):
                    np.testing.assert_array_equal(ea[key], eb[key])


def test_single_kv_head_layer_equals_head_sharing():
    sh = Shape(batch=1, n_layers=2, n_q_heads=4, n_kv_heads=1, head_dim=16, prompt_len=80, window=8)
    a, oa = _run(_cfg(sh, 40, "head"), sh, 24, 3, [[0.7, 0.4]])
    b, ob = _run(_cfg(sh, 40, "layer"), sh, 24, 3, [[0.7, 0.4]])
    np.testing.assert_array_equal(oa, ob)
    _exports_equal(a, b, sh)


def test_identical_heads_layer_equals_head_sharing():
    sh = Shape(batch=1, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, prompt_len=80, window=8)
    a, oa = _run(_cfg(sh, 40, "head"), sh, 24, 5, [[0.5]], dup_heads=True)
    b, ob = _run(_cfg(sh, 40, "layer"), sh, 24, 5, [[0.5]], dup_heads=True)
    np.testing.assert_array_equal(oa, ob)
    _exports_equal(a, b, sh)


def test_layer_sharing_states_identical_and_brute_force():
    sh = Shape(batch=2, n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=16, prompt_len=96, window=8)
    cfg = _cfg(sh, 48, "layer")
    ora, _ = _run(cfg, sh, 30, 7, [[0.6, 0.3], [1.0, 0.5]])
    n_t = 0
    for b in range(2):
        for l in range(2):
            st = [ora.export(b, l, h)["state"] for h in range(4)]
            for h in range(1, 4):
                np.testing.assert_array_equal(st[h], st[0])
            n_t += len(ora.units[(b, l, 0)].tailors)
    assert n_t >= 8
    # the prefill-end selection equals a brute-force sort of the group-averaged scores
    qw, k, v = prefill_inputs(sh, seed=7, recipe="margin")
    qw, k = _np(qw), _np(k)
    P, W, G = sh.prompt_len, sh.window, 2
    a = O.windowed_attention(qw[0, 0], k[0, 0], cfg)
    S = np.mean([O.hh_scores(a[h * G:(h + 1) * G].reshape(G * W, P - W), cfg.gamma) for h in range(4)], axis=0)
    n_oe, n_q = O.tailor_counts(P, 0.6, cfg)
    order = sorted(range(P - W), key=lambda i: (-S[i], i))
    ref = np.full(P - W, 3)
    ref[order[:n_oe]] = 1
    ref[order[n_oe:n_oe + n_q]] = 2
    ora2 = O.OracleARKV(cfg)
    ora2.prefill(qw, k, _np(v), rho_override=[[0.6, 0.3], [1.0, 0.5]])
    np.testing.assert_array_equal(ora2.export(0, 0, 2)["state"][:P - W], ref)
