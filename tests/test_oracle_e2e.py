"""End-to-end pins for the oracle driver (Alg. 1): dense-attention special case,
closed forms, plan invariants and the count schedule."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth import Shape, prefill_inputs, decode_inputs


def _np(t):
    return t.double().numpy()


def _brute_attention(q, K, V, sm):
    out = np.zeros((q.shape[0], V.shape[1]))
    for h in range(q.shape[0]):
        logits = [sum(float(q[h, x]) * float(K[j, x]) for x in range(q.shape[1])) * sm for j in range(K.shape[0])]
        m = max(logits)
        e = [math.exp(s - m) for s in logits]
        Z = sum(e)
        for j in range(K.shape[0]):
            out[h] += e[j] / Z * V[j]
    return out


def test_no_pressure_equals_dense_attention():
    """Budget >= all tokens -> no tailor; the decode output is textbook softmax
    attention over the full bf16 cache (Base model P:330)."""
    sh = Shape(batch=1, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=8, prompt_len=12, window=4)
    cfg = O.Cfg(n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=8, window=4, budget_tokens=64)
    qw, k, v = prefill_inputs(sh, seed=3)
    ora = O.OracleARKV(cfg)
    ora.prefill(_np(qw), _np(k), _np(v))
    Ks, Vs = _np(k), _np(v)
    for step in range(6):
        q, kn, vn = decode_inputs(sh, step, seed=3)
        out = ora.decode_step(_np(q), _np(kn), _np(vn))
        Ks = np.concatenate([Ks, _np(kn)[:, :, :, None]], axis=3)
        Vs = np.concatenate([Vs, _np(vn)[:, :, :, None]], axis=3)
        for l in range(2):
            for h in range(4):
                exp = _brute_attention(_np(q)[0, l, h:h + 1], Ks[0, l, h // 2], Vs[0, l, h // 2], cfg.sm_scale)
                np.testing.assert_allclose(out[0, l, h], exp[0], rtol=1e-10, atol=1e-12)
    for kvh in range(2):
        e = ora.export(0, 0, kvh)
        assert (e["state"] == 1).all()
        np.testing.assert_array_equal(e["o_k"][:12], Ks[0, 0, kvh, :12])   # bitwise-exact bf16 copies


def test_constant_keys_give_mean_of_values():
    cfg = O.Cfg(n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=4, window=2, budget_tokens=64)
    ora = O.OracleARKV(cfg)
    rng = np.random.default_rng(0)
    P = 6
    k = np.ones((1, 1, 1, P, 4)) * 0.5
    v = rng.normal(size=(1, 1, 1, P, 4))
    ora.prefill(rng.normal(size=(1, 1, 2, 2, 4)), k, v, rho_override=[[1.0]])
    vn = rng.normal(size=(1, 1, 1, 4))
    out = ora.decode_step(rng.normal(size=(1, 1, 2, 4)), np.ones((1, 1, 1, 4)) * 0.5, vn)
    exp = np.concatenate([v[0, 0, 0], vn[0, 0]], axis=0).mean(axis=0)
    np.testing.assert_allclose(out[0, 0, 0], exp, rtol=1e-12)
    np.testing.assert_allclose(out[0, 0, 1], exp, rtol=1e-12)


def test_gqa_group1_equals_mha():
    """G = 1 (MHA): each head reads its own KV head."""
    cfg = O.Cfg(n_layers=1, n_q_heads=2, n_kv_heads=2, head_dim=4, window=2, budget_tokens=64)
    rng = np.random.default_rng(1)
    P = 7
    qw, k, v = rng.normal(size=(1, 1, 2, 2, 4)), rng.normal(size=(1, 1, 2, P, 4)), rng.normal(size=(1, 1, 2, P, 4))
    ora = O.OracleARKV(cfg)
    ora.prefill(qw, k, v)
    q, kn, vn = rng.normal(size=(1, 1, 2, 4)), rng.normal(size=(1, 1, 2, 4)), rng.normal(size=(1, 1, 2, 4))
    out = ora.decode_step(q, kn, vn)
    for h in range(2):
        K = np.concatenate([k[0, 0, h], kn[0, 0, h][None]])
        V = np.concatenate([v[0, 0, h], vn[0, 0, h][None]])
        np.testing.assert_allclose(out[0, 0, h], _brute_attention(q[0, 0, h:h + 1], K, V, cfg.sm_scale)[0], rtol=1e-12)


@pytest.mark.parametrize("rho", [1.0, 0.5, 0.25])
def test_toy_pipeline_invariants(rho):
    """BASELINE configs[0] toy (R29: W=8, injected rho): the data-driven tailors
    match the count-only schedule, every state export partitions the positions,
    the W newest positions are Original, Eq. 1 holds, Q tokens dequantize within
    s/2, and O tokens are bitwise the prompt/decode bf16 values or promotions."""
    sh = Shape(batch=1, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, prompt_len=64, window=8)
    cfg = O.Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, window=8, budget_tokens=32,
                quant_bits=4, group_size=16)
    qw, k, v = prefill_inputs(sh, seed=11, recipe="margin")
    ora = O.OracleARKV(cfg)
    ora.prefill(_np(qw), _np(k), _np(v), rho_override=[[rho]])
    allk = [_np(k)[0, 0]]
    steps = 16
    for s in range(steps):
        q, kn, vn = decode_inputs(sh, s, seed=11, recipe="margin")
        ora.decode_step(_np(q), _np(kn), _np(vn))
        allk.append(_np(kn)[0, 0][:, None])
    allk = np.concatenate(allk, axis=1)      # [Hkv][P+steps][d]
    sched = O.schedule(64, steps, rho, cfg)
    for kvh in range(2):
        u = ora.units[(0, 0, kvh)]
        got = [(-1 if t == 64 and i == 0 else t - 64, n_o, n_q, ev) for i, (t, n_o, n_q, ev) in enumerate(u.tailors)]
        assert got == sched
        e = ora.export(0, 0, kvh)
        n = 64 + steps
        assert len(e["state"]) == n and set(np.unique(e["state"]).tolist()) <= {1, 2, 3}
        assert (e["state"][-8:] == 1).all()
        assert e["n_o"] == (e["state"] == 1).sum() and e["n_q"] == (e["state"] == 2).sum()
        assert O.usage_bytes(cfg, e["n_o"], e["n_q"]) <= O.budget_bytes(cfg)
        for p in np.where(e["state"] == 2)[0]:
            xt = O.dequantize(e["q_k"][p], e["k_scale"][p], e["k_zero"][p], 16)
            assert np.abs(xt - allk[kvh, p]).max() <= e["k_scale"][p][0] * 0.5 * (1 + 1e-5)


def test_determinism():
    sh = Shape(batch=1, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, prompt_len=64, window=8)
    cfg = O.Cfg(n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, window=8, budget_tokens=32)
    outs = []
    for _ in range(2):
        qw, k, v = prefill_inputs(sh, seed=5)
        ora = O.OracleARKV(cfg)
        ora.prefill(_np(qw), _np(k), _np(v), rho_override=[[0.5]])
        o = [ora.decode_step(*[_np(t) for t in decode_inputs(sh, s, seed=5)]) for s in range(10)]
        outs.append((np.stack(o), ora.export(0, 0, 1)["state"]))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("mode,bits,g", [("asym", 4, 8), ("sym", 8, 16), ("asym", 2, 16), ("fp8", 8, 16), ("sym", 4, 32)])
def test_all_quantized_equals_dense_attention_over_dequantized(mode, bits, g):
    """SURVEY §8(c) C3 pin of the Q-token attention (Alg. 1 'Reconstruction Before
    Attention'; P:253 'dequantized and concatenated ... attention is
    unmodified'): with rho = 0 and alpha = 1 every non-window token is Quantized; the
    decode output must equal textbook softmax attention over the dequantized keys/values,
    rebuilt here element by element from the exported codes, scales and zeros (x~ = code*s
    + z per group of g along head_dim) — independently of UnitCache.keys_values.  The
    codes are also checked against the prompt (|x - x~| <= s/2 (+ e4m3 half-step)) so a
    group-axis or scale/zero slip in the export fails too."""
    d, W, P, H_q, H_kv = 32, 4, 40, 4, 2
    sh = Shape(batch=1, n_layers=1, n_q_heads=H_q, n_kv_heads=H_kv, head_dim=d, prompt_len=P, window=W)
    cfg = O.Cfg(n_layers=1, n_q_heads=H_q, n_kv_heads=H_kv, head_dim=d, window=W, budget_tokens=40,
                quant_bits=bits, group_size=g, quant_mode=mode, alpha=1.0)
    assert O.prefill_needs_tailor(P, cfg)
    qw, k, v = prefill_inputs(sh, seed=11)
    ora = O.OracleARKV(cfg)
    ora.prefill(_np(qw), _np(k), _np(v), rho_override=[[0.0]])
    q, kn, vn = decode_inputs(sh, 0, seed=11)
    out = ora.decode_step(_np(q), _np(kn), _np(vn))
    G = H_q // H_kv
    for kvh in range(H_kv):
        e = ora.export(0, 0, kvh)
        st = e["state"]
        assert (st[:P - W] == 2).all() and (st[P - W:] == 1).all(), "every non-window token Quantized"
        Kt, Vt = [], []
        for p in range(P + 1):
            if st[p] == 1:
                Kt.append([float(x) for x in e["o_k"][p]]); Vt.append([float(x) for x in e["o_v"][p]])
                continue
            kd, vd = [], []
            for x in range(d):
                gi = x // g
                ck, cv = int(e["q_k"][p, x]), int(e["q_v"][p, x])
                if mode == "fp8":
                    ck, cv = float(O.e4m3_decode(ck)), float(O.e4m3_decode(cv))
                kd.append(ck * float(e["k_scale"][p, gi]) + float(e["k_zero"][p, gi]))
                vd.append(cv * float(e["v_scale"][p, gi]) + float(e["v_zero"][p, gi]))
                for xv, xt, s in ((kd[-1], float(_np(k)[0, 0, kvh, p, x]), float(e["k_scale"][p, gi])),
                                  (vd[-1], float(_np(v)[0, 0, kvh, p, x]), float(e["v_scale"][p, gi]))):
                    bound = s / 2 if mode != "fp8" else abs(xt) / 16 + s * 2.0 ** -10
                    assert abs(xv - xt) <= bound * (1 + 1e-6) + 1e-7
            Kt.append(kd); Vt.append(vd)
        Kt, Vt = np.array(Kt), np.array(Vt)
        assert Kt.shape == (P + 1, d)
        exp = _brute_attention(_np(q)[0, 0, kvh * G:(kvh + 1) * G], Kt, Vt, cfg.sm_scale)
        np.testing.assert_allclose(out[0, 0, kvh * G:(kvh + 1) * G], exp, rtol=1e-10, atol=1e-12)
