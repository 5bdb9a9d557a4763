"""The lattice input recipe (synth/generators.py) delivers what the full-size GPU parity
tests rely on: exact logits on a lattice (q.k = 2^-e L in fp32 AND fp64), quantization
groups with min 0 / max 1 (exact codes), and a heavy-hitter score margin at every rank
threshold of every tailor (checked by the oracle)."""
import numpy as np
import torch

import oracle as O
from synth import Shape, decode_inputs_lattice, lattice_exponent, prefill_inputs_lattice


SH = Shape(batch=1, n_layers=4, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=1024, window=32)


def test_lattice_logits_exact_in_fp32():
    qw, k, v = prefill_inputs_lattice(SH, seed=3)
    for l in range(SH.n_layers):
        e = lattice_exponent(SH, l)
        q = qw[0, l, 0, 0]
        for h in range(SH.n_kv_heads):
            kk = k[0, l, h]
            bits = kk[:, :18].double().numpy()
            lev = (bits * (2.0 ** np.arange(18))).sum(axis=1)
            exact = lev * 2.0 ** -e
            f64 = kk.double().numpy() @ q.double().numpy()
            f32 = (kk.float() @ q.float()).double().numpy()
            np.testing.assert_array_equal(f64, exact)
            np.testing.assert_array_equal(f32, exact)
            assert (lev % 2 == 0).all()                            # prompt levels are even
            blocks = kk.float().view(-1, 4, 32)
            assert (blocks.amin(-1) == 0).all() and (blocks.amax(-1) == 1).all()
        assert torch.equal(qw[0, l], q.expand_as(qw[0, l]))       # one query per layer
    q, kn, vn = decode_inputs_lattice(SH, 5, seed=3)
    lev = (kn[..., :18].double() * 2.0 ** torch.arange(18, dtype=torch.float64)).sum(-1)
    assert (lev % 2 == 1).all() and (lev < 2 * SH.prompt_len).all()   # decode levels are odd


def test_lattice_margins_hold_in_the_oracle():
    qw, k, v = prefill_inputs_lattice(SH, seed=3)
    cfg = O.Cfg(n_layers=4, n_q_heads=8, n_kv_heads=2, head_dim=128, window=32, budget_tokens=256)
    ora = O.OracleARKV(cfg)
    f = lambda t: t.double().numpy()  # noqa: E731
    _, _, rho, _ = O.prefill_stats(f(qw), f(k), cfg)
    assert rho.min() < 0.6                                          # some layers quantize heavily
    ora.prefill(f(qw), f(k), f(v))
    for s in range(80):
        ora.decode_step(*[f(t) for t in decode_inputs_lattice(SH, s, seed=3)])
    margins = [m for u in ora.units.values() for m in u.margins]
    assert sum(len(u.tailors) for u in ora.units.values()) >= 16
    assert min(margins) > 1e-4
    assert any((ora.export(0, l, h)["state"] == 2).any() for l in range(4) for h in range(2))   # Q tokens exist
