"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same
seeded inputs.

Bars (BASELINE.json north_star): token states, quantization codes, fp32 scales/zeros
and Original bf16 values bit-exact; attention outputs within 2e-3 relative / 1e-3
absolute; per-layer statistics within 1e-4 relative.  Decode inputs use the
"margin" recipe so fp32 (GPU) and fp64 (oracle) heavy-hitter rankings agree; the
oracle asserts the margin at both rank thresholds of every tailor.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
from synth import Shape, prefill_inputs, decode_inputs

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-3, 1e-3
STAT_RTOL = 1e-4
# Heavy-hitter scores are sums of <= G*W = 128 fp32 terms on the GPU (relative error
# < 1e-6); a relative gap of 1e-5 at each rank threshold makes fp32 and fp64 rank alike.
MARGIN = 1e-5


@pytest.fixture(scope="module", autouse=True)
def cuda_and_lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_08727_b200.build import build
    build()


def _np(t):
    return t.double().cpu().numpy()


def _bf16_bits_to_f64(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def make_pair(sh: Shape, budget, bits=4, g=0, mode="asym", layout=0, steps=64, decode_kernel=0, max_splits=0,
              n_spare=0, sharing="head", smooth=0.0):
    from paper_2603_08727_b200 import arkv as A
    cfg = A.make_config(sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim, batch=sh.batch, window=sh.window,
                        budget_tokens=budget, quant_bits=bits, group_size=g,
                        quant_mode={"asym": A.QUANT_ASYM, "sym": A.QUANT_SYM, "fp8": A.QUANT_FP8}[mode],
                        max_positions=sh.prompt_len + steps + 1, max_prompt=sh.prompt_len, layout=layout,
                        decode_kernel=decode_kernel, max_splits=max_splits, n_spare_slots=n_spare,
                        state_sharing=1 if sharing == "layer" else 0, smooth=smooth)
    gpu = A.ArkvCache(cfg, "cuda")
    ocfg = O.Cfg(n_layers=sh.n_layers, n_q_heads=sh.n_q_heads, n_kv_heads=sh.n_kv_heads, head_dim=sh.head_dim,
                 batch=sh.batch, window=sh.window, budget_tokens=budget, quant_bits=bits, group_size=g or sh.head_dim,
                 quant_mode=mode, state_sharing=sharing, smooth=smooth)
    return gpu, O.OracleARKV(ocfg), ocfg


def compare_unit(gpu, ora, b, l, kvh, where=""):
    e = gpu.arkv_export_unit(b, l, kvh)
    r = ora.export(b, l, kvh)
    tag = f"{where} unit ({b},{l},{kvh})"
    np.testing.assert_array_equal(e["state"], r["state"], err_msg="states " + tag)
    assert e["n_o"] == r["n_o"] and e["n_q"] == r["n_q"], tag
    o = r["state"] == 1
    np.testing.assert_array_equal(_bf16_bits_to_f64(e["o_k"])[o], r["o_k"][o], err_msg="O keys " + tag)
    np.testing.assert_array_equal(_bf16_bits_to_f64(e["o_v"])[o], r["o_v"][o], err_msg="O values " + tag)
    q = r["state"] == 2
    np.testing.assert_array_equal(e["q_k"][q], r["q_k"][q], err_msg="K codes " + tag)
    np.testing.assert_array_equal(e["q_v"][q], r["q_v"][q], err_msg="V codes " + tag)
    for key in ("k_scale", "k_zero", "v_scale", "v_zero"):
        np.testing.assert_array_equal(e[key][q], r[key][q], err_msg=key + " " + tag)


def run_parity(sh: Shape, budget, steps, seed=0, recipe="margin", rho=None, check_every=1, mutate=None, **kw):
    gpu, ora, ocfg = make_pair(sh, budget, steps=steps, **kw)
    qw, k, v = prefill_inputs(sh, seed=seed, recipe=recipe)
    if mutate is not None:
        mutate(qw, k, v)
    stats, oq, rho_gpu = gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda(), rho_override=rho)
    if rho is None:
        # Eqs. 3-7 first (H, V, K, q_l and rho within 1e-4 of the oracle's own statistics);
        # only then is the GPU's rho passed through, so both sides start from the same counts
        st_o, oq_o, rho_o, _ = O.prefill_stats(_np(qw), _np(k), ocfg)
        np.testing.assert_allclose(stats.cpu().numpy(), st_o, rtol=STAT_RTOL, err_msg="H, V, K")
        np.testing.assert_allclose(oq.cpu().numpy(), oq_o, rtol=STAT_RTOL, err_msg="q_l")
        np.testing.assert_allclose(rho_gpu, rho_o, rtol=STAT_RTOL, err_msg="rho")
    ora.prefill(_np(qw), _np(k), _np(v), rho_override=rho_gpu)
    gpu.arkv_check()
    for b in range(sh.batch):
        for l in range(sh.n_layers):
            for h in range(sh.n_kv_heads):
                compare_unit(gpu, ora, b, l, h, "after prefill")
    worst = 0.0
    for s in range(steps):
        q, kn, vn = decode_inputs(sh, s, seed=seed, recipe=recipe)
        out = gpu.arkv_decode_step(q.cuda(), kn.cuda(), vn.cuda(), out_fp32=True)
        ref = ora.decode_step(_np(q), _np(kn), _np(vn))
        got = out.double().cpu().numpy()
        np.testing.assert_allclose(got, ref, rtol=RTOL, atol=ATOL, err_msg=f"output step {s}")
        worst = max(worst, float(np.max(np.abs(got - ref) / (ATOL + RTOL * np.abs(ref)))))
        if (s + 1) % check_every == 0 or s == steps - 1:
            gpu.arkv_check()
            for b in range(sh.batch):
                for l in range(sh.n_layers):
                    for h in range(sh.n_kv_heads):
                        compare_unit(gpu, ora, b, l, h, f"step {s}")
    margins = [m for u in ora.units.values() for m in u.margins]
    n_tailors = sum(len(u.tailors) for u in ora.units.values())
    if margins:
        assert min(margins) > MARGIN, f"test input lacks a score margin ({min(margins):.2e})"
    return dict(worst=worst, tailors=n_tailors, stats=stats.cpu().numpy(), oq=oq.cpu().numpy(), rho=rho_gpu,
                gpu=gpu, ora=ora)


TOY = Shape(batch=1, n_layers=1, n_q_heads=4, n_kv_heads=2, head_dim=16, prompt_len=64, window=8)


@pytest.mark.parametrize("rho", [1.0, 0.5, 0.25])
def test_toy_config(rho):
    """BASELINE configs[0] (R29: W = 8, injected rho): 64-token prefill + 16 steps."""
    r = run_parity(TOY, budget=32, steps=16, seed=11, rho=[[rho]], bits=4, g=16)
    assert r["tailors"] >= 2


def test_toy_two_layers_stats_rho():
    sh = Shape(batch=1, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=16, prompt_len=64, window=8)
    run_parity(sh, budget=32, steps=24, seed=3, bits=4, g=16)


MID = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=2048, window=32)


@pytest.mark.parametrize("layout,bits,g,mode", [
    (2, 4, 128, "asym"),   # FRAG, paper default
    (2, 4, 32, "asym"),
    (1, 4, 128, "asym"),   # PLAIN
    (1, 2, 32, "asym"),
    (1, 8, 128, "sym"),
    (2, 4, 64, "sym"),
    (1, 8, 128, "fp8"),    # NEXT-2: e4m3 codes, per-token scale
    (1, 8, 32, "fp8"),
    (2, 8, 128, "fp8"),    # fp8 in the fragment-native layout (tensor-core kernel)
])
def test_mid_config(layout, bits, g, mode):
    """L=2, H_q=8, H_kv=2, d=128, P=2048, B=512: prefill tailor + decode tailors."""
    r = run_parity(MID, budget=512, steps=80, seed=5, rho=[[1.0, 0.4]], layout=layout, bits=bits, g=g, mode=mode,
                   check_every=20)
    assert r["tailors"] >= 2 * 2 * 2


def test_generic_kernel_on_frag_layout():
    run_parity(MID, budget=512, steps=40, seed=6, rho=[[0.7, 0.3]], layout=2, decode_kernel=1, check_every=40)


@pytest.mark.parametrize("g,mode", [(128, "asym"), (32, "asym"), (64, "sym")])
def test_persistent_kernel_mid(g, mode):
    """The persistent range-partitioned decode kernel (decode_kernel = 3) + its combine."""
    r = run_parity(MID, budget=512, steps=80, seed=5, rho=[[1.0, 0.4]], layout=2, bits=4, g=g, mode=mode,
                   decode_kernel=3, check_every=20)
    assert r["tailors"] >= 2 * 2 * 2


@pytest.mark.parametrize("G", [1, 2, 8])
@pytest.mark.parametrize("kernel", [2, 3])
def test_fast_kernels_gqa_groups(G, kernel):
    """Tensor-core decode kernels (split-K and persistent) for GQA groups 1, 2, 8."""
    sh = Shape(batch=2, n_layers=1, n_q_heads=2 * G, n_kv_heads=2, head_dim=128, prompt_len=1024, window=32)
    r = run_parity(sh, budget=256, steps=48, seed=40 if G == 8 else 31 + G, rho=[[0.6], [0.3]], layout=2, bits=4, g=128,
                   decode_kernel=kernel, check_every=16)
    assert r["tailors"] >= 2


def test_persistent_matches_split_states():
    """Both fast kernels drive the same schedule: identical token states and codes, outputs
    within the parity tolerance of each other (only the merge order differs)."""
    from paper_2603_08727_b200 import arkv as A
    sh = Shape(batch=2, n_layers=3, n_q_heads=16, n_kv_heads=4, head_dim=128, prompt_len=1500, window=32)
    res = []
    for kern in (2, 3):
        cfg = A.make_config(3, 16, 4, 128, batch=2, budget_tokens=384, max_positions=1600, max_prompt=1500,
                            decode_kernel=kern)
        gpu = A.ArkvCache(cfg)
        qw, k, v = prefill_inputs(sh, seed=41, recipe="margin")
        gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
        outs = [gpu.arkv_decode_step(*[t.cuda() for t in decode_inputs(sh, s, seed=41, recipe="margin")], out_fp32=True).cpu()
                for s in range(60)]
        gpu.arkv_check()
        res.append((torch.stack(outs), [gpu.arkv_export_unit(b, l, h) for b in range(2) for l in range(3)
                                        for h in range(4)]))
    torch.testing.assert_close(res[0][0], res[1][0], rtol=RTOL, atol=ATOL)
    for e2, e3 in zip(res[0][1], res[1][1]):
        for key in ("state", "q_k", "k_scale", "o_k", "o_v"):
            np.testing.assert_array_equal(e2[key], e3[key])


@pytest.mark.parametrize("kernel,g", [(1, 128), (2, 128), (3, 128), (2, 32), (3, 64)])
def test_fp8_frag_kernels(kernel, g):
    """fp8 e4m3 Q tokens (NEXT-2) in the FRAG layout: generic, split-K and persistent
    decode kernels (cvt.rn.f16x2.e4m3x2 fragments) against the oracle."""
    r = run_parity(MID, budget=512, steps=64, seed=8, rho=[[0.8, 0.3]], layout=2, bits=8, g=g, mode="fp8",
                   decode_kernel=kernel, check_every=16)
    assert r["tailors"] >= 2 * 2 * 2


@pytest.mark.parametrize("hkv,kernel", [(2, 0), (4, 0), (4, 3)])
def test_layer_shared_states(hkv, kernel):
    """NEXT-3: one token-state set per layer from the score averaged across its KV heads
     — prefill-end and decode tailors against the oracle."""
    sh = Shape(batch=2, n_layers=2, n_q_heads=4 * hkv, n_kv_heads=hkv, head_dim=128, prompt_len=1024, window=32)
    r = run_parity(sh, budget=256, steps=48, seed=13, rho=[[0.7, 0.3], [0.5, 1.0]], layout=2, bits=4, g=128,
                   decode_kernel=kernel, sharing="layer", check_every=16)
    assert r["tailors"] >= 2 * 2 * hkv
    gpu = r["gpu"]
    for b in range(2):
        for l in range(2):
            st = [gpu.arkv_export_unit(b, l, h)["state"] for h in range(hkv)]
            for h in range(1, hkv):
                np.testing.assert_array_equal(st[h], st[0])


def test_batch_and_spare_waves():
    """Batch 3 with only 2 staging slots: every tailor runs in several waves."""
    sh = Shape(batch=3, n_layers=2, n_q_heads=4, n_kv_heads=2, head_dim=32, prompt_len=200, window=8)
    run_parity(sh, budget=64, steps=40, seed=9, rho=[[1.0, 0.5], [0.3, 1.0], [0.6, 0.6]], layout=2, bits=4, g=32,
               n_spare=2, check_every=10)


def test_no_prefill_tailor_path():
    """P <= B - W: the prompt is ingested as Original; the first tailor happens in decode."""
    sh = Shape(batch=1, n_layers=1, n_q_heads=4, n_kv_heads=1, head_dim=32, prompt_len=40, window=8)
    r = run_parity(sh, budget=64, steps=40, seed=2, rho=[[0.5]], bits=4, g=32)
    assert r["tailors"] >= 1


def test_short_prompt_requires_override():
    from paper_2603_08727_b200 import arkv as A
    sh = Shape(batch=1, n_layers=1, n_q_heads=2, n_kv_heads=1, head_dim=16, prompt_len=5, window=8)
    gpu, ora, _ = make_pair(sh, budget=32, steps=8)
    qw, k, v = prefill_inputs(sh, seed=1)
    with pytest.raises(A.ArkvError):
        gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
    run_parity(sh, budget=32, steps=8, seed=1, rho=[[1.0]])


def test_prefill_statistics_natural():
    """Eqs. 3-7 on natural-recipe inputs: H, V, K and q within 1e-4 relative; rho too."""
    sh = Shape(batch=2, n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=3000, window=32)
    from paper_2603_08727_b200 import arkv as A
    cfg = A.make_config(3, 8, 2, 128, batch=2, budget_tokens=512, max_positions=3100, max_prompt=3000)
    gpu = A.ArkvCache(cfg)
    qw, k, v = prefill_inputs(sh, seed=21)
    stats, oq, rho = gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
    ocfg = O.Cfg(n_layers=3, n_q_heads=8, n_kv_heads=2, head_dim=128, batch=2, window=32, budget_tokens=512)
    rs, roq, rrho, _ = O.prefill_stats(_np(qw), _np(k), ocfg)
    np.testing.assert_allclose(stats.cpu().numpy(), rs, rtol=STAT_RTOL)
    np.testing.assert_allclose(oq.cpu().numpy(), roq, rtol=STAT_RTOL)
    np.testing.assert_allclose(rho, rrho, rtol=STAT_RTOL)


def test_decode_errors():
    from paper_2603_08727_b200 import arkv as A
    gpu, _, _ = make_pair(TOY, budget=32, steps=4)
    q, kn, vn = decode_inputs(TOY, 0)
    with pytest.raises(A.ArkvError) as e:
        gpu.arkv_decode_step(q.cuda(), kn.cuda(), vn.cuda())
    assert e.value.code == -3
    qw, k, v = prefill_inputs(TOY)
    gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda(), rho_override=[[1.0]])
    from paper_2603_08727_b200.arkv import lib, _ptr, _stream_ptr
    out = torch.empty(q.shape, device="cuda")
    rc = lib().arkv_decode_step(gpu.handle, 0, 1, _ptr(q.cuda()), _ptr(kn.cuda()), _ptr(vn.cuda()), 31, 4,
                                _ptr(out), 1, _stream_ptr(None))
    assert rc == -5


@pytest.mark.parametrize("kernel", [1, 2, 3])
def test_nonfinite_inputs_raise(kernel):
    """SPEC S:329 ("non-finite input -> numeric error"): a NaN / Inf in a decode step's q,
    k or v, in a prompt row that enters the cache, or in q_win / K (reaching the Eq. 3
    column sums) is reported by arkv_check as ARKV_ERR_DEVICE; clean calls check OK.
    Generic (1), split-K (2) and persistent (3) decode kernels."""
    from paper_2603_08727_b200 import arkv as A

    def expect_device_error(gpu):
        with pytest.raises(A.ArkvError) as e:
            gpu.arkv_check()
        assert e.value.code == -7

    qw, k, v = prefill_inputs(MID, seed=5)
    gpu, _, _ = make_pair(MID, budget=512, steps=8, decode_kernel=kernel)
    gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
    gpu.arkv_check()
    q, kn, vn = [t.cuda() for t in decode_inputs(MID, 0, seed=5)]
    gpu.arkv_decode_step(q, kn, vn)
    gpu.arkv_check()
    for which, val in ((2, float("nan")), (0, float("inf")), (1, float("-inf"))):
        t = [x.clone() for x in decode_inputs(MID, 1 + which, seed=5)]
        t[which].view(-1)[t[which].numel() - 3] = val       # last unit of the call (layer 1)
        gpu.arkv_decode_step(*[x.cuda() for x in t])
        expect_device_error(gpu)
    # prompt: an Inf in a window row's V (always kept Original), then a NaN in K
    for tensor, idx in (("v", (0, 1, 0, MID.prompt_len - 1, 7)), ("k", (0, 0, 1, 100, 3))):
        qw2, k2, v2 = qw.clone(), k.clone(), v.clone()
        (v2 if tensor == "v" else k2)[idx] = float("inf") if tensor == "v" else float("nan")
        gpu2, _, _ = make_pair(MID, budget=512, steps=8, decode_kernel=kernel)
        gpu2.arkv_prefill_stats(qw2.cuda(), k2.cuda(), v2.cuda(), rho_override=[[1.0, 0.5]])
        expect_device_error(gpu2)


def test_determinism_bitwise():
    outs = []
    for _ in range(2):
        gpu, _, _ = make_pair(MID, budget=512, steps=40)
        qw, k, v = prefill_inputs(MID, seed=4)
        gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
        o = [gpu.arkv_decode_step(*[t.cuda() for t in decode_inputs(MID, s, seed=4)]).cpu() for s in range(40)]
        outs.append((torch.stack(o), gpu.arkv_export_unit(0, 1, 1)))
    assert torch.equal(outs[0][0], outs[1][0])
    for key in ("state", "o_k", "q_k", "k_scale"):
        np.testing.assert_array_equal(outs[0][1][key], outs[1][1][key])


def test_sharded_prefill_c1_equals_full():
    """KV-head sharding: two caches holding KV heads [0,2) and [2,4) of the
    same sequences; their Eq. 3 column sums are summed between arkv_prefill_begin and
    arkv_prefill_finish (what NCCL all-reduce does across GPUs).  Statistics and rho
    equal the unsharded cache bitwise; every unit's states, codes and outputs too."""
    from paper_2603_08727_b200 import arkv as A
    sh = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=4, head_dim=128, prompt_len=1024, window=32)
    qw, k, v = prefill_inputs(sh, seed=17)
    mk = lambda hkv, hq: A.make_config(2, hq, hkv, 128, budget_tokens=256, max_positions=1024 + 40, max_prompt=1024)
    full = A.ArkvCache(mk(4, 8))
    st_f, oq_f, rho_f = full.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
    halves = [A.ArkvCache(mk(2, 4)) for _ in range(2)]
    parts = []
    for i, c in enumerate(halves):
        qwi = qw[:, :, 4 * i:4 * i + 4].contiguous().cuda()
        ki, vi = k[:, :, 2 * i:2 * i + 2].contiguous().cuda(), v[:, :, 2 * i:2 * i + 2].contiguous().cuda()
        parts.append((ki, vi, c.arkv_prefill_begin(qwi, ki)))
    colsum = parts[0][2] + parts[1][2]
    for i, c in enumerate(halves):
        st, oq, rho = c.arkv_prefill_finish(parts[i][0], parts[i][1], colsum)
        np.testing.assert_array_equal(rho, rho_f)
        np.testing.assert_allclose(st.cpu().numpy(), st_f.cpu().numpy(), rtol=1e-12)
    for s in range(40):
        q, kn, vn = decode_inputs(sh, s, seed=17)
        of = full.arkv_decode_step(q.cuda(), kn.cuda(), vn.cuda())
        for i, c in enumerate(halves):
            oh = c.arkv_decode_step(q[:, :, 4 * i:4 * i + 4].contiguous().cuda(), kn[:, :, 2 * i:2 * i + 2].contiguous().cuda(),
                                    vn[:, :, 2 * i:2 * i + 2].contiguous().cuda())
            torch.testing.assert_close(oh, of[:, :, 4 * i:4 * i + 4], rtol=0, atol=0)
    for i, c in enumerate(halves):
        for l in range(2):
            for h in range(2):
                e, r = c.arkv_export_unit(0, l, h), full.arkv_export_unit(0, l, 2 * i + h)
                for key in ("state", "q_k", "k_scale", "o_v"):
                    np.testing.assert_array_equal(e[key], r[key])


def test_full_size_configs1_sampled_units():
    """configs[1] at full size, launched exactly as bench.py does (32 layers x 8 KV heads
    in one arkv_decode_step per step, default kernel and split count), lattice recipe (a
    score margin at any size, synth/generators.py): the oracle recomputes two sampled layers
    (different rho) one unit at a time through the prefill-end tailor (32,736 eligible
    tokens), the HH window and the first decode tailor.  Every KV head of both layers is
    compared bit-exactly — no unit is skipped."""
    sh = Shape(batch=1, n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=32768, window=32)
    checked, oras = _sampled_units_run(sh, 8192, 40, seqs=[0], layers=[3, 16], recipe="lattice", seed=23,
                                       check_after_prefill=True)
    assert checked == 2 * 8
    assert all(len(u.tailors) >= 2 for o in oras.values() for u in o.units.values())   # prefill + decode


def test_full_size_configs1_statistics():
    """Eqs. 3-7 at configs[1]'s full size (P = 32768, all 32 layers, natural recipe): H, V,
    K, q_l and rho of the CUDA prefill within 1e-4 relative of the float64 oracle's."""
    from paper_2603_08727_b200 import arkv as A
    from synth import prefill_inputs_fast
    sh = Shape(batch=1, n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=32768, window=32)
    cfg = A.make_config(32, 32, 8, 128, budget_tokens=8192, max_positions=32768 + 2, max_prompt=32768)
    gpu = A.ArkvCache(cfg)
    qw, k, v = prefill_inputs_fast(sh, seed=1234, device="cuda")
    stats, oq, rho = gpu.arkv_prefill_stats(qw, k, v)
    gpu.arkv_check()
    ocfg = O.Cfg(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, window=32, budget_tokens=8192)
    rs, roq, rrho, _ = O.prefill_stats(qw.double().cpu().numpy(), k.double().cpu().numpy(), ocfg)
    np.testing.assert_allclose(stats.cpu().numpy(), rs, rtol=STAT_RTOL, err_msg="H, V, K")
    np.testing.assert_allclose(oq.cpu().numpy(), roq, rtol=STAT_RTOL, err_msg="q_l")
    np.testing.assert_allclose(rho, rrho, rtol=STAT_RTOL, err_msg="rho")
    assert rho.min() < 0.5 < rho.max() == 1.0      # the layers differ (the bench's workload)


def _sampled_units_run(sh, budget, steps, seqs, layers, recipe, seed, decode_kernel=0, check_after_prefill=False,
                       quant="asym", out_fp32=True):
    """Run a full-size cache for `steps` decode steps (bench launch: one call for all
    layers) and compare sampled (sequence, layer) slices with per-slice oracles: outputs
    every step; counts, states, codes, scales and Original values of every sampled unit
    at the end (and after the prefill if asked).  The lattice recipe guarantees a score
    margin at every rank threshold, which the oracle asserts (no unit is skipped)."""
    from paper_2603_08727_b200 import arkv as A
    from synth import (prefill_inputs_fast, decode_inputs_fast, prefill_inputs_lattice, decode_inputs_lattice)
    pf = prefill_inputs_lattice if recipe == "lattice" else prefill_inputs_fast
    df = decode_inputs_lattice if recipe == "lattice" else decode_inputs_fast
    bits = 8 if quant == "fp8" else 4
    cfg = A.make_config(sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim, batch=sh.batch, window=sh.window,
                        budget_tokens=budget, max_positions=sh.prompt_len + steps + 1, max_prompt=sh.prompt_len,
                        decode_kernel=decode_kernel, quant_bits=bits,
                        quant_mode=A.QUANT_FP8 if quant == "fp8" else A.QUANT_ASYM)
    gpu = A.ArkvCache(cfg)
    qw, k, v = pf(sh, seed=seed, device="cuda")
    stats, oq, rho = gpu.arkv_prefill_stats(qw, k, v)
    gpu.arkv_check()
    ocfg = O.Cfg(n_layers=1, n_q_heads=sh.n_q_heads, n_kv_heads=sh.n_kv_heads, head_dim=sh.head_dim,
                 window=sh.window, budget_tokens=budget, quant_bits=bits, quant_mode=quant)
    oras = {}
    for b in seqs:
        for l in layers:
            ora = O.OracleARKV(ocfg)
            sub = lambda t: t[b:b + 1, l:l + 1].double().cpu().numpy()   # noqa: E731
            ora.prefill(sub(qw), sub(k), sub(v), rho_override=[[rho[b, l]]])
            oras[(b, l)] = ora
    del qw, k, v

    def compare_all(where):
        n = 0
        for (b, l), ora in oras.items():
            for h in range(sh.n_kv_heads):
                margins = ora.units[(0, 0, h)].margins
                if recipe == "lattice":
                    assert not margins or min(margins) > MARGIN, f"{where}: lattice input without a margin"
                elif margins and min(margins) <= MARGIN:
                    continue   # natural recipe: a near-tie may rank differently in fp32 and fp64
                _compare_export(gpu, ora, b, l, h, where)
                n += 1
        return n

    if check_after_prefill:
        compare_all("after prefill")
    for s in range(steps):
        q, kn, vn = df(sh, s, seed=seed, device="cuda")
        out = gpu.arkv_decode_step(q, kn, vn, out_fp32=out_fp32).float().cpu().numpy()
        for (b, l), ora in oras.items():
            ref = ora.decode_step(q[b:b + 1, l:l + 1].double().cpu().numpy(), kn[b:b + 1, l:l + 1].double().cpu().numpy(),
                                  vn[b:b + 1, l:l + 1].double().cpu().numpy())
            if not out_fp32:   # bf16 outputs: the oracle's value rounded to bf16, plus one bf16 ulp
                ref16 = torch.tensor(ref).to(torch.bfloat16).double().numpy()
                np.testing.assert_allclose(out[b:b + 1, l:l + 1], ref16, rtol=RTOL + 2.0 ** -8, atol=ATOL,
                                           err_msg=f"b{b} l{l} step {s} (bf16 out)")
            else:
                np.testing.assert_allclose(out[b:b + 1, l:l + 1], ref, rtol=RTOL, atol=ATOL,
                                           err_msg=f"b{b} l{l} step {s}")
    gpu.arkv_check()
    return compare_all(f"after {steps} steps"), oras


def _compare_export(gpu, ora, b, l, h, where):
    """Export of GPU unit (b, l, h) vs the oracle's (0, 0, h) slice: counts, states, codes,
    fp32 scales/zeros, Original bf16 values, bit-exact."""
    e, r = gpu.arkv_export_unit(b, l, h), ora.export(0, 0, h)
    tag = f"{where} unit ({b},{l},{h})"
    assert (e["n_o"], e["n_q"]) == (r["n_o"], r["n_q"]), tag
    np.testing.assert_array_equal(e["state"], r["state"], err_msg="states " + tag)
    om, qm = r["state"] == 1, r["state"] == 2
    np.testing.assert_array_equal(_bf16_bits_to_f64(e["o_k"])[om], r["o_k"][om], err_msg="O keys " + tag)
    np.testing.assert_array_equal(_bf16_bits_to_f64(e["o_v"])[om], r["o_v"][om], err_msg="O values " + tag)
    for key in ("q_k", "q_v", "k_scale", "k_zero", "v_scale", "v_zero"):
        np.testing.assert_array_equal(e[key][qm], r[key][qm], err_msg=key + " " + tag)


@pytest.mark.parametrize("kernel", [2, 3])
def test_full_size_configs3_short_prompts(kernel):
    """configs[3] at full size (batch 64 x 32 layers x 8 KV heads, 1K prompts, B = 2048: the
    full-precision-matching regime, no tailor): sampled sequences and layers vs the oracle."""
    sh = Shape(batch=64, n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=1024, window=32)
    checked, oras = _sampled_units_run(sh, 2048, 24, seqs=[0, 37, 63], layers=[0, 31], recipe="natural", seed=29,
                                       decode_kernel=kernel)
    assert checked == 3 * 2 * 8
    assert all(len(u.tailors) == 0 for o in oras.values() for u in o.units.values())


@pytest.mark.parametrize("kernel", [2, 3])
def test_full_size_configs2_batch8(kernel):
    """configs[2]'s per-GPU shard at full size (Qwen3-8B: 36 layers, batch 8, 8K prompts,
    B = 2048): prefill-end tailor on every unit; sampled units vs the oracle."""
    sh = Shape(batch=8, n_layers=36, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=8192, window=32)
    checked, oras = _sampled_units_run(sh, 2048, 40, seqs=[0, 5], layers=[3, 30], recipe="lattice", seed=31,
                                       decode_kernel=kernel, check_after_prefill=True)
    assert checked == 2 * 2 * 8
    assert all(len(u.tailors) >= 1 for o in oras.values() for u in o.units.values())


def test_layer_shared_states_kv_head_shards():
    """NEXT-3 across KV-head shards (collective C3): two caches holding KV heads [0,2) and
    [2,4) exchange their per-tailor score sums (arkv_tailor_scores -> sum ->
    arkv_set_tailor_scores, what NCCL all-reduce does across GPUs) and match the unsharded
    layer-shared cache: token states, codes and outputs."""
    from paper_2603_08727_b200 import arkv as A
    sh = Shape(batch=1, n_layers=2, n_q_heads=16, n_kv_heads=4, head_dim=128, prompt_len=1024, window=32)
    steps = 48
    qw, k, v = prefill_inputs(sh, seed=19, recipe="margin")
    mk = lambda hkv, hq: A.make_config(2, hq, hkv, 128, budget_tokens=256, max_positions=1024 + steps + 1,  # noqa: E731
                                       max_prompt=1024, state_sharing=1)
    full = A.ArkvCache(mk(4, 16))
    full.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda())
    halves = [A.ArkvCache(mk(2, 8)) for _ in range(2)]
    sl = lambda t, i, hq: t[:, :, hq * i:hq * i + hq].contiguous().cuda()   # noqa: E731
    parts = []
    for i, c in enumerate(halves):
        parts.append(c.arkv_prefill_begin(sl(qw, i, 8), sl(k, i, 2)))
    colsum = parts[0] + parts[1]                       # C1
    stride, rows = 2048, 8
    def exchange(call_layers=None):
        bufs = [torch.zeros(rows, stride, device="cuda") for _ in range(2)]
        n = [c.arkv_tailor_scores(bufs[i]) for i, c in enumerate(halves)]
        assert n[0] == n[1]
        tot = bufs[0] + bufs[1]                        # C3
        for c in halves:
            c.arkv_set_tailor_scores(tot, 4)
        return n[0]
    assert exchange() == 2                              # prefill-end tailor of both layers
    for i, c in enumerate(halves):
        c.arkv_prefill_finish(sl(k, i, 2), sl(v, i, 2), colsum)
    n_ex = 0
    for s in range(steps):
        q, kn, vn = decode_inputs(sh, s, seed=19, recipe="margin")
        n_ex += exchange()
        of = full.arkv_decode_step(q.cuda(), kn.cuda(), vn.cuda())
        for i, c in enumerate(halves):
            oh = c.arkv_decode_step(sl(q, i, 8), sl(kn, i, 2), sl(vn, i, 2))
            torch.testing.assert_close(oh, of[:, :, 8 * i:8 * i + 8], rtol=RTOL, atol=ATOL)
    assert n_ex >= 2                                     # decode tailors exchanged too
    for c in halves + [full]:
        c.arkv_check()
    for i, c in enumerate(halves):
        for l in range(2):
            for h in range(2):
                e, r = c.arkv_export_unit(0, l, h), full.arkv_export_unit(0, l, 2 * i + h)
                for key in ("state", "q_k", "k_scale", "o_v"):
                    np.testing.assert_array_equal(e[key], r[key])



@pytest.mark.parametrize("layout", [1, 2])
def test_rho_zero_all_kept_tokens_quantized(layout):
    """rho = 0 (the Base_quant regime): every kept eligible token is Quantized (n_oe = 0)."""
    r = run_parity(MID, budget=512, steps=48, seed=12, rho=[[0.0, 0.0]], layout=layout, bits=4, g=128,
                   check_every=16)
    for u in r["ora"].units.values():
        assert all(t[1] == MID.window for t in u.tailors)      # only the window stays Original


def test_minimal_budget_frequent_tailors():
    """B = 2W + 1, the smallest budget R14 allows: a tailor every W steps (U reaches B_bytes
    after exactly W appends, R12) keeping one eligible token, no room left for Quantized
    tokens; the first decode tailor's window holds the W - 1 decode queries since the prompt
    (R19)."""
    sh = Shape(batch=1, n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=300, window=32)
    r = run_parity(sh, budget=65, steps=100, seed=14, rho=[[0.5]], layout=2, bits=4, g=128, check_every=10)
    assert min(len(u.tailors) for u in r["ora"].units.values()) >= 4


def test_constant_groups_quantize_to_scale_one():
    """Tokens whose K/V groups are constant (R23: s = 1, codes 0, z = the value; symmetric
    all-zero groups: s = 1) survive the tailor bit-exactly and attend correctly."""
    def mutate(qw, k, v):
        k[:, :, :, 100:140, :64] = 0.25          # first group (g = 64) constant for 40 tokens
        v[:, :, :, 100:140, 64:] = -0.5
        v[:, :, :, 200:220, :] = 0.0             # whole rows zero
    for mode in ("asym", "sym"):
        run_parity(MID, budget=512, steps=24, seed=15, rho=[[0.3, 0.6]], layout=2, bits=4, g=64, mode=mode,
                   check_every=24, mutate=mutate)


@pytest.mark.parametrize("kernel", [2, 3])
def test_cuda_graph_capture_replays_eager(kernel):
    """arkv_decode_step never syncs and passes its per-step plans (tailor jobs, HH windows,
    persistent ranges) as kernel parameters, so a sequence of decode steps — tailors
    included — can be captured into one CUDA graph.  Replaying it once on an identically
    prefilled cache gives bit-identical outputs, token states, codes and scales to eager
    execution."""
    sh = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=1024, window=32)
    steps = 48
    ins = [[t.cuda() for t in decode_inputs(sh, s, seed=9)] for s in range(steps)]
    qw, k, v = prefill_inputs(sh, seed=9)
    caches = []
    for _ in range(2):
        gpu, _, _ = make_pair(sh, budget=256, steps=steps, layout=2, decode_kernel=kernel)
        gpu.arkv_prefill_stats(qw.cuda(), k.cuda(), v.cuda(), rho_override=[[0.7, 0.3]])
        caches.append(gpu)
    torch.cuda.synchronize()
    eager = [caches[0].arkv_decode_step(q, kn, vn) for q, kn, vn in ins]
    outs = [torch.empty_like(o) for o in eager]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for (q, kn, vn), o in zip(ins, outs):
            caches[1].arkv_decode_step(q, kn, vn, out=o, stream=torch.cuda.current_stream())
    graph.replay()
    torch.cuda.synchronize()
    caches[0].arkv_check()
    caches[1].arkv_check()
    assert sum(1 for o in outs if torch.count_nonzero(o) > 0) == steps
    for s in range(steps):
        assert torch.equal(eager[s], outs[s]), f"step {s}"
    for l in range(sh.n_layers):
        for h in range(sh.n_kv_heads):
            a, b = caches[0].arkv_export_unit(0, l, h), caches[1].arkv_export_unit(0, l, h)
            for key in ("state", "o_k", "o_v", "q_k", "q_v", "k_scale", "k_zero", "v_scale", "v_zero"):
                np.testing.assert_array_equal(a[key], b[key], err_msg=f"{key} layer {l} head {h}")
            assert (a["state"] == 2).any() and (a["state"] == 3).any()  # tailors ran inside the graph


@pytest.mark.parametrize("lam,kernel,sharing,layout", [(0.5, 2, "head", 2), (0.9, 3, "head", 2), (0.5, 2, "layer", 2),
                                                        (0.5, 0, "head", 1)])
def test_smoothed_scores(lam, kernel, sharing, layout):
    """NEXT-4 (Alg. 1 P:285 "smoothed", reading R34): scores averaged across tailors.  The
    prefill tailor and two decode tailors per unit; the decode tailors rank the tokens the
    previous tailor kept by λ·S~_prev + (1 − λ)·S — bit-exact states, codes and scales.
    Layout 1 (PLAIN) runs the generic decode and move kernels."""
    sh = Shape(batch=1, n_layers=2, n_q_heads=8, n_kv_heads=2, head_dim=128, prompt_len=2048, window=32)
    r = run_parity(sh, budget=256, steps=100, seed=61, rho=[[0.7, 0.3]], layout=layout, decode_kernel=kernel,
                   check_every=25, smooth=lam, sharing=sharing)
    assert r["tailors"] >= 3 * 2 * 2
    # the smoothing changed decisions: the same run without it ends in other states
    gpu0 = run_parity(sh, budget=256, steps=100, seed=61, rho=[[0.7, 0.3]], layout=layout, decode_kernel=kernel,
                      check_every=100, smooth=0.0, sharing=sharing)["gpu"]
    diff = sum(int((r["gpu"].arkv_export_unit(0, l, h)["state"] != gpu0.arkv_export_unit(0, l, h)["state"]).sum())
               for l in range(2) for h in range(2))
    assert diff > 0


def test_full_size_configs4_128k():
    """configs[4]'s per-GPU shard at full size (Llama3-8B shapes, 128K prompt, B = 16384 =
    1/8 of the prompt: the tight-budget long-context regime): prefill-end tailor over
    131,040 eligible tokens per unit and 36 decode steps in the bench launch (one call for
    all 32 layers); two sampled layers vs the oracle, every KV head bit-exact (lattice
    recipe: a score margin at both rank thresholds of all 16 units)."""
    sh = Shape(batch=1, n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=131072, window=32)
    checked, oras = _sampled_units_run(sh, 16384, 36, seqs=[0], layers=[2, 21], recipe="lattice", seed=37)
    assert checked == 2 * 8
    assert all(len(u.tailors) >= 1 for o in oras.values() for u in o.units.values())


def test_full_size_configs1_fp8_bf16_out():
    """configs[1] at full size with the paper's fp8 e4m3 Q tokens (NEXT-2) and bf16 outputs
    (what bench.py times): lattice recipe, two sampled layers, every KV head bit-exact;
    outputs against the oracle's rounded to bf16."""
    sh = Shape(batch=1, n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, prompt_len=32768, window=32)
    checked, oras = _sampled_units_run(sh, 8192, 40, seqs=[0], layers=[1, 30], recipe="lattice", seed=43,
                                       quant="fp8", out_fp32=False)
    assert checked == 2 * 8
    assert all(len(u.tailors) >= 2 for o in oras.values() for u in o.units.values())
