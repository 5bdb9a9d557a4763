"""CPU-only checks of the C ABI: the library builds/loads without a GPU, exports every
symbol include/arkv.h declares, and its host logic (count schedule, OQ score) equals
the oracle's independent implementation."""
import ctypes
import math
import os
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle as O
from paper_2603_08727_b200 import arkv as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2603_08727_b200.build import build
    build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "arkv.h")).read()
    declared = set(re.findall(r"\b(arkv_[a-z_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = A.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(A.EXPORTED) <= declared


def test_version_and_status_strings():
    assert "sm_100a" in A.arkv_version()
    assert A.lib().arkv_status_string(-4).decode().startswith("prompt shorter")


def test_config_validation():
    c = A.make_config(1, 4, 3, 16)          # H_q % H_kv != 0
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    c = A.make_config(1, 4, 2, 16, window=8, budget_tokens=16)   # B <= 2W (R14)
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    c = A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, quant_bits=3)
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    c = A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, layout=A.LAYOUT_FRAG)  # d % 32 != 0
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    c = A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, quant_bits=4, quant_mode=A.QUANT_FP8)  # fp8 is 8-bit
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    a, w = A.arkv_cache_bytes(A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, max_positions=128))
    assert a > 0 and w > 0
    c = A.make_config(1, 8, 4, 16, window=8, budget_tokens=32, state_sharing=1, n_spare_slots=2)  # < H_kv spares
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    c = A.make_config(1, 8, 4, 16, window=8, budget_tokens=32, state_sharing=2)
    with pytest.raises(A.ArkvError):
        A.arkv_cache_bytes(c)
    a8, _ = A.arkv_cache_bytes(A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, max_positions=128,
                                             quant_bits=8, quant_mode=A.QUANT_FP8))
    assert a8 > 0
    for lam in (-0.1, 1.0, 1.5):        # smoothed scores (R34): lambda in [0, 1)
        with pytest.raises(A.ArkvError):
            A.arkv_cache_bytes(A.make_config(1, 4, 2, 16, window=8, budget_tokens=32, smooth=lam))


def test_smoothing_storage():
    """R34 keeps one fp32 smoothed score per cached row (slot meta) and one per old row of a
    tailor wave (workspace) — only when smoothing is on."""
    kw = dict(window=32, budget_tokens=2048, max_positions=8192 + 64, max_prompt=8192)
    a0, w0 = A.arkv_cache_bytes(A.make_config(4, 32, 8, 128, **kw))
    a1, w1 = A.arkv_cache_bytes(A.make_config(4, 32, 8, 128, smooth=0.5, **kw))
    assert a1 > a0 and w1 > w0
    slots = 4 * 8 + 8                   # units + default spares (batch x H_kv)
    cap_o = (2048 + 1 + 31) // 32 * 32
    assert a1 - a0 >= slots * cap_o * 4  # at least 4 B per Original row slot
    assert a1 - a0 < 0.05 * a0           # a few percent of the arena


def test_arena_respects_budget():
    """The persistent arena is ~B_bytes per unit (+ tile slack and metadata), i.e. the
    4x reduction of configs[1] is physical: arena < dense bf16 / 3."""
    c = A.make_config(32, 32, 8, 128, budget_tokens=8192, max_positions=32768 + 4096, max_prompt=32768)
    arena, _ = A.arkv_cache_bytes(c)
    dense = 32 * 8 * (32768 + 4096) * 512
    assert arena < dense / 3


def _ocfg(c: A.ArkvConfig) -> O.Cfg:
    return O.Cfg(n_layers=c.n_layers, n_q_heads=c.n_q_heads, n_kv_heads=c.n_kv_heads, head_dim=c.head_dim,
                 window=c.window, budget_tokens=c.budget_tokens, quant_bits=c.quant_bits,
                 group_size=c.group_size or c.head_dim, alpha=c.alpha)


def test_schedule_appendix_config2():
    c = A.make_config(32, 32, 8, 128, budget_tokens=8192, max_positions=40000, max_prompt=32768)
    for rho in (1.0, 0.5, 0.3):
        assert A.arkv_schedule(c, 32768, rho, 4096) == O.schedule(32768, 4096, rho, _ocfg(c))


@settings(max_examples=200, deadline=None)
@given(st.integers(4, 3000), st.integers(0, 1500), st.floats(0.01, 1.0), st.integers(1, 48),
       st.sampled_from([(16, 4, 16), (128, 4, 128), (128, 4, 32), (64, 2, 64), (128, 8, 64), (32, 8, 8)]))
def test_host_schedule_equals_oracle(P, steps, rho, W, dbg):
    d, bits, g = dbg
    B = 2 * W + 1 + (P // 3)
    c = A.make_config(1, 1, 1, d, window=W, budget_tokens=B, quant_bits=bits, group_size=g,
                      max_positions=P + steps + 1, max_prompt=P)
    assert A.arkv_schedule(c, P, rho, steps) == O.schedule(P, steps, rho, _ocfg(c))


@pytest.mark.parametrize("p", [[0.25] * 4, [1, 0, 0, 0], [0.5, 0.25, 0.125, 0.125], [0.1, 0.2, 0.3, 0.4]])
def test_host_oq_score_equals_oracle(p):
    p = np.array(p, dtype=float)
    n = len(p)
    nz = p > 0
    H = float(-(p[nz] * np.log(p[nz])).sum())
    m2 = float(((p - 1 / n) ** 2).sum() / n)
    m4 = float(((p - 1 / n) ** 4).sum() / n)
    c = A.make_config(1, 1, 1, 16, window=1, budget_tokens=8)
    stats, score = A.arkv_oq_score(c, H, m2, m4)
    ref = O.compute_stats(p)
    np.testing.assert_allclose(stats, ref, rtol=1e-12)
    assert score == pytest.approx(O.oq_score(*ref), rel=1e-12)


@pytest.mark.parametrize("d,bits,g,layout", [
    (16, 4, 16, 1), (16, 2, 16, 1), (16, 8, 8, 1), (32, 4, 32, 2), (64, 4, 32, 2), (128, 4, 128, 2),
    (128, 4, 64, 2), (128, 4, 32, 2), (128, 2, 32, 1), (128, 8, 128, 1), (64, 4, 16, 1), (32, 2, 8, 1),
    (128, 8, 128, 2), (128, 8, 16, 2), (64, 8, 32, 2), (32, 8, 32, 2)])
def test_tile_layouts_are_bijections(d, bits, g, layout):
    """PLAIN and FRAG tile layouts: element -> byte maps are bijections covering the tile,
    and the code-slot inverse used by the tailor's packing pass inverts them."""
    mode = A.QUANT_FP8 if (bits == 8 and layout == 2) else A.QUANT_ASYM   # 8-bit FRAG = fp8 codes
    c = A.make_config(1, 4, 2, d, window=8, budget_tokens=64, quant_bits=bits, group_size=g, layout=layout,
                      max_positions=256, quant_mode=mode)
    n = A.arkv_layout_check(c)
    assert n == 32 * d * 2 + 32 * d * 2 + 32 * 4 * (d // g)


@pytest.mark.parametrize("d", [48, 80, 96, 160, 192, 256])
def test_unsupported_head_dims_rejected(d):
    """Only head dims every kernel path covers (prefill passes, both decode kernels, both
    move kernels) are accepted: others fail at configuration, never mid-tailor."""
    c = A.make_config(1, 4, 2, d, window=8, budget_tokens=64, group_size=16, max_positions=256)
    with pytest.raises(A.ArkvError) as e:
        A.arkv_cache_bytes(c)
    assert e.value.code == -2


@settings(max_examples=300, deadline=None)
@given(n_layers=st.integers(1, 6), batch=st.integers(1, 3), hkv=st.sampled_from([1, 2, 8]),
       max_ctas=st.sampled_from([1, 3, 40, 296, 320]), data=st.data())
def test_persist_plan_replay(n_layers, batch, hkv, max_ctas, data):
    """The persistent decode kernel's plan (host C++), replayed on the host: every item
    streamed once, partial slots disjoint, each unit's combine merges exactly its own
    partials — for arbitrary per-unit O/Q counts, including empty units and more CTAs
    than items."""
    B = 2048
    c = A.make_config(n_layers, 4 * hkv, hkv, 128, batch=batch, window=32, budget_tokens=B,
                      max_positions=4 * B, layout=2)
    U = batch * n_layers * hkv
    counts = st.tuples(st.integers(0, B + 1), st.integers(0, 3 * B))
    pairs = data.draw(st.lists(counts, min_size=U, max_size=U))
    n_o = [p[0] for p in pairs]
    n_q = [p[1] for p in pairs]
    if sum(n_o) + sum(n_q) == 0:
        n_o[0] = 1
    used = A.arkv_persist_plan_check(c, n_o, n_q, max_ctas)
    assert 1 <= used <= max_ctas


def test_persist_plan_configs1_keeps_full_grid():
    """configs[1]-like counts (per-layer rho): the plan keeps 2 CTAs per SM."""
    c = A.make_config(32, 32, 8, 128, window=32, budget_tokens=8192, max_positions=40000, layout=2)
    rng = np.random.default_rng(0)
    n_o, n_q = [], []
    for _ in range(32):
        rho = rng.uniform(0.05, 0.95)
        o = int(rho * 8160) + 32
        q = int((8192 - o) * 512 / 144)
        n_o += [o] * 8
        n_q += [q] * 8
    assert A.arkv_persist_plan_check(c, n_o, n_q, 296) == 296


@settings(max_examples=300, deadline=None)
@given(n_layers=st.integers(1, 8), batch=st.integers(1, 3), hkv=st.sampled_from([1, 2, 8]),
       num_sms=st.sampled_from([1, 8, 148]), data=st.data())
def test_split_order_replay(n_layers, batch, hkv, num_sms, data):
    """The split-K kernel's cost-balanced launch order (host C++), replayed on the host:
    every unit once, split counts within bounds and equal across a pair's KV heads, the
    kernel's split ranges tile each unit exactly, LPT order, at most 2 CTAs per slot."""
    B = 2048
    c = A.make_config(n_layers, 4 * hkv, hkv, 128, batch=batch, window=32, budget_tokens=B,
                      max_positions=4 * B, layout=2)
    n_pairs = batch * n_layers
    counts = st.tuples(st.integers(0, B - 1), st.integers(0, 3 * B))
    pairs = data.draw(st.lists(counts, min_size=n_pairs, max_size=n_pairs))
    n_ctas = A.arkv_split_order_check(c, [p[0] for p in pairs], [p[1] for p in pairs], num_sms)
    assert n_pairs * hkv <= n_ctas <= (max(n_pairs, 4 * num_sms // hkv) + n_pairs) * hkv


def test_split_order_configs1_exact_waves():
    """configs[1]-like counts (per-layer rho): exactly 2 CTAs per slot (2 x 296)."""
    c = A.make_config(32, 32, 8, 128, window=32, budget_tokens=8192, max_positions=40000, layout=2)
    rng = np.random.default_rng(0)
    n_o, n_q = [], []
    for _ in range(32):
        rho = rng.uniform(0.05, 0.95)
        o = int(rho * 8160) + 32
        n_o.append(o)
        n_q.append(int((8192 - o) * 512 / 144))
    assert A.arkv_split_order_check(c, n_o, n_q, 148) == 592


def test_bench_traffic_record_window():
    """bench.py's roofline traffic comes from the ncu capture of the same kind of step as
    the timed window: the HH-window capture for the driver's --steps 20 --warmup 5 at
    configs[1] (all steps before the first decode tailor), the steady capture otherwise."""
    import argparse
    import bench
    key = "auto (split-K chunked pipeline with cost-balanced LPT splits; persistent at >= 32 units per SM)"
    a = argparse.Namespace(mode="arkv", workload="llama3-8b-32k")
    hh = bench.traffic_record(a, key, "hh_window")
    st = bench.traffic_record(a, key, "steady")
    assert hh and st and hh["dram_bytes_per_launch"] > st["dram_bytes_per_launch"]
    assert "launch 8" in hh["source"] and "launch 150" in st["source"]
    assert bench.traffic_record(argparse.Namespace(mode="quant", workload="llama3-8b-32k"), key, "steady") is None
