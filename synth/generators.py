"""Seeded synthetic q/k/v generators (DESIGN.md §4 "input recipe").

Shapes follow the paper's LLaMA3-8B / Qwen3-8B workloads (32 q heads,
8 KV heads, head_dim 128) at the BASELINE.json configs.  Everything is drawn in
float32 and rounded to bfloat16 by torch (round-to-nearest-even).  Two recipes:

* "natural": keys k_j = N(0, I) + a_j u_{l,h} with attention sinks (j < 4),
  ~5 % log-normal heavy hitters and a recency bump over the last 256 prompt
  positions; queries q = beta_l u + N(0, I) with beta_l spread over layers so that
  entropy (and therefore rho) differs by layer; values N(0, 1) with two outlier
  channels x8 to stress quantization.
* "margin": keys k_j = level_j * u (+ tiny noise) with levels from a shuffled
  arithmetic progression, so heavy-hitter scores are well separated and the
  oracle's float64 ranking equals the GPU's float32 ranking; a few keys are exact
  bitwise duplicates of their predecessor to exercise the position tie-break.

Random numbers only — no step of the method is computed here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Tuple

import torch


@dataclasses.dataclass(frozen=True)
class Shape:
    batch: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    prompt_len: int
    window: int


def _gen(seed: int, *salt: int, device="cpu") -> torch.Generator:
    h = seed & 0xFFFFFFFF
    for s in salt:
        h = (h * 1000003 + (int(s) & 0xFFFFFFFF) + 0x9E3779B9) & 0xFFFFFFFFFFFF
    g = torch.Generator(device=device)
    g.manual_seed(h)
    return g


def _directions(sh: Shape, seed: int, device) -> torch.Tensor:
    """u_{l,h}: one random direction per (layer, KV head), norm sqrt(d)."""
    g = _gen(seed, 7)
    u = torch.randn(sh.n_layers, sh.n_kv_heads, sh.head_dim, generator=g)
    u = u / u.norm(dim=-1, keepdim=True) * math.sqrt(sh.head_dim)
    return u.to(device)


def _betas(sh: Shape) -> torch.Tensor:
    L = sh.n_layers
    return torch.tensor([0.15 + 0.85 * (l / max(L - 1, 1)) for l in range(L)])


def _key_levels(n: int, start: int, total: int, g: torch.Generator, heavy_frac=0.05) -> torch.Tensor:
    """Natural recipe: per-position amplitude a_j along u."""
    pos = torch.arange(start, start + n)
    a = torch.zeros(n)
    hh = torch.rand(n, generator=g) < heavy_frac
    a = torch.where(hh, 0.35 * torch.exp(0.5 * torch.randn(n, generator=g)), a)
    a = torch.where(pos < 4, torch.full_like(a, 0.8), a)                   # attention sinks
    a = torch.where(pos >= total - 256, a + 0.12, a)                       # recency bump
    return a


def prefill_inputs(sh: Shape, seed: int = 0, recipe: str = "natural", device="cpu"
                   ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """q_win [B][L][H_q][W][d], k, v [B][L][H_kv][P][d] as bfloat16 tensors."""
    B, L, Hq, Hkv, d, P, W = (sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads,
                              sh.head_dim, sh.prompt_len, sh.window)
    G = Hq // Hkv
    u = _directions(sh, seed, "cpu")
    beta = _betas(sh)
    qw = torch.empty(B, L, Hq, W, d, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    for b in range(B):
        for l in range(L):
            for h in range(Hkv):
                g = _gen(seed, 1, b, l, h)
                uh = u[l, h]
                if recipe == "margin":
                    lev = _margin_levels(P, g)
                    kk = lev[:, None] * uh[None, :] / math.sqrt(d) * 1.0 + 0.02 * torch.randn(P, d, generator=g)
                    dup = torch.rand(P, generator=g) < 0.03
                    idx = torch.arange(P)
                    src = torch.where(dup & (idx > 0), idx - 1, idx)
                    kk = kk[src]
                else:
                    a = _key_levels(P, 0, P, g)
                    kk = torch.randn(P, d, generator=g) + a[:, None] * uh[None, :]
                vv = torch.randn(P, d, generator=g)
                vv[:, :2] *= 8.0
                k[b, l, h] = kk.to(torch.bfloat16).to(device)
                v[b, l, h] = vv.to(torch.bfloat16).to(device)
                for j in range(G):
                    gq = _gen(seed, 2, b, l, h * G + j)
                    qq = beta[l] * uh[None, :] + torch.randn(W, d, generator=gq)
                    if recipe == "margin":
                        qq = (0.6 + 0.4 * torch.rand(W, 1, generator=gq)) * uh[None, :] * 4.0 + 0.02 * torch.randn(W, d, generator=gq)
                    qw[b, l, h * G + j] = qq.to(torch.bfloat16).to(device)
    return qw, k, v


def _margin_levels(n: int, g: torch.Generator) -> torch.Tensor:
    """Shuffled arithmetic progression of key levels (distinct, well separated)."""
    lev = torch.linspace(0.0, 1.0, n)
    perm = torch.randperm(n, generator=g)
    return lev[perm]


def decode_inputs(sh: Shape, step: int, seed: int = 0, recipe: str = "natural", device="cpu"
                  ) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """q [B][L][H_q][d], k, v [B][L][H_kv][d] (bf16) for decode step `step`
    (position prompt_len + step)."""
    B, L, Hq, Hkv, d = sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim
    G = Hq // Hkv
    u = _directions(sh, seed, "cpu")
    beta = _betas(sh)
    q = torch.empty(B, L, Hq, d)
    k = torch.empty(B, L, Hkv, d)
    v = torch.empty(B, L, Hkv, d)
    for b in range(B):
        g = _gen(seed, 3, b, step)
        for l in range(L):
            for h in range(Hkv):
                uh = u[l, h]
                if recipe == "margin":
                    lev = torch.rand(1, generator=g)
                    k[b, l, h] = lev * uh / math.sqrt(d) + 0.02 * torch.randn(d, generator=g)
                    for j in range(G):
                        q[b, l, h * G + j] = (0.6 + 0.4 * torch.rand(1, generator=g)) * uh * 4.0 + 0.02 * torch.randn(d, generator=g)
                else:
                    a = 0.35 * torch.exp(0.5 * torch.randn(1, generator=g)) if torch.rand(1, generator=g).item() < 0.05 else torch.zeros(1)
                    k[b, l, h] = torch.randn(d, generator=g) + a * uh
                    for j in range(G):
                        q[b, l, h * G + j] = beta[l] * uh + torch.randn(d, generator=g)
                vv = torch.randn(d, generator=g)
                vv[:2] *= 8.0
                v[b, l, h] = vv
    return (q.to(torch.bfloat16).to(device), k.to(torch.bfloat16).to(device),
            v.to(torch.bfloat16).to(device))


def decode_inputs_fast(sh: Shape, step: int, seed: int = 0, device="cpu"):
    """Vectorised natural-recipe decode inputs for large shapes (bench): same
    distributions as decode_inputs(recipe="natural"), drawn in bulk."""
    B, L, Hq, Hkv, d = sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim
    G = Hq // Hkv
    u = _directions(sh, seed, device)
    beta = _betas(sh).to(device)
    g = _gen(seed, 4, step, device=device)
    a = torch.where(torch.rand(B, L, Hkv, 1, generator=g, device=device) < 0.05,
                    0.35 * torch.exp(0.5 * torch.randn(B, L, Hkv, 1, generator=g, device=device)),
                    torch.zeros(B, L, Hkv, 1, device=device))
    k = torch.randn(B, L, Hkv, d, generator=g, device=device) + a * u[None]
    q = beta[None, :, None, None] * u.repeat_interleave(G, dim=1)[None] + torch.randn(B, L, Hq, d, generator=g, device=device)
    v = torch.randn(B, L, Hkv, d, generator=g, device=device)
    v[..., :2] *= 8.0
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)


def prefill_inputs_fast(sh: Shape, seed: int = 0, device="cpu"):
    """Vectorised natural-recipe prefill inputs for large shapes (bench)."""
    B, L, Hq, Hkv, d, P, W = (sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads,
                              sh.head_dim, sh.prompt_len, sh.window)
    G = Hq // Hkv
    u = _directions(sh, seed, device)
    beta = _betas(sh).to(device)
    qw = torch.empty(B, L, Hq, W, d, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    pos = torch.arange(P, device=device)
    for b in range(B):
        for l in range(L):
            g = _gen(seed, 5, b, l, device=device)
            hh = torch.rand(Hkv, P, generator=g, device=device) < 0.05
            a = torch.where(hh, 0.35 * torch.exp(0.5 * torch.randn(Hkv, P, generator=g, device=device)),
                            torch.zeros(Hkv, P, device=device))
            a = torch.where(pos[None] < 4, torch.full_like(a, 0.8), a)
            a = torch.where(pos[None] >= P - 256, a + 0.12, a)
            kk = torch.randn(Hkv, P, d, generator=g, device=device) + a[..., None] * u[l][:, None, :]
            k[b, l] = kk.to(torch.bfloat16)
            vv = torch.randn(Hkv, P, d, generator=g, device=device)
            vv[..., :2] *= 8.0
            v[b, l] = vv.to(torch.bfloat16)
            qq = beta[l] * u[l].repeat_interleave(G, dim=0)[:, None, :] + torch.randn(Hq, W, d, generator=g, device=device)
            qw[b, l] = qq.to(torch.bfloat16)
    return qw, k, v


def prefill_inputs_margin_fast(sh: Shape, seed: int = 0, device="cpu"):
    """Vectorised margin recipe (see module docstring) for full-size parity runs:
    keys = level * u / sqrt(d) + 0.02 N with levels a shuffled arithmetic progression per
    (sequence, layer, KV head) and ~3 % of keys bitwise copies of their predecessor."""
    B, L, Hq, Hkv, d, P, W = (sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim,
                              sh.prompt_len, sh.window)
    G = Hq // Hkv
    u = _directions(sh, seed, device)
    qw = torch.empty(B, L, Hq, W, d, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    idx = torch.arange(P, device=device)
    lin = torch.linspace(0.0, 1.0, P, device=device)
    for b in range(B):
        for l in range(L):
            g = _gen(seed, 6, b, l, device=device)
            for h in range(Hkv):
                lev = lin[torch.randperm(P, generator=g, device=device)]
                kk = lev[:, None] * u[l, h][None, :] / math.sqrt(d) + 0.02 * torch.randn(P, d, generator=g, device=device)
                dup = torch.rand(P, generator=g, device=device) < 0.03
                src = torch.where(dup & (idx > 0), idx - 1, idx)
                k[b, l, h] = kk[src].to(torch.bfloat16)
            vv = torch.randn(Hkv, P, d, generator=g, device=device)
            vv[..., :2] *= 8.0
            v[b, l] = vv.to(torch.bfloat16)
            amp = 0.6 + 0.4 * torch.rand(Hq, W, 1, generator=g, device=device)
            qq = amp * u[l].repeat_interleave(G, dim=0)[:, None, :] * 4.0 + 0.02 * torch.randn(Hq, W, d, generator=g, device=device)
            qw[b, l] = qq.to(torch.bfloat16)
    return qw, k, v


def decode_inputs_margin_fast(sh: Shape, step: int, seed: int = 0, device="cpu"):
    """Vectorised margin-recipe decode inputs (new key at a random level along u)."""
    B, L, Hq, Hkv, d = sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim
    G = Hq // Hkv
    u = _directions(sh, seed, device)
    g = _gen(seed, 8, step, device=device)
    lev = torch.rand(B, L, Hkv, 1, generator=g, device=device)
    k = lev * u[None] / math.sqrt(d) + 0.02 * torch.randn(B, L, Hkv, d, generator=g, device=device)
    amp = 0.6 + 0.4 * torch.rand(B, L, Hq, 1, generator=g, device=device)
    q = amp * u.repeat_interleave(G, dim=1)[None] * 4.0 + 0.02 * torch.randn(B, L, Hq, d, generator=g, device=device)
    v = torch.randn(B, L, Hkv, d, generator=g, device=device)
    v[..., :2] *= 8.0
    return q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)


# ---------------------------------------------------------------------------------------
# "lattice" recipe: a score margin at ANY prompt length (full-size parity, n_e up to 131K).
#
# Every key carries an integer level L_j in binary in dims 0..17 (bits 0/1, bf16-exact);
# the other dims are random bits, with a fixed 0 and 1 in every 32-dim block (dims 18, 19
# in the first) so every quantization group has min 0 and max 1.  Every query of layer l is
# q[m] = 2^(m - e_l) for m < 18, else 0 (the same for all heads, window rows and steps).
# So q.k_j = 2^-e_l * L_j EXACTLY in fp32 and fp64 (integer sums of powers of two), and
# it stays a common multiple (1 + eps, |eps| < 1e-7) of L_j after the exact-code group
# quantization of {0, 1} values (int2/4/8 asymmetric: codes 0 / 2^b - 1; fp8: 0 / 448).
# Attention weights are then exp(c L_j) / Z with c = 2^-e_l / sqrt(d): adjacent levels
# give heavy-hitter scores a relative gap >= c (>= 2e-5 here), far above fp32 rounding,
# while bitwise-equal keys (3 % duplicated prompt keys, repeated decode levels) tie
# EXACTLY in both implementations and exercise the position tie-break.  Prompt levels
# are 2 * (a permutation of 0..P-1); decode keys take odd levels 2 * randint(P) + 1.
# e_l = e0 + (l mod 4) with e0 = ceil(log2(2 P / (80 sqrt(d)))): the level range spans
# <= 80 nats, and rho differs by layer.  Values: N(0, 1) with two x8 outlier channels.
# ---------------------------------------------------------------------------------------
LATTICE_BITS = 18


def lattice_exponent(sh: Shape, layer: int) -> int:
    e0 = max(0, math.ceil(math.log2(2 * sh.prompt_len / (80.0 * math.sqrt(sh.head_dim)))))
    return e0 + (layer % 4)


def _lattice_keys(lev: torch.Tensor, d: int, g: torch.Generator, device) -> torch.Tensor:
    n = lev.shape[0]
    k = torch.randint(0, 2, (n, d), generator=g, device=device, dtype=torch.int64)
    bits = torch.arange(LATTICE_BITS, device=device)
    k[:, :LATTICE_BITS] = (lev[:, None] >> bits[None, :]) & 1
    k[:, LATTICE_BITS] = 0
    k[:, LATTICE_BITS + 1] = 1
    for blk in range(32, d, 32):
        k[:, blk] = 0
        k[:, blk + 1] = 1
    return k.to(torch.bfloat16)


def _lattice_query(sh: Shape, layer: int, device) -> torch.Tensor:
    e = lattice_exponent(sh, layer)
    q = torch.zeros(sh.head_dim, device=device)
    q[:LATTICE_BITS] = torch.pow(2.0, torch.arange(LATTICE_BITS, device=device, dtype=torch.float32) - e)
    return q.to(torch.bfloat16)


def prefill_inputs_lattice(sh: Shape, seed: int = 0, device="cpu"):
    """Lattice recipe (above): q_win [B][L][H_q][W][d], k, v [B][L][H_kv][P][d] bf16."""
    B, L, Hq, Hkv, d, P, W = (sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim,
                              sh.prompt_len, sh.window)
    assert d >= 64 and d % 32 == 0 and 2 * P <= (1 << LATTICE_BITS)
    qw = torch.empty(B, L, Hq, W, d, dtype=torch.bfloat16, device=device)
    k = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    v = torch.empty(B, L, Hkv, P, d, dtype=torch.bfloat16, device=device)
    idx = torch.arange(P, device=device)
    for b in range(B):
        for l in range(L):
            g = _gen(seed, 9, b, l, device=device)
            for h in range(Hkv):
                lev = 2 * torch.randperm(P, generator=g, device=device)
                dup = torch.rand(P, generator=g, device=device) < 0.03
                lev = lev[torch.where(dup & (idx > 0), idx - 1, idx)]
                kk = _lattice_keys(lev, d, g, device)
                kk[1:][dup[1:]] = kk[:-1][dup[1:]]        # duplicated keys: bitwise copies
                k[b, l, h] = kk
            vv = torch.randn(Hkv, P, d, generator=g, device=device)
            vv[..., :2] *= 8.0
            v[b, l] = vv.to(torch.bfloat16)
            qw[b, l] = _lattice_query(sh, l, device)[None, None, :].expand(Hq, W, d)
    return qw, k, v


def decode_inputs_lattice(sh: Shape, step: int, seed: int = 0, device="cpu"):
    """Lattice recipe decode inputs: q as in the prefill window; new key at an odd level."""
    B, L, Hq, Hkv, d, P = sh.batch, sh.n_layers, sh.n_q_heads, sh.n_kv_heads, sh.head_dim, sh.prompt_len
    g = _gen(seed, 10, step, device=device)
    lev = 2 * torch.randint(0, P, (B * L * Hkv,), generator=g, device=device) + 1
    k = _lattice_keys(lev, d, g, device).view(B, L, Hkv, d)
    q = torch.stack([_lattice_query(sh, l, device) for l in range(L)])       # [L][d]
    q = q[None, :, None, :].expand(B, L, Hq, d).contiguous()
    v = torch.randn(B, L, Hkv, d, generator=g, device=device)
    v[..., :2] *= 8.0
    return q, k, v.to(torch.bfloat16)
