"""ARKV oracle: plain CPU reference of the decode hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  It shares no code with paper_2603_08727_b200/ and
imports nothing from it.

Citations: "P:n" = /root/reference/PAPER.md line n (section / equation given);
"S:n" = SPEC.md line n; "R<k>" = reading k in DESIGN.md §3 (where the paper is
silent, ambiguous or garbled).  Arithmetic is float64 except where the method's
integer decisions must be bit-exact with the GPU (quantization codes, fp32 scales,
promotion to bf16), which is emulated with numpy float32 scalars op by op.

Parity pins (tests/test_oracle_*.py) tie every function below to something other
than itself: printed SPEC examples, closed forms, brute force, textbook special
cases.  Functions whose behaviour the paper does not fix at all are marked
"parity unpinned" here and in DESIGN.md §3.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Tuple

import numpy as np

# ----------------------------------------------------------------------------
# Configuration (P:368 hyper-parameters; R10/R11 budget unit; R23 quant format)
# ----------------------------------------------------------------------------


@dataclasses.dataclass
class Cfg:
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    batch: int = 1
    window: int = 32                 # W, "window size is set to 32"
    budget_tokens: int = 512         # B in bf16-token equivalents per (seq, layer, kv head) (R10, R11)
    quant_bits: int = 4              # R23
    group_size: int = 0              # 0 -> head_dim ("per-token scale")
    state_sharing: str = "head"      # "head": one state set per KV head (R20) | "layer": SPEC's
                                     # S:231 score averaged across the layer's groups (NEXT-3)
    quant_mode: str = "asym"         # "asym" (scale, zero=min) | "sym" |
                                     # "fp8" (e4m3 codes, per-group scale: P:333; NEXT-2)
    alpha: float = 0.75
    tau: Tuple[float, float, float] = (7.774, 5.407, 5.528)
    gamma: float = 263.81
    stat_eps: float = 1e-30          # R6
    sm_scale: float = 0.0            # 0 -> 1/sqrt(head_dim) (R27)
    smooth: float = 0.0              # λ of the "smoothed" scores (Alg. 1; R34, NEXT-4); 0 = off (R21)

    def __post_init__(self):
        if self.group_size == 0:
            self.group_size = self.head_dim
        if self.sm_scale == 0.0:
            self.sm_scale = 1.0 / math.sqrt(self.head_dim)

    @property
    def G(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def n_groups(self) -> int:
        return self.head_dim // self.group_size


def validate(cfg: Cfg) -> None:
    """Configuration errors (SPEC S:184 'B <= W', R14 'B > 2W', R23 formats)."""
    if cfg.n_q_heads % cfg.n_kv_heads:
        raise ValueError("n_q_heads % n_kv_heads != 0")
    if cfg.quant_bits not in (2, 4, 8):
        raise ValueError("quant_bits must be 2, 4 or 8")
    if cfg.head_dim % cfg.group_size:
        raise ValueError("group_size must divide head_dim")
    if (cfg.head_dim * cfg.quant_bits) % 8:
        raise ValueError("head_dim*bits must be a whole number of bytes")
    if cfg.budget_tokens <= 2 * cfg.window:
        raise ValueError("budget must exceed 2W (R14)")
    if cfg.state_sharing not in ("head", "layer"):
        raise ValueError("state_sharing")
    if cfg.quant_mode not in ("asym", "sym", "fp8"):
        raise ValueError("quant_mode")
    if cfg.quant_mode == "fp8" and cfg.quant_bits != 8:
        raise ValueError("fp8 codes are 8 bits")
    if not 0.0 <= cfg.smooth < 1.0:
        raise ValueError("smooth must lie in [0, 1)")


# ----------------------------------------------------------------------------
# Byte costs and Eq. 1 accounting (§IV-B Eq. 1; R10)
# ----------------------------------------------------------------------------

def cost_orig(cfg: Cfg) -> int:
    """C_orig in bytes per (token, KV head): K and V in bf16."""
    return 4 * cfg.head_dim


def cost_quant(cfg: Cfg) -> int:
    """C_quant in bytes per (token, KV head): K and V codes plus an fp32 scale and an
    fp32 zero per group for each of K and V (R10, R23)."""
    d, b, g = cfg.head_dim, cfg.quant_bits, cfg.group_size
    return 2 * (d * b // 8 + 8 * (d // g))


def budget_bytes(cfg: Cfg) -> int:
    """B in bytes (Eq. 1 'B (in bytes)') from the token budget."""
    return cfg.budget_tokens * cost_orig(cfg)


def usage_bytes(cfg: Cfg, n_o: int, n_q: int) -> int:
    """Eq. 1 left-hand side for one (seq, layer, KV head) unit: n_o*C_orig + n_q*C_quant."""
    return n_o * cost_orig(cfg) + n_q * cost_quant(cfg)


# ----------------------------------------------------------------------------
# Prefill statistics (§IV-C Eqs. 2-5) and OQ ratio (Eqs. 6-8)
# ----------------------------------------------------------------------------

def windowed_attention(q_win: np.ndarray, k: np.ndarray, cfg: Cfg) -> np.ndarray:
    """Eq. 2 with reading R1: post-softmax attention A of the last W
    queries (positions P-W..P-1) over all causally visible keys, then sliced to keys
    [0, P-W).  q_win: [H_q][W][d], k: [H_kv][P][d] (post-RoPE values).  Returns
    Ã[H_q][W][P-W] in float64.  Query head h reads KV head h // G (R27)."""
    Hq, W, d = q_win.shape
    P = k.shape[1]
    G = Hq // k.shape[0]
    out = np.empty((Hq, W, P - W), dtype=np.float64)
    qpos = P - W + np.arange(W)
    kpos = np.arange(P)
    mask = kpos[None, :] > qpos[:, None]           # causal: key j visible iff j <= query position
    for h in range(Hq):
        s = (q_win[h].astype(np.float64) @ k[h // G].astype(np.float64).T) * cfg.sm_scale
        s = np.where(mask, -np.inf, s)
        s = s - s.max(axis=1, keepdims=True)
        e = np.exp(s)
        a = e / e.sum(axis=1, keepdims=True)       # rows sum to 1 over visible keys
        out[h] = a[:, : P - W]                      # slice AFTER normalisation (R1)
    return out


def key_mass(a_tilde: np.ndarray) -> np.ndarray:
    """Eq. 3 p_k: p_k = (1/Z) Σ_{h,q} Ã[h,q,k], Z the grand total (R3)."""
    col = a_tilde.sum(axis=tuple(range(a_tilde.ndim - 1)))
    Z = col.sum()
    if not Z > 0:
        raise ValueError("degenerate distribution (Z = 0)")
    return col / Z


def compute_stats(p: np.ndarray, stat_eps: float = 1e-30) -> Tuple[float, float, float]:
    """Eq. 3 entropy (natural log, R2; 0 ln 0 = 0), Eq. 4 variance with p̄ = 1/n (R4,
    population divisor), Eq. 5 Pearson kurtosis m4/m2² (R5).  Degenerate cases (R6):
    each statistic is clamped below at stat_eps, and 𝓚 := 1 when m2 <= stat_eps.
    Parity unpinned: the value of stat_eps (the paper is silent); the moments themselves
    are pinned to closed forms and SPEC's printed values."""
    p = np.asarray(p, dtype=np.float64)
    n = p.shape[0]
    nz = p > 0
    H = float(-(p[nz] * np.log(p[nz])).sum())
    dev = p - 1.0 / n
    m2 = float((dev ** 2).sum() / n)
    m4 = float((dev ** 4).sum() / n)
    K = m4 / (m2 * m2) if m2 > stat_eps else 1.0
    return max(H, stat_eps), max(m2, stat_eps), max(K, stat_eps)


def oq_score(H: float, V: float, K: float, tau=(7.774, 5.407, 5.528)) -> float:
    """Eq. 6: q = 𝓗^{1/τ1} 𝓥^{1/τ2} 𝓚^{1/τ3} (R7)."""
    return (H ** (1.0 / tau[0])) * (V ** (1.0 / tau[1])) * (K ** (1.0 / tau[2]))


def oq_ratios(q: np.ndarray) -> np.ndarray:
    """Eq. 7: ρ_ℓ = q_ℓ / max_k q_k, max over the L layers of one
    sequence (R8)."""
    q = np.asarray(q, dtype=np.float64)
    m = q.max()
    if not m > 0:
        raise ValueError("all OQ scores are zero")
    return q / m


def prefill_stats(q_win: np.ndarray, k: np.ndarray, cfg: Cfg):
    """Alg. 1 prefill phase for every (sequence, layer).
    q_win [B][L][H_q][W][d], k [B][L][H_kv][P][d].  Returns (stats [B][L][3],
    oq [B][L], rho [B][L], a_tilde dict[(b,l)] -> Ã)."""
    Bn, L = q_win.shape[0], q_win.shape[1]
    stats = np.zeros((Bn, L, 3))
    oq = np.zeros((Bn, L))
    at = {}
    for b in range(Bn):
        for l in range(L):
            a = windowed_attention(q_win[b, l], k[b, l], cfg)
            at[(b, l)] = a
            H, V, K = compute_stats(key_mass(a), cfg.stat_eps)
            stats[b, l] = (H, V, K)
            oq[b, l] = oq_score(H, V, K, cfg.tau)
    rho = np.stack([oq_ratios(oq[b]) for b in range(Bn)])
    return stats, oq, rho, at


# ----------------------------------------------------------------------------
# Budget split and tailor counts (Alg. 1 P:279 (R9); Eq. 10; R14, R15)
# ----------------------------------------------------------------------------

def origin_quota(rho: float, cfg: Cfg) -> int:
    """Alg. 1 (reading R9): eligible-token O quota ⌊ρ (B − W)⌋; the W window
    tokens are added on top (R17)."""
    return int(math.floor(rho * (cfg.budget_tokens - cfg.window)))


def tailor_counts(K: int, rho: float, cfg: Cfg) -> Tuple[int, int]:
    """Counts of one tailor on a unit holding K tokens (Eq. 10; R14, R15).
    Eligible n_e = K − W; keep b = ⌊α n_e⌋; of the kept, n_oe Original
    (Top-B_o, capped so that the post-tailor usage leaves W tokens of headroom,
    R14) and n_q Quantized (the rest of the keep set, capped by bytes).
    Parity unpinned: the headroom rule (R14) is this design's reading; the formula is
    pinned to a brute-force byte walk of the same rule.
    Returns (n_oe, n_q): eligible tokens kept Original, tokens kept Quantized."""
    W, B = cfg.window, cfg.budget_tokens
    Co, Cq, Bb = cost_orig(cfg), cost_quant(cfg), budget_bytes(cfg)
    n_e = K - W
    b = int(math.floor(cfg.alpha * n_e))
    n_oe = min(origin_quota(rho, cfg), b, B - 2 * W)
    n_q = min(b - n_oe, (Bb - (n_oe + 2 * W) * Co) // Cq)
    return n_oe, n_q


def prefill_needs_tailor(P: int, cfg: Cfg) -> bool:
    """R12/R14: the prompt is tailored at prefill end iff it leaves fewer than W
    tokens of headroom, i.e. P > B − W."""
    return P > cfg.budget_tokens - cfg.window


def decode_needs_tailor(n_o: int, n_q: int, cfg: Cfg) -> bool:
    """R12: after the append, tailor iff the unit has reached its budget, U >= B_bytes
    ("triggered when the KV cache reaches the limit"; "true iff usage
    >= budget.total", with its boundary case usage 512.0 of 512 -> true)."""
    return usage_bytes(cfg, n_o, n_q) >= budget_bytes(cfg)


def schedule(P: int, n_steps: int, rho: float, cfg: Cfg):
    """Data-independent count schedule of one unit (R15).  Returns a list of events
    (step, n_o, n_q, n_evicted) where step = -1 is the prefill tailor and step s >= 0
    is the s-th decode call (position P + s); n_o counts all Original tokens
    (window included) after the event."""
    ev = []
    W = cfg.window
    if prefill_needs_tailor(P, cfg):
        n_oe, n_q = tailor_counts(P, rho, cfg)
        ev.append((-1, n_oe + W, n_q, P - W - n_oe - n_q))
        n_o = n_oe + W
    else:
        n_o, n_q = P, 0
    for s in range(n_steps):
        n_o += 1
        if decode_needs_tailor(n_o, n_q, cfg):
            K = n_o + n_q
            n_oe, nq2 = tailor_counts(K, rho, cfg)
            ev.append((s, n_oe + W, nq2, K - W - n_oe - nq2))
            n_o, n_q = n_oe + W, nq2
    return ev


# ----------------------------------------------------------------------------
# Heavy-hitter score (§IV-E Eq. 9) and the tri-state plan (Eq. 10)
# ----------------------------------------------------------------------------

def hh_scores(samples: np.ndarray, gamma: float) -> np.ndarray:
    """Eq. 9 with reading R18: S_k = μ_k + γ Var_k, μ and the population variance
    taken over the N samples (rows) of the windowed attention that share the KV
    head (R20: h in the GQA group × window queries).  samples: [N][n_keys]."""
    s = np.asarray(samples, dtype=np.float64)
    mu = s.mean(axis=0)
    var = s.var(axis=0)             # population divisor N (R18)
    return mu + gamma * var


def smooth_scores(S: np.ndarray, positions: np.ndarray, prev: Dict[int, float], lam: float) -> np.ndarray:
    """Alg. 1 P:285 ranks tokens by "smoothed" heavy-hitter scores without defining the
    smoothing; reading R34 (NEXT-4; parity unpinned by the paper): an exponential moving
    average across tailors, S~_j = λ·S~_j(previous tailor) + (1 − λ)·S_j for a token that
    the previous tailor scored and kept, S~_j = S_j for a token it did not score (appended
    since, or inside its protected window).  λ = 0 is the unsmoothed Eq. 9 score."""
    S = np.asarray(S, dtype=np.float64)
    if lam == 0.0:
        return S
    out = S.copy()
    for i, p in enumerate(np.asarray(positions).tolist()):
        if p in prev:
            out[i] = lam * prev[p] + (1.0 - lam) * S[i]
    return out


def rank_order(scores: np.ndarray, positions: np.ndarray) -> np.ndarray:
    """Eq. 10 "Top-b" ordering with the tie-break of R22: score descending, then
    position ascending (older token first).  Returns indices best-first."""
    return np.lexsort((np.asarray(positions), -np.asarray(scores, dtype=np.float64)))


def plan_states(scores: np.ndarray, positions: np.ndarray, n_oe: int, n_q: int) -> np.ndarray:
    """Eq. 10 / Alg. 1 on the eligible tokens: ranks < n_oe ->
    Original (1), next n_q -> Quantized (2), the rest -> Evicted (3).  The keep set
    𝓘 = Top-b and 𝓘_o = Top-B_o(𝓘) nest because both rank by the same score (R16,
    R17).  Window tokens are not passed in: they are Original by construction."""
    order = rank_order(scores, positions)
    st = np.full(len(order), 3, dtype=np.int8)
    st[order[:n_oe]] = 1
    st[order[n_oe:n_oe + n_q]] = 2
    return st


# ----------------------------------------------------------------------------
# Quantization (Alg. 1 "x̃ = q̂ s", R23, R24) — fp32 emulated op by op
# ----------------------------------------------------------------------------

F32 = np.float32


def quantize(x: np.ndarray, bits: int, g: int, mode: str = "asym"):
    """Group quantization of one vector x[d] (exact bf16 values) with an fp32 scale
    and zero per group of g (R23).  fp32 operation order (R23 / SURVEY C1.6):
      asym: mn, mx = min, max; s = f32(f32(mx-mn) / f32(2^b-1)); z = mn;
            code = clamp(rint_even(f32(f32(x-mn)/s)), 0, 2^b-1); constant group: s=1, codes 0.
      sym:  a = max|x|; s = f32(a / f32(2^(b-1)-1)); z = 0;
            code = clamp(rint_even(f32(x/s)), ±(2^(b-1)-1)); zero group: s=1, codes 0.
      fp8:  a = max|x|; s = f32(a / 448); z = 0; code = e4m3_rne_satfinite(f32(x/s))
            (byte, NEXT-2); zero group: s=1, codes 0x00.
    Returns (codes int64[d], scale f32[d/g], zero f32[d/g])."""
    xf = np.asarray(x, dtype=np.float64).astype(F32)
    d = xf.shape[0]
    ng = d // g
    codes = np.zeros(d, dtype=np.int64)
    sc = np.zeros(ng, dtype=F32)
    zr = np.zeros(ng, dtype=F32)
    for gi in range(ng):
        xs = xf[gi * g:(gi + 1) * g]
        if mode == "asym":
            mn, mx = F32(xs.min()), F32(xs.max())
            if mx == mn:
                s, z, c = F32(1.0), mn, np.zeros(g, dtype=np.int64)
            else:
                s = F32(F32(mx - mn) / F32(2 ** bits - 1))
                z = mn
                # float32 array ops round each element exactly like the scalar ops
                c = np.rint((xs - mn).astype(F32) / s).astype(np.int64)
                c = np.clip(c, 0, 2 ** bits - 1)
        elif mode == "fp8":
            # per-group scale s = f32(a / 448) with a = max|x|; code = e4m3(f32(x / s))
            a = F32(np.abs(xs).max())
            if a == 0:
                s, z, c = F32(1.0), F32(0.0), np.zeros(g, dtype=np.int64)
            else:
                s = F32(a / F32(E4M3_MAX))
                z = F32(0.0)
                c = e4m3_encode((xs / s).astype(F32))
        else:
            a = F32(np.abs(xs).max())
            qmax = 2 ** (bits - 1) - 1
            if a == 0:
                s, z, c = F32(1.0), F32(0.0), np.zeros(g, dtype=np.int64)
            else:
                s = F32(a / F32(qmax))
                z = F32(0.0)
                c = np.rint((xs / s).astype(F32)).astype(np.int64)
                c = np.clip(c, -qmax, qmax)
        codes[gi * g:(gi + 1) * g] = c
        sc[gi] = s
        zr[gi] = z
    return codes, sc, zr


# ---- OCP FP8 E4M3 ("FP8"): 1 sign, 4 exponent bits (bias 7), 3 mantissa
# bits; no infinities; S.1111.111 is NaN, so the largest finite magnitude is 448 ----
def _e4m3_magnitudes() -> np.ndarray:
    v = np.empty(127)
    for c in range(127):
        e, m = c >> 3, c & 7
        v[c] = (m / 8.0) * 2.0 ** -6 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return v


E4M3 = _e4m3_magnitudes()       # magnitude of codes 0x00..0x7E, strictly increasing
E4M3_MAX = 448.0


def e4m3_encode(x) -> np.ndarray:
    """float32 values -> e4m3 code bytes: round to nearest, ties to the even code,
    magnitudes above 448 saturate to 448 ("satfinite"); the sign bit is kept (-0 -> 0x80)."""
    xf = np.asarray(x, dtype=F32).astype(np.float64)
    a = np.minimum(np.abs(xf), E4M3_MAX)
    hi = np.searchsorted(E4M3, a, side="left")          # first magnitude >= a
    hi = np.minimum(hi, 126)
    lo = np.maximum(hi - 1, 0)
    dlo, dhi = a - E4M3[lo], E4M3[hi] - a
    pick_lo = (dlo < dhi) | ((dlo == dhi) & (lo % 2 == 0))
    c = np.where(E4M3[hi] == a, hi, np.where(pick_lo, lo, hi)).astype(np.int64)
    return c | (np.signbit(xf).astype(np.int64) << 7)


def e4m3_decode(codes) -> np.ndarray:
    c = np.asarray(codes, dtype=np.int64)
    return np.where(c & 0x80, -1.0, 1.0) * E4M3[c & 0x7F]


def code_values(codes: np.ndarray, mode: str) -> np.ndarray:
    """The number a stored code stands for: the integer itself, or the e4m3 value."""
    return e4m3_decode(codes) if mode == "fp8" else np.asarray(codes, dtype=np.float64)


def dequantize(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray, g: int, mode: str = "asym") -> np.ndarray:
    """Alg. 1: x̃ = q̂·s (+ z for the asymmetric zero point), evaluated
    in float64 from the fp32 scale and zero — the values attention sees (R23)."""
    s = np.repeat(np.asarray(scale, dtype=np.float64), g)
    z = np.repeat(np.asarray(zero, dtype=np.float64), g)
    return code_values(codes, mode) * s + z


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even), returned as float64."""
    u = np.asarray(x, dtype=F32).reshape(-1).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(F32).astype(np.float64).reshape(np.shape(x))


def promote(codes: np.ndarray, scale: np.ndarray, zero: np.ndarray, g: int, mode: str = "asym") -> np.ndarray:
    """Q -> O re-materialisation (R24): bf16_rne(f32(f32(code·s) + z)), per element
    (code = its e4m3 value in fp8 mode)."""
    d = len(codes)
    cv = code_values(codes, mode)
    out = np.empty(d, dtype=F32)
    for i in range(d):
        gi = i // g
        out[i] = F32(F32(F32(cv[i]) * scale[gi]) + zero[gi])
    return f32_to_bf16_rne(out)


# ----------------------------------------------------------------------------
# Decode attention over O ∪ Q (R26, R27)
# ----------------------------------------------------------------------------

def attention(q: np.ndarray, keys: np.ndarray, vals: np.ndarray, sm_scale: float):
    """Softmax attention of G query heads over n cached (possibly dequantized) keys:
    o_h = Σ_j softmax_j(sm q_h·k_j) v_j.  Order-free (R26).  Returns (out [G][d],
    probs [G][n])."""
    s = (np.asarray(q, dtype=np.float64) @ np.asarray(keys, dtype=np.float64).T) * sm_scale
    s = s - s.max(axis=1, keepdims=True)
    e = np.exp(s)
    p = e / e.sum(axis=1, keepdims=True)
    return p @ np.asarray(vals, dtype=np.float64), p


# ----------------------------------------------------------------------------
# The unit cache and the multi-step driver (Alg. 1)
# ----------------------------------------------------------------------------

class UnitCache:
    """Tri-state cache of one (sequence, layer, KV head) unit (DS1).
    O tokens hold exact bf16 values (as float64); Q tokens hold integer codes and
    fp32 scale/zero per group; evicted tokens are dropped."""

    def __init__(self, cfg: Cfg):
        self.cfg = cfg
        d = cfg.head_dim
        self.o_pos = np.zeros(0, dtype=np.int64)
        self.o_k = np.zeros((0, d))
        self.o_v = np.zeros((0, d))
        self.q_pos = np.zeros(0, dtype=np.int64)
        self.q_kc = np.zeros((0, d), dtype=np.int64)
        self.q_vc = np.zeros((0, d), dtype=np.int64)
        ng = cfg.n_groups
        self.q_ks = np.zeros((0, ng), dtype=F32)
        self.q_kz = np.zeros((0, ng), dtype=F32)
        self.q_vs = np.zeros((0, ng), dtype=F32)
        self.q_vz = np.zeros((0, ng), dtype=F32)
        self.evicted: List[int] = []
        self.n_pos = 0                     # positions seen so far
        self.history: List[Tuple[int, np.ndarray, np.ndarray]] = []   # (query pos, key positions, probs [G][n])
        self.last_tailor_pos = -1          # position of the query at/after which the last tailor took effect
        self.q0 = 0                        # first query position on the current cache (R19): the
                                           # first decode call after the prompt, or the last tailor's step
        self.tailors: List[Tuple[int, int, int, int]] = []
        self.margins: List[float] = []     # relative score gaps at the rank thresholds
        self.prev_score: Dict[int, float] = {}   # R34: smoothed score of each kept token at the last tailor

    @property
    def n_o(self):
        return len(self.o_pos)

    @property
    def n_q(self):
        return len(self.q_pos)

    def usage(self):
        return usage_bytes(self.cfg, self.n_o, self.n_q)

    def append(self, pos: int, k: np.ndarray, v: np.ndarray):
        """D1: the new token enters as Original."""
        if pos != self.n_pos:
            raise ValueError("sequencing error (S:57)")
        self.o_pos = np.append(self.o_pos, pos)
        self.o_k = np.vstack([self.o_k, np.asarray(k, dtype=np.float64)[None]])
        self.o_v = np.vstack([self.o_v, np.asarray(v, dtype=np.float64)[None]])
        self.n_pos = pos + 1

    def ingest(self, k: np.ndarray, v: np.ndarray):
        """The prompt's P tokens enter as Original at positions 0..P-1 (equivalent to
        P appends on an empty unit)."""
        if self.n_pos != 0:
            raise ValueError("sequencing error (S:57)")
        P = k.shape[0]
        self.o_pos = np.arange(P, dtype=np.int64)
        self.o_k = np.asarray(k, dtype=np.float64).copy()
        self.o_v = np.asarray(v, dtype=np.float64).copy()
        self.n_pos = P
        self.q0 = P          # the prompt's own queries are not samples of decode tailors (R19)

    def keys_values(self):
        """Dequantized view of O ∪ Q (Alg. 1 'Reconstruction'), by state
        segment; the order does not affect attention (R26)."""
        g = self.cfg.group_size
        # dequantize() applied to every Quantized row (vectorised over rows)
        mode = self.cfg.quant_mode
        qk = code_values(self.q_kc, mode) * np.repeat(self.q_ks.astype(np.float64), g, axis=1) + \
            np.repeat(self.q_kz.astype(np.float64), g, axis=1)
        qv = code_values(self.q_vc, mode) * np.repeat(self.q_vs.astype(np.float64), g, axis=1) + \
            np.repeat(self.q_vz.astype(np.float64), g, axis=1)
        pos = np.concatenate([self.o_pos, self.q_pos])
        return pos, np.vstack([self.o_k, qk]), np.vstack([self.o_v, qv])

    def eligible(self):
        """(eligible positions ascending, window positions): the window is the W highest
        positions, all Original (A13)."""
        W = self.cfg.window
        allpos = np.concatenate([self.o_pos, self.q_pos])
        win = set(np.sort(allpos)[-W:].tolist())
        assert all(p in set(self.o_pos.tolist()) for p in win), "window must be Original"
        elig = np.array(sorted(p for p in allpos.tolist() if p not in win), dtype=np.int64)
        return elig, win

    def scores(self, rows) -> np.ndarray:
        """Eq. 9 scores of the eligible tokens (ascending positions) from the Eq. 2 window
        rows: list of (key positions [n], probs [r][n]) (R19)."""
        elig, _ = self.eligible()
        if not rows:         # no query has run on the current cache (W = 1 edge case): S = 0
            return np.zeros(len(elig))
        blocks = []
        for kpos, pr in rows:
            col = {int(p): i for i, p in enumerate(np.asarray(kpos).tolist())}
            missing = [p for p in elig.tolist() if p not in col]
            assert not missing, "eligible token without window samples"
            blocks.append(np.asarray(pr, dtype=np.float64)[:, [col[int(p)] for p in elig]])
        return hh_scores(np.concatenate(blocks, axis=0), self.cfg.gamma)

    def tailor(self, rho: float, rows, tailor_pos: int, scores=None):
        """Eq. 10 tailor (Alg. 1) with the D6 transitions:
        O->Q quantize, Q->O promote (R24), Q->Q keep codes (R25), ->E drop.
        rows: list of (key positions [n], probs [r][n]) — the Eq. 2 window rows
        (R19); every eligible token must appear in every row.  Parity unpinned: which
        queries form the decode-time window (R19) is this design's reading.
        scores: precomputed eligible-token scores (layer-shared states, NEXT-3)."""
        cfg = self.cfg
        W = cfg.window
        K = self.n_o + self.n_q
        n_oe, n_q = tailor_counts(K, rho, cfg)
        elig, win = self.eligible()
        S = self.scores(rows) if scores is None else np.asarray(scores, dtype=np.float64)
        assert len(S) == len(elig)
        S = smooth_scores(S, elig, self.prev_score, cfg.smooth)   # R34 (identity when λ = 0)
        st = plan_states(S, elig, n_oe, n_q)
        self.prev_score = {int(p): float(x) for p, x, s_ in zip(elig, S, st) if s_ in (1, 2)}
        # score margin at the two rank thresholds (exact ties are resolved by position
        # identically on both sides; near-ties would make fp32 vs fp64 rankings differ)
        Ss = np.sort(S)[::-1]
        for r in (n_oe, n_oe + n_q):
            if 0 < r < len(Ss) and Ss[r - 1] != Ss[r]:
                self.margins.append(float((Ss[r - 1] - Ss[r]) / max(abs(Ss[r - 1]), 1e-300)))
        new_state = {int(p): int(s) for p, s in zip(elig, st)}
        for p in win:
            new_state[int(p)] = 1
        g, bits, mode = cfg.group_size, cfg.quant_bits, cfg.quant_mode
        o_pos, o_k, o_v = [], [], []
        q_pos, q_kc, q_vc, q_ks, q_kz, q_vs, q_vz = [], [], [], [], [], [], []
        for i, p in enumerate(self.o_pos.tolist()):
            s = new_state[p]
            if s == 1:
                o_pos.append(p); o_k.append(self.o_k[i]); o_v.append(self.o_v[i])
            elif s == 2:
                kc, ks, kz = quantize(self.o_k[i], bits, g, mode)
                vc, vs, vz = quantize(self.o_v[i], bits, g, mode)
                q_pos.append(p); q_kc.append(kc); q_vc.append(vc)
                q_ks.append(ks); q_kz.append(kz); q_vs.append(vs); q_vz.append(vz)
            else:
                self.evicted.append(p)
        for i, p in enumerate(self.q_pos.tolist()):
            s = new_state[p]
            if s == 1:
                o_pos.append(p)
                o_k.append(promote(self.q_kc[i], self.q_ks[i], self.q_kz[i], g, mode))
                o_v.append(promote(self.q_vc[i], self.q_vs[i], self.q_vz[i], g, mode))
            elif s == 2:
                q_pos.append(p); q_kc.append(self.q_kc[i]); q_vc.append(self.q_vc[i])
                q_ks.append(self.q_ks[i]); q_kz.append(self.q_kz[i]); q_vs.append(self.q_vs[i]); q_vz.append(self.q_vz[i])
            else:
                self.evicted.append(p)
        d, ng = cfg.head_dim, cfg.n_groups
        oo = np.argsort(o_pos, kind="stable")
        self.o_pos = np.array(o_pos, dtype=np.int64)[oo]
        self.o_k = np.array(o_k).reshape(-1, d)[oo]
        self.o_v = np.array(o_v).reshape(-1, d)[oo]
        qo = np.argsort(q_pos, kind="stable")
        self.q_pos = np.array(q_pos, dtype=np.int64)[qo]
        self.q_kc = np.array(q_kc, dtype=np.int64).reshape(-1, d)[qo]
        self.q_vc = np.array(q_vc, dtype=np.int64).reshape(-1, d)[qo]
        self.q_ks = np.array(q_ks, dtype=F32).reshape(-1, ng)[qo]
        self.q_kz = np.array(q_kz, dtype=F32).reshape(-1, ng)[qo]
        self.q_vs = np.array(q_vs, dtype=F32).reshape(-1, ng)[qo]
        self.q_vz = np.array(q_vz, dtype=F32).reshape(-1, ng)[qo]
        assert self.n_o == n_oe + W and self.n_q == n_q
        assert self.usage() <= budget_bytes(cfg) - W * cost_orig(cfg)
        self.tailors.append((tailor_pos, self.n_o, self.n_q, K - W - n_oe - n_q))
        self.last_tailor_pos = tailor_pos
        self.q0 = tailor_pos     # the tailor step's own query runs after it (R13)
        self.history = []

    def export(self):
        """State by position (0 absent, 1 O, 2 Q, 3 E) with O values and Q codes,
        scales and zeros by position (the arkv_export_unit contract)."""
        cfg = self.cfg
        n, d, ng = self.n_pos, cfg.head_dim, cfg.n_groups
        st = np.zeros(n, dtype=np.int8)
        st[np.asarray(self.evicted, dtype=np.int64)] = 3
        ok = np.zeros((n, d)); ov = np.zeros((n, d))
        qk = np.zeros((n, d), dtype=np.int64); qv = np.zeros((n, d), dtype=np.int64)
        ks = np.zeros((n, ng), dtype=F32); kz = np.zeros((n, ng), dtype=F32)
        vs = np.zeros((n, ng), dtype=F32); vz = np.zeros((n, ng), dtype=F32)
        st[self.o_pos] = 1
        ok[self.o_pos] = self.o_k; ov[self.o_pos] = self.o_v
        st[self.q_pos] = 2
        qk[self.q_pos] = self.q_kc; qv[self.q_pos] = self.q_vc
        ks[self.q_pos] = self.q_ks; kz[self.q_pos] = self.q_kz
        vs[self.q_pos] = self.q_vs; vz[self.q_pos] = self.q_vz
        return dict(state=st, o_k=ok, o_v=ov, q_k=qk, q_v=qv, k_scale=ks, k_zero=kz,
                    v_scale=vs, v_zero=vz, n_o=self.n_o, n_q=self.n_q)


class OracleARKV:
    """Alg. 1 end to end for B sequences × L layers × H_kv KV heads (units are
    independent given ρ, R11/R20).  Prefill: stats (Eqs. 2-7) → counts (R9) →
    ingest + prefill-end tailor (R14) seeded with Ã.  Decode step: per unit
    append → tailor if over budget (R12, R13) → attention over O ∪ Q (D7), and the
    step's attention rows are kept for the next tailor's Eq. 2 window (R19)."""

    def __init__(self, cfg: Cfg):
        validate(cfg)
        self.cfg = cfg
        self.units: Dict[Tuple[int, int, int], UnitCache] = {}
        self.rho = None
        self.P = None

    def prefill(self, q_win, k, v, rho_override=None):
        cfg = self.cfg
        Bn, L, Hkv, P, d = k.shape
        G, W = cfg.G, cfg.window
        self.P = P
        stats = oq = None
        at = None
        if P - W >= 2:
            stats, oq, rho, at = prefill_stats(q_win, k, cfg)
        else:
            rho = np.ones((Bn, L))           # R28
        if rho_override is not None:
            rho = np.asarray(rho_override, dtype=np.float64).reshape(Bn, L)
        self.rho = rho
        for b in range(Bn):
            for l in range(L):
                rows = {}
                for kvh in range(Hkv):
                    u = UnitCache(cfg)
                    u.ingest(k[b, l, kvh], v[b, l, kvh])
                    self.units[(b, l, kvh)] = u
                    if prefill_needs_tailor(P, cfg):
                        if at is None:
                            at = {}
                        a = at.get((b, l))
                        if a is None:
                            a = windowed_attention(q_win[b, l], k[b, l], cfg)
                            at[(b, l)] = a
                        rows[kvh] = [(np.arange(P - W), a[kvh * G:(kvh + 1) * G].reshape(G * W, P - W))]
                if rows:
                    self._tailor_layer(b, l, rows, P)
        return stats, oq, rho

    def _tailor_layer(self, b, l, rows, pos):
        """Tailor of every KV head of (b, l): independent selections (R20), or one
        selection from the score averaged across the groups (NEXT-3)."""
        units = [self.units[(b, l, kvh)] for kvh in range(self.cfg.n_kv_heads)]
        if self.cfg.state_sharing == "head":
            for kvh, u in enumerate(units):
                u.tailor(self.rho[b, l], rows[kvh], pos)
            return
        elig = [u.eligible()[0] for u in units]
        assert all(np.array_equal(e, elig[0]) for e in elig), "layer-shared units hold the same tokens"
        S = np.mean([u.scores(rows[kvh]) for kvh, u in enumerate(units)], axis=0)
        for kvh, u in enumerate(units):
            u.tailor(self.rho[b, l], rows[kvh], pos, scores=S)

    def decode_step(self, q, k, v, layer0: int = 0):
        """q [B][n][H_q][d], k, v [B][n][H_kv][d] for layers layer0..layer0+n-1.
        Returns out [B][n][H_q][d] (float64)."""
        cfg = self.cfg
        Bn, n = q.shape[0], q.shape[1]
        G, W = cfg.G, cfg.window
        out = np.zeros(q.shape, dtype=np.float64)
        for b in range(Bn):
            for li in range(n):
                l = layer0 + li
                rows = {}
                for kvh in range(cfg.n_kv_heads):
                    u = self.units[(b, l, kvh)]
                    t = u.n_pos
                    u.append(t, k[b, li, kvh], v[b, li, kvh])
                    if decode_needs_tailor(u.n_o, u.n_q, cfg):
                        # R19: the last W queries before the tailor that ran on the current
                        # cache, i.e. positions max(t - W, q0) .. t - 1 (fewer than W only for
                        # the first tailor after the prompt)
                        hist = [h for h in u.history[-W:] if h[0] >= u.q0]
                        assert [h[0] for h in hist] == list(range(max(t - W, u.q0), t)), \
                            "tailor window must be the last W queries on the current cache"
                        rows[kvh] = [(h[1], h[2]) for h in hist]
                if rows:
                    assert len(rows) == cfg.n_kv_heads   # counts are identical across KV heads (R15)
                    self._tailor_layer(b, l, rows, t)
                for kvh in range(cfg.n_kv_heads):
                    u = self.units[(b, l, kvh)]
                    t = u.n_pos - 1
                    pos, keys, vals = u.keys_values()
                    o, p = attention(q[b, li, kvh * G:(kvh + 1) * G], keys, vals, cfg.sm_scale)
                    out[b, li, kvh * G:(kvh + 1) * G] = o
                    u.history.append((t, pos, p))
                    if len(u.history) > W:
                        u.history.pop(0)
        return out

    def export(self, b, l, kvh):
        return self.units[(b, l, kvh)].export()


def dense_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, sm_scale: float) -> np.ndarray:
    """Textbook softmax attention (the Base model) — used as a pin."""
    return attention(q, K, V, sm_scale)[0]
