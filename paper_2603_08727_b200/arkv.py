"""Thin ctypes binding of libarkv.so (include/arkv.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; torch supplies
device memory (arena / workspace tensors) and streams.  There is no fallback: if
libarkv.so is missing or the device is not sm_100 the calls raise.
The function names mirror the C ABI: arkv_prefill_stats, arkv_decode_step, ...
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ARKV_LIBRARY: path of an A/B measurement build (libarkv_tuning.so, build.py --tuning);
# bench.py records it and refuses to print a bench line with it set
LIB_PATH = os.environ.get("ARKV_LIBRARY") or os.path.join(HERE, "libarkv.so")

LAYOUT_AUTO, LAYOUT_PLAIN, LAYOUT_FRAG = 0, 1, 2
QUANT_ASYM, QUANT_SYM, QUANT_FP8 = 0, 1, 2


class ArkvConfig(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int32), ("n_q_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("batch", ctypes.c_int32), ("window", ctypes.c_int32),
        ("budget_tokens", ctypes.c_int32), ("quant_bits", ctypes.c_int32), ("group_size", ctypes.c_int32),
        ("quant_mode", ctypes.c_int32), ("max_positions", ctypes.c_int32), ("max_prompt", ctypes.c_int32),
        ("layout", ctypes.c_int32), ("n_spare_slots", ctypes.c_int32), ("max_splits", ctypes.c_int32),
        ("decode_kernel", ctypes.c_int32),
        ("alpha", ctypes.c_double), ("tau", ctypes.c_double * 3), ("gamma", ctypes.c_double),
        ("stat_eps", ctypes.c_double), ("sm_scale", ctypes.c_float), ("state_sharing", ctypes.c_int32),
        ("smooth", ctypes.c_float),
    ]


class ArkvUnitExport(ctypes.Structure):
    _fields_ = [
        ("state", ctypes.c_void_p), ("o_k", ctypes.c_void_p), ("o_v", ctypes.c_void_p),
        ("q_k", ctypes.c_void_p), ("q_v", ctypes.c_void_p), ("k_scale", ctypes.c_void_p),
        ("k_zero", ctypes.c_void_p), ("v_scale", ctypes.c_void_p), ("v_zero", ctypes.c_void_p),
        ("n_pos", ctypes.c_int32), ("n_o", ctypes.c_int32), ("n_q", ctypes.c_int32), ("pad_", ctypes.c_int32),
    ]


EXPORTED = [
    "arkv_config_default", "arkv_cache_bytes", "arkv_cache_create", "arkv_cache_destroy",
    "arkv_prefill_stats", "arkv_decode_step", "arkv_unit_counts", "arkv_export_unit",
    "arkv_check", "arkv_schedule", "arkv_oq_score", "arkv_launch_count", "arkv_version",
    "arkv_status_string", "arkv_cache_info", "arkv_prefill_begin", "arkv_prefill_finish",
    "arkv_profile", "arkv_profile_read", "arkv_layout_check", "arkv_persist_plan_check",
    "arkv_tailor_scores", "arkv_set_tailor_scores", "arkv_split_order_check",
]

_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2603_08727_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
        P = ctypes.POINTER
        L.arkv_config_default.argtypes = [P(ArkvConfig)]
        L.arkv_cache_bytes.argtypes = [P(ArkvConfig), P(ctypes.c_size_t), P(ctypes.c_size_t)]
        L.arkv_cache_create.argtypes = [P(ArkvConfig), vp, ctypes.c_size_t, vp, ctypes.c_size_t, P(vp)]
        L.arkv_cache_destroy.argtypes = [vp]
        L.arkv_prefill_stats.argtypes = [vp, vp, vp, vp, i32, vp, vp, vp, vp, vp]
        L.arkv_decode_step.argtypes = [vp, i32, i32, vp, vp, vp, i32, i32, vp, i32, vp]
        L.arkv_unit_counts.argtypes = [vp, i32, i32, P(i32), P(i32), P(i32), P(i32)]
        L.arkv_export_unit.argtypes = [vp, i32, i32, i32, P(ArkvUnitExport), vp]
        L.arkv_check.argtypes = [vp, vp]
        L.arkv_schedule.argtypes = [P(ArkvConfig), i32, dbl, i32, P(i32), i32, P(i32)]
        L.arkv_oq_score.argtypes = [P(ArkvConfig), dbl, dbl, dbl, P(dbl), P(dbl)]
        L.arkv_layout_check.argtypes = [P(ArkvConfig), P(ctypes.c_int64)]
        L.arkv_persist_plan_check.argtypes = [P(ArkvConfig), P(i32), P(i32), i32, i32, P(i32)]
        L.arkv_split_order_check.argtypes = [P(ArkvConfig), P(i32), P(i32), i32, i32, P(i32)]
        L.arkv_tailor_scores.argtypes = [vp, i32, i32, vp, ctypes.c_int64, i32, P(i32), vp]
        L.arkv_set_tailor_scores.argtypes = [vp, vp, ctypes.c_int64, i32]
        L.arkv_cache_info.argtypes = [vp, i32]
        L.arkv_cache_info.restype = ctypes.c_int32
        L.arkv_prefill_begin.argtypes = [vp, vp, vp, i32, vp, vp]
        L.arkv_prefill_finish.argtypes = [vp, vp, vp, i32, vp, vp, vp, vp, vp, vp]
        L.arkv_profile.argtypes = [vp, i32]
        L.arkv_profile_read.argtypes = [vp, i32, P(dbl), P(ctypes.c_int64), P(dbl)]
        L.arkv_launch_count.argtypes = [vp]
        L.arkv_launch_count.restype = ctypes.c_int64
        L.arkv_version.restype = ctypes.c_char_p
        L.arkv_status_string.restype = ctypes.c_char_p
        L.arkv_status_string.argtypes = [ctypes.c_int]
        for n in EXPORTED:
            if n not in ("arkv_launch_count", "arkv_version", "arkv_status_string", "arkv_cache_info"):
                getattr(L, n).restype = ctypes.c_int
        _lib = L
    return _lib


class ArkvError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {lib().arkv_status_string(code).decode()} ({code})")


def _ok(code: int, what: str):
    if code != 0:
        raise ArkvError(code, what)


def make_config(n_layers, n_q_heads, n_kv_heads, head_dim, batch=1, window=32, budget_tokens=512,
                quant_bits=4, group_size=0, quant_mode=QUANT_ASYM, max_positions=4096, max_prompt=None,
                layout=LAYOUT_AUTO, n_spare_slots=0, max_splits=0, decode_kernel=0, alpha=0.75,
                tau=(7.774, 5.407, 5.528), gamma=263.81, stat_eps=1e-30, sm_scale=0.0,
                state_sharing=0, smooth=0.0) -> ArkvConfig:
    c = ArkvConfig()
    _ok(lib().arkv_config_default(ctypes.byref(c)), "arkv_config_default")
    c.n_layers, c.n_q_heads, c.n_kv_heads, c.head_dim, c.batch = n_layers, n_q_heads, n_kv_heads, head_dim, batch
    c.window, c.budget_tokens, c.quant_bits, c.group_size = window, budget_tokens, quant_bits, group_size
    c.quant_mode, c.max_positions = quant_mode, max_positions
    c.max_prompt = max_prompt if max_prompt is not None else max_positions - 1
    c.layout, c.n_spare_slots, c.max_splits, c.decode_kernel = layout, n_spare_slots, max_splits, decode_kernel
    c.alpha, c.gamma, c.stat_eps, c.sm_scale = alpha, gamma, stat_eps, sm_scale
    c.state_sharing = state_sharing
    c.smooth = smooth
    for i in range(3):
        c.tau[i] = tau[i]
    return c


def arkv_cache_bytes(cfg: ArkvConfig):
    a, w = ctypes.c_size_t(), ctypes.c_size_t()
    _ok(lib().arkv_cache_bytes(ctypes.byref(cfg), ctypes.byref(a), ctypes.byref(w)), "arkv_cache_bytes")
    return a.value, w.value


def arkv_schedule(cfg: ArkvConfig, prompt_len: int, rho: float, n_steps: int, max_events: int = 4096):
    ev = (ctypes.c_int32 * (4 * max_events))()
    n = ctypes.c_int32()
    _ok(lib().arkv_schedule(ctypes.byref(cfg), prompt_len, rho, n_steps, ev, max_events, ctypes.byref(n)),
        "arkv_schedule")
    return [tuple(ev[4 * i:4 * i + 4]) for i in range(min(n.value, max_events))]


def arkv_layout_check(cfg: ArkvConfig) -> int:
    n = ctypes.c_int64()
    _ok(lib().arkv_layout_check(ctypes.byref(cfg), ctypes.byref(n)), "arkv_layout_check")
    return n.value


def arkv_persist_plan_check(cfg: ArkvConfig, n_o, n_q, max_ctas: int) -> int:
    """Builds the persistent kernel's plan for these per-unit counts and replays it on the
    host (include/arkv.h); raises ArkvError on a violated invariant.  Returns the grid size."""
    n = len(n_o)
    a = (ctypes.c_int32 * n)(*[int(x) for x in n_o])
    b = (ctypes.c_int32 * n)(*[int(x) for x in n_q])
    used = ctypes.c_int32()
    _ok(lib().arkv_persist_plan_check(ctypes.byref(cfg), a, b, n, max_ctas, ctypes.byref(used)),
        "arkv_persist_plan_check")
    return used.value


def arkv_split_order_check(cfg: ArkvConfig, n_o, n_q, num_sms: int = 148) -> int:
    """Builds the split-K decode kernel's cost-balanced launch order for these per-(sequence,
    layer) counts and replays it on the host (include/arkv.h); raises ArkvError on a violated
    invariant.  Returns the grid size."""
    n = len(n_o)
    a = (ctypes.c_int32 * n)(*[int(x) for x in n_o])
    b = (ctypes.c_int32 * n)(*[int(x) for x in n_q])
    used = ctypes.c_int32()
    _ok(lib().arkv_split_order_check(ctypes.byref(cfg), a, b, n, num_sms, ctypes.byref(used)),
        "arkv_split_order_check")
    return used.value


def arkv_oq_score(cfg: ArkvConfig, entropy: float, m2: float, m4: float):
    st = (ctypes.c_double * 3)()
    sc = ctypes.c_double()
    _ok(lib().arkv_oq_score(ctypes.byref(cfg), entropy, m2, m4, st, ctypes.byref(sc)), "arkv_oq_score")
    return tuple(st), sc.value


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class ArkvCache:
    """Owns the torch-allocated arena/workspace and the library cache handle."""

    def __init__(self, cfg: ArkvConfig, device="cuda"):
        import torch
        self.cfg = cfg
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        a, w = arkv_cache_bytes(cfg)
        self.arena_bytes, self.workspace_bytes = a, w
        self.arena = torch.empty(a + 256, dtype=torch.uint8, device=self.device)
        self.workspace = torch.empty(w + 256, dtype=torch.uint8, device=self.device)
        ap = (self.arena.data_ptr() + 255) // 256 * 256
        wp = (self.workspace.data_ptr() + 255) // 256 * 256
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _ok(lib().arkv_cache_create(ctypes.byref(cfg), ap, a, wp, w, ctypes.byref(h)), "arkv_cache_create")
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().arkv_cache_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    # --- C ABI mirrors ---------------------------------------------------------
    def arkv_prefill_stats(self, q_win, k, v, rho_override=None, stats=None, oq=None, stream=None):
        import torch
        B, L = self.cfg.batch, self.cfg.n_layers
        P = k.shape[-2]
        for t in (q_win, k, v):
            assert t is None or (t.dtype == torch.bfloat16 and t.is_contiguous() and t.device == self.device)
        if stats is None:
            stats = torch.empty(B, L, 3, dtype=torch.float64, device=self.device)
        if oq is None:
            oq = torch.empty(B, L, dtype=torch.float64, device=self.device)
        rho = (ctypes.c_double * (B * L))()
        ro = None
        if rho_override is not None:
            arr = np.ascontiguousarray(np.asarray(rho_override, dtype=np.float64).reshape(B * L))
            ro = (ctypes.c_double * (B * L))(*arr.tolist())
        _ok(lib().arkv_prefill_stats(self.handle, _ptr(q_win), _ptr(k), _ptr(v), P, ro, _ptr(stats), _ptr(oq), rho,
                                     _stream_ptr(stream)), "arkv_prefill_stats")
        return stats, oq, np.array(rho[:]).reshape(B, L)

    def arkv_prefill_begin(self, q_win, k, colsum=None, stream=None):
        """Passes 1-2 and the local Eq. 3 column sums [B][L][max_positions] (float64)."""
        import torch
        B, L = self.cfg.batch, self.cfg.n_layers
        if colsum is None:
            colsum = torch.zeros(B, L, self.cfg.max_positions, dtype=torch.float64, device=self.device)
        _ok(lib().arkv_prefill_begin(self.handle, _ptr(q_win), _ptr(k), k.shape[-2], _ptr(colsum),
                                     _stream_ptr(stream)), "arkv_prefill_begin")
        return colsum

    def arkv_prefill_finish(self, k, v, colsum, rho_override=None, stats=None, oq=None, stream=None):
        import torch
        B, L = self.cfg.batch, self.cfg.n_layers
        if stats is None:
            stats = torch.empty(B, L, 3, dtype=torch.float64, device=self.device)
        if oq is None:
            oq = torch.empty(B, L, dtype=torch.float64, device=self.device)
        rho = (ctypes.c_double * (B * L))()
        ro = None
        if rho_override is not None:
            arr = np.asarray(rho_override, dtype=np.float64).reshape(B * L)
            ro = (ctypes.c_double * (B * L))(*arr.tolist())
        _ok(lib().arkv_prefill_finish(self.handle, _ptr(k), _ptr(v), k.shape[-2], _ptr(colsum), ro, _ptr(stats),
                                      _ptr(oq), rho, _stream_ptr(stream)), "arkv_prefill_finish")
        return stats, oq, np.array(rho[:]).reshape(B, L)

    def arkv_profile(self, enable: bool):
        _ok(lib().arkv_profile(self.handle, 1 if enable else 0), "arkv_profile")

    def arkv_profile_read(self, which: int = 0):
        ms, n, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _ok(lib().arkv_profile_read(self.handle, which, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by)),
            "arkv_profile_read")
        return ms.value, n.value, by.value

    def arkv_cache_info(self, what: int) -> int:
        return int(lib().arkv_cache_info(self.handle, what))

    def arkv_decode_step(self, q, k, v, layer0=0, out=None, out_fp32=True, stream=None):
        import torch
        n = q.shape[1]
        for t in (q, k, v):
            assert t.dtype == torch.bfloat16 and t.is_contiguous() and t.device == self.device
        if out is None:
            out = torch.empty(q.shape, dtype=torch.float32 if out_fp32 else torch.bfloat16, device=self.device)
        _ok(lib().arkv_decode_step(self.handle, layer0, n, _ptr(q), _ptr(k), _ptr(v), self.cfg.budget_tokens,
                                   self.cfg.quant_bits, _ptr(out), 1 if out.dtype == torch.float32 else 0,
                                   _stream_ptr(stream)), "arkv_decode_step")
        return out

    def arkv_tailor_scores(self, scores, layer0=0, n_layers=None, stream=None) -> int:
        """Layer-shared states across KV-head shards (include/arkv.h): this cache's score
        sums for the tailors the next call runs, into scores [max_rows][stride] (fp32,
        device).  Returns the number of rows written."""
        n = ctypes.c_int32()
        n_layers = self.cfg.n_layers - layer0 if n_layers is None else n_layers
        _ok(lib().arkv_tailor_scores(self.handle, layer0, n_layers, _ptr(scores), scores.shape[1], scores.shape[0],
                                     ctypes.byref(n), _stream_ptr(stream)), "arkv_tailor_scores")
        return n.value

    def arkv_set_tailor_scores(self, scores, total_kv_heads):
        """Exchanged score sums (summed over every shard) for the next call's tailors."""
        _ok(lib().arkv_set_tailor_scores(self.handle, _ptr(scores) if scores is not None else None,
                                         scores.shape[1] if scores is not None else 0, total_kv_heads),
            "arkv_set_tailor_scores")
        self._ext_scores = scores   # keep the buffer alive until the next call has run

    def arkv_unit_counts(self, b, layer):
        n_o, n_q, p, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _ok(lib().arkv_unit_counts(self.handle, b, layer, ctypes.byref(n_o), ctypes.byref(n_q), ctypes.byref(p),
                                   ctypes.byref(t)), "arkv_unit_counts")
        return n_o.value, n_q.value, p.value, t.value

    def arkv_export_unit(self, b, layer, kvh, stream=None) -> Dict[str, np.ndarray]:
        _, _, n_pos, _ = self.arkv_unit_counts(b, layer)
        d = self.cfg.head_dim
        g = self.cfg.group_size or d
        ng = d // g
        out = dict(state=np.zeros(n_pos, np.int8), o_k=np.zeros((n_pos, d), np.uint16), o_v=np.zeros((n_pos, d), np.uint16),
                   q_k=np.zeros((n_pos, d), np.int16), q_v=np.zeros((n_pos, d), np.int16),
                   k_scale=np.zeros((n_pos, ng), np.float32), k_zero=np.zeros((n_pos, ng), np.float32),
                   v_scale=np.zeros((n_pos, ng), np.float32), v_zero=np.zeros((n_pos, ng), np.float32))
        ex = ArkvUnitExport()
        for key in ("state", "o_k", "o_v", "q_k", "q_v", "k_scale", "k_zero", "v_scale", "v_zero"):
            setattr(ex, key, out[key].ctypes.data)
        ex.n_pos = n_pos
        _ok(lib().arkv_export_unit(self.handle, b, layer, kvh, ctypes.byref(ex), _stream_ptr(stream)),
            "arkv_export_unit")
        out["n_o"], out["n_q"] = ex.n_o, ex.n_q
        return out

    def arkv_check(self, stream=None):
        _ok(lib().arkv_check(self.handle, _stream_ptr(stream)), "arkv_check")

    def arkv_launch_count(self) -> int:
        return int(lib().arkv_launch_count(self.handle))


def arkv_version() -> str:
    return lib().arkv_version().decode()
