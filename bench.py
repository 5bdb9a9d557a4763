#!/usr/bin/env python
"""bench.py — ARKV decode-step throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload llama3-8b-32k] [--impl arkv|reference]

A step = one decode token for every sequence through all L layers of the workload
(append -> tailor when due -> attention over O ∪ Q with HH accumulation), issued as
one arkv_decode_step call covering all layers.  The prompt (prefill statistics,
ingest, prefill-end tailor) runs before the timed region.  Inputs are synthetic
(synth/, natural recipe), resident in HBM before timing; the cache (> 1 GB at
configs[1]) is far larger than the 126 MB L2, so no flush is needed between steps.

Multi-GPU (torchrun, one process per GPU): weak scaling — every rank holds whole
sequences (batch x all KV heads), so the decode loop has no collective; NCCL only
gathers per-layer statistics and the max-over-ranks time.  `--impl reference` times
the float64 CPU oracle (oracle/) on the box's host cores on a bounded sample of the
same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the headline configuration (1 GPU)
    "llama3-8b-32k": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=1, prompt_len=32768,
                          budget=8192, window=32, bits=4, group=128, baseline_cfg=1),
    # configs[2]
    "qwen3-8b-8k-b8": dict(n_layers=36, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=8, prompt_len=8192,
                           budget=2048, window=32, bits=4, group=128, baseline_cfg=2),
    # configs[3]
    "llama3-8b-1k-b64": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=64, prompt_len=1024,
                             budget=2048, window=32, bits=4, group=128, baseline_cfg=3),
    # configs[4] (per-GPU share: 1 sequence of 128K)
    "llama3-8b-128k": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=1, prompt_len=131072,
                           budget=16384, window=32, bits=4, group=128, baseline_cfg=4),
}

METRIC = "ARKV decode tokens/s + HBM GB/s vs peak, Llama3-8B shape 32K ctx, 1/2/4/8 GPU"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def unit_counts_summary(cache, wl):
    import numpy as np
    B, L = wl["batch"], wl["n_layers"]
    n_o = np.zeros((B, L), np.int64)
    n_q = np.zeros((B, L), np.int64)
    pos = np.zeros((B, L), np.int64)
    for b in range(B):
        for l in range(L):
            n_o[b, l], n_q[b, l], pos[b, l], _ = cache.arkv_unit_counts(b, l)
    return n_o, n_q, pos


def cache_bytes_per_step(cache, wl, n_o, n_q):
    d, G, Hkv = wl["head_dim"], wl["n_q_heads"] // wl["n_kv_heads"], wl["n_kv_heads"]
    co = 4 * d
    cq = 2 * (d * wl["bits"] // 8 + 8 * (d // wl["group"]))
    return float(Hkv * ((n_o * co + n_q * cq).sum() + n_o.size * (2 * co + 2 * G * d)))


def run_arkv(args, wl):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2603_08727_b200 import arkv as A
    from synth import Shape, prefill_inputs_fast, decode_inputs_fast

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, L, Hq, Hkv, d, P = (wl["batch"], wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"],
                           wl["prompt_len"])
    K, Wm = args.steps, args.warmup
    n_e2e = args.e2e_steps
    # kernel window: the decode kernel's duration is read from CUDA event pairs the library
    # records around each launch; event records between PDL launches add 5-9 us per step,
    # so they run in a second window of the same workload right after the timed one
    Kk = 0 if args.no_kernel_events else min(K, 512)
    total_steps = Wm + K + Kk + n_e2e
    budget = wl["budget"]
    if args.mode == "base":            # Base: no cache limit -> every token stays bf16
        budget = P + total_steps + 2 * wl["window"] + 1
    cfg = A.make_config(L, Hq, Hkv, d, batch=B, window=wl["window"], budget_tokens=budget,
                        quant_bits=wl["bits"], group_size=wl["group"], max_positions=P + total_steps + 1,
                        quant_mode={"asym": A.QUANT_ASYM, "fp8": A.QUANT_FP8}[wl["qmode"]],
                        state_sharing=1 if args.sharing == "layer" else 0, smooth=args.smooth,
                        max_prompt=P, decode_kernel=args.kernel)
    cache = A.ArkvCache(cfg, dev)
    sh = Shape(batch=B, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=wl["window"])
    seed = 1234 + 7919 * rank
    # ---- prefill (untimed) ----
    qw, k, v = prefill_inputs_fast(sh, seed=seed, device=dev)
    torch.cuda.synchronize()
    t0 = time.time()
    rho_override = None
    if args.mode == "origin":          # Base_origin: budgeted heavy hitters, all bf16
        rho_override = [[1.0] * L for _ in range(B)]
    elif args.mode == "quant":         # Base_quant: every kept eligible token quantized
        rho_override = [[0.0] * L for _ in range(B)]
    # P1-P4 timed on the device: one warm-up prefill on a throwaway cache (first-launch
    # costs), then CUDA events around arkv_prefill_begin (P1 both passes + column sums) and
    # arkv_prefill_finish (P2-P4: moments, rho, ingest, prefill-end tailor)
    colsum = torch.zeros(B, L, cfg.max_positions, dtype=torch.float64, device=dev)
    warm = A.ArkvCache(cfg, dev)  # a throwaway cache takes the first-launch costs of every prefill kernel
    warm.arkv_prefill_finish(k, v, warm.arkv_prefill_begin(qw, k, colsum=colsum), rho_override=rho_override)
    warm.arkv_check()
    del warm
    colsum.zero_()
    pev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    pev[0].record()
    cache.arkv_prefill_begin(qw, k, colsum=colsum)
    pev[1].record()
    stats, oq, rho = cache.arkv_prefill_finish(k, v, colsum, rho_override=rho_override)
    pev[2].record()
    cache.arkv_check()
    prefill_s = time.time() - t0
    p1_ms, p24_ms = pev[0].elapsed_time(pev[1]), pev[1].elapsed_time(pev[2])
    k_pass_bytes = 2.0 * B * L * Hkv * P * d * 2  # K read once per pass (P1 algorithmic bytes)
    del colsum
    del qw, k, v
    torch.cuda.empty_cache()
    # ---- decode inputs, resident in HBM ----
    pool = [decode_inputs_fast(sh, s, seed=seed, device=dev) for s in range(Wm + K)]
    out = torch.empty(B, L, Hq, d, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    for s in range(Wm):
        q, kk, vv = pool[s]
        cache.arkv_decode_step(q, kk, vv, out=out)
    cache.arkv_check()
    n_o0, n_q0, pos0 = unit_counts_summary(cache, wl)
    sched = [A.arkv_schedule(cfg, P, float(rho[b, l]), Wm + K) for b in range(B) for l in range(L)]
    tailors_timed = sum(1 for ev in sched for e in ev if Wm <= e[0] < Wm + K) * Hkv
    launches0 = cache.arkv_launch_count()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    bytes_total = 0.0
    e0.record(stream)
    for s in range(Wm, Wm + K):
        q, kk, vv = pool[s]
        cache.arkv_decode_step(q, kk, vv, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    launches = cache.arkv_launch_count() - launches0
    n_o1, n_q1, pos1 = unit_counts_summary(cache, wl)
    # ---- kernel window (event pairs around every decode-kernel launch) ----
    cache.arkv_profile(True)
    for i in range(Kk):
        q, kk, vv = pool[Wm + i % K]
        cache.arkv_decode_step(q, kk, vv, out=out)
    torch.cuda.synchronize()
    k_ms, k_cnt, k_by = cache.arkv_profile_read(0)
    cache.arkv_profile(False)
    cache.arkv_check()
    # ---- e2e through the public API with host buffers ----
    e2e = None
    if n_e2e > 0:
        # serving-style pipeline: step s+1's q/k/v are copied host->device on one stream
        # while step s computes; each step's output is copied device->host on another
        n_host = min(16, len(pool))
        hq = [[t.cpu().pin_memory() for t in pool[i]] for i in range(n_host)]
        dq = [[torch.empty_like(t) for t in pool[0]] for _ in range(2)]
        hout = [torch.empty(out.shape, dtype=out.dtype, pin_memory=True) for _ in range(2)]
        outs = [torch.empty_like(out) for _ in range(2)]
        h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        copied = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        computed = [torch.cuda.Event() for _ in range(2)]
        drained = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        h2d.wait_event(f0)

        def issue_copy(step):
            b2 = step % 2
            with torch.cuda.stream(h2d):
                if step >= 2:
                    h2d.wait_event(consumed[b2])
                for dd, hh in zip(dq[b2], hq[step % n_host]):
                    dd.copy_(hh, non_blocking=True)
                copied[b2].record(h2d)

        issue_copy(0)
        for s in range(n_e2e):
            b2 = s % 2
            if s + 1 < n_e2e:
                issue_copy(s + 1)
            stream.wait_event(copied[b2])
            if s >= 2:
                stream.wait_event(drained[b2])           # outs[b2] free again
            cache.arkv_decode_step(dq[b2][0], dq[b2][1], dq[b2][2], out=outs[b2])
            consumed[b2].record(stream)
            computed[b2].record(stream)
            with torch.cuda.stream(d2h):
                d2h.wait_event(computed[b2])
                hout[b2].copy_(outs[b2], non_blocking=True)
                drained[b2].record(d2h)
        stream.wait_event(drained[(n_e2e - 1) % 2])
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1)
        if ws > 1:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": ws * B * n_e2e / (e2e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in hq[0])),
               "d2h_bytes_per_step": int(hout[0].numel() * hout[0].element_size()),
               "pipeline": "H2D of step s+1 and D2H of step s overlap step s's compute (two copy streams)",
               "window": f"{n_e2e} decode steps following the device-timed and kernel windows"}
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        rr = torch.tensor(rho.reshape(-1), device=dev, dtype=torch.float64)
        gathered = [torch.empty_like(rr) for _ in range(ws)]
        dist.all_gather(gathered, rr)
        rho_all = torch.cat(gathered).cpu().numpy()
    else:
        rho_all = rho.reshape(-1)
    peak, peak_src = peaks()
    read_ceiling = read_ceiling_gbs(dev) if not args.no_ceiling else None
    value = ws * B * K / (ms / 1e3)
    step_bytes = (cache_bytes_per_step(cache, wl, n_o0, n_q0) + cache_bytes_per_step(cache, wl, n_o1, n_q1)) / 2
    kernel_ms = k_ms / max(k_cnt, 1)
    achieved = (k_by / max(k_cnt, 1)) / (kernel_ms / 1e3) / 1e9 if k_cnt else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if args.mode == "arkv":
                traffic = tj.get(args.workload, {}).get(cache_kernel(cache), {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    budget_tokens = B * L * Hkv * budget
    evicted = float(((pos1 - n_o1 - n_q1)).sum())
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": ws,
        "steps": K,
        "warmup": Wm,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16+int4 (fp32 accumulate)" if wl["qmode"] == "asym" else "bf16+fp8e4m3 (fp32 accumulate)",
        "data": "synthetic (synth/ natural recipe: sinks, 5% log-normal heavy hitters, recency bump, x8 outlier V channels)",
        "config": {"workload": f"{args.workload} (BASELINE.json configs[{wl['baseline_cfg']}])",
                   "layers": L, "q_heads": Hq, "kv_heads": Hkv, "head_dim": d, "batch_per_gpu": B,
                   "global_batch": B * ws, "prompt_len": P, "budget_tokens": budget, "window": wl["window"], "mode": args.mode,
                   "state_sharing": args.sharing, "smooth": args.smooth,
                   "quant": (f"int{wl['bits']} g{wl['group']} asym" if wl["qmode"] == "asym"
                             else f"fp8 e4m3 g{wl['group']}"), "alpha": 0.75,
                   "launch": "one arkv_decode_step per step covering all layers (layer-batched)",
                   "decode_kernel": cache_kernel(cache),
                   "parallelism": f"dp{ws} (whole sequences per GPU, no collective in the loop)",
                   "l2": "no flush: cache arena %.2f GB >> 126 MB L2" % (cache.arena_bytes / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "decode attention kernel (%s)" % cache_kernel(cache), "kernel_ms_per_launch": kernel_ms,
                     "alg_bytes_per_launch": k_by / max(k_cnt, 1), "peak_source": peak_src,
                     "timing": f"CUDA event pairs around each of {k_cnt} decode-kernel launches on the launching "
                               f"stream, in a window of {Kk} steps right after the timed one (event records "
                               f"between PDL launches would slow the timed steps)"},
        "step_hbm": {"alg_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms / K / 1e3) / 1e9,
                     "frac_of_peak": step_bytes / (ms / K / 1e3) / 1e9 / peak,
                     "frac_of_8tbs_nominal": step_bytes / (ms / K / 1e3) / 1e12 / 8.0},
        "read_ceiling": {"gbs": read_ceiling, "how": "best of torch amax/sum over a 2 GiB bf16 tensor (reference only)"},
        "gpu_launches": int(launches),
        "tailors_in_timed_region": int(tailors_timed),
        "memory": {"arena_bytes": cache.arena_bytes, "dense_bf16_bytes": B * L * Hkv * (P + total_steps) * 4 * d,
                   "quant_ratio": float(n_q1.sum() * Hkv / budget_tokens), "evict_ratio": evicted / float(pos1.sum()),
                   "n_o_range": [int(n_o1.min()), int(n_o1.max())], "n_q_range": [int(n_q1.min()), int(n_q1.max())]},
        "rho": {"min": float(rho_all.min()), "median": float(statistics.median(rho_all.tolist())),
                "max": float(rho_all.max())},
        "prefill_s": prefill_s,
        "prefill": {"stats_ms": p1_ms, "finish_ms": p24_ms, "stats_alg_bytes": k_pass_bytes,
                    "stats_gbs": k_pass_bytes / (p1_ms / 1e3) / 1e9,
                    "stats_frac": k_pass_bytes / (p1_ms / 1e3) / 1e9 / peak,
                    "kernel": "prefill_ws_kernel (P1: tcgen05 + TMA, two passes over K) + column sums",
                    "timing": "CUDA events around arkv_prefill_begin / arkv_prefill_finish, after one warm-up "
                              "prefill on a throwaway cache"},
        "clocks": clocks,
        "e2e": e2e,
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, rho[0], samples=args.cpu_steps)
    if ws > 1:
        dist.destroy_process_group()
    return line, rank


def read_ceiling_gbs(dev) -> float:
    """Reference read-only HBM ceiling: best of two torch reductions over 2 GiB."""
    import torch
    x = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev).uniform_()
    best = 0.0
    for fn in (lambda: x.amax(), lambda: x.sum(dtype=torch.float32)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 10 * x.numel() * 2 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    del x
    torch.cuda.empty_cache()
    return best


def cache_kernel(cache) -> str:
    from paper_2603_08727_b200 import arkv as A
    return {0: "generic", 1: "fast", 2: "persistent"}[A.lib().arkv_cache_info(cache.handle, 1)]


def cpu_baseline(wl, rho_seq, samples=4):
    """The float64 oracle as it stands on the host cores: one layer (median rho of the
    sequence) x all KV heads; untimed prefill, then `samples` timed decode steps;
    tokens/s extrapolated to all L layers."""
    import numpy as np
    import oracle as O
    from synth import Shape, prefill_inputs_fast, decode_inputs_fast
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
    except Exception:
        threads = os.cpu_count() or 1
    L, Hq, Hkv, d, P = wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"], wl["prompt_len"]
    li = int(np.argsort(rho_seq)[len(rho_seq) // 2])
    r = float(rho_seq[li])
    sh1 = Shape(batch=1, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=wl["window"])
    qw, k, v = prefill_inputs_fast(sh1, seed=1234, device="cpu")
    cfg = O.Cfg(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, window=wl["window"], budget_tokens=wl["budget"],
                quant_bits=wl["bits"], group_size=wl["group"], quant_mode=wl.get("qmode", "asym"))
    ora = O.OracleARKV(cfg)
    f = lambda t: t.double().numpy()  # noqa: E731
    ora.prefill(f(qw[:, li:li + 1]), f(k[:, li:li + 1]), f(v[:, li:li + 1]), rho_override=[[r]])
    times = []
    for s in range(samples):
        q, kn, vn = decode_inputs_fast(sh1, s, seed=1234, device="cpu")
        t0 = time.perf_counter()
        ora.decode_step(f(q[:, li:li + 1]), f(kn[:, li:li + 1]), f(vn[:, li:li + 1]))
        times.append(time.perf_counter() - t0)
    per_layer = statistics.mean(times)
    return {"value": 1.0 / (per_layer * L), "unit": "tokens/s", "cores": int(threads), "kind": "oracle",
            "sample": f"layer {li} (rho={r:.3f}) x {Hkv} KV heads x {samples} decode steps after a {P}-token "
                      f"prefill; float64 numpy; tokens/s extrapolated to {L} layers"}


def run_reference(args, wl):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return None, rank
    import numpy as np
    import oracle as O
    from synth import Shape, prefill_inputs_fast, decode_inputs_fast
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
    except Exception:
        threads = os.cpu_count() or 1
    L, Hq, Hkv, d, P = wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"], wl["prompt_len"]
    sh1 = Shape(batch=1, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=wl["window"])
    qw, k, v = prefill_inputs_fast(sh1, seed=1234, device="cpu")
    li = L // 2
    cfg = O.Cfg(n_layers=1, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, window=wl["window"], budget_tokens=wl["budget"],
                quant_bits=wl["bits"], group_size=wl["group"], quant_mode=wl.get("qmode", "asym"))
    ora = O.OracleARKV(cfg)
    f = lambda t: t.double().numpy()  # noqa: E731
    ora.prefill(f(qw[:, li:li + 1]), f(k[:, li:li + 1]), f(v[:, li:li + 1]), rho_override=[[0.6]])
    for s in range(args.warmup):
        q, kn, vn = decode_inputs_fast(sh1, s, seed=1234, device="cpu")
        ora.decode_step(f(q[:, li:li + 1]), f(kn[:, li:li + 1]), f(vn[:, li:li + 1]))
    t0 = time.perf_counter()
    for s in range(args.warmup, args.warmup + args.steps):
        q, kn, vn = decode_inputs_fast(sh1, s, seed=1234, device="cpu")
        ora.decode_step(f(q[:, li:li + 1]), f(kn[:, li:li + 1]), f(vn[:, li:li + 1]))
    el = time.perf_counter() - t0
    per_step = el / args.steps * L      # one sampled layer per step, extrapolated to L layers
    value = wl["batch"] / per_step
    sample = (f"each step: layer {li} of {L} (rho=0.6) x {Hkv} KV heads of one sequence, float64 numpy oracle; "
              f"time x {L} layers")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload} (BASELINE.json configs[{wl['baseline_cfg']}])"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": int(threads), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}, 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="arkv", choices=["arkv", "reference"])
    ap.add_argument("--workload", default="llama3-8b-32k", choices=sorted(WORKLOADS))
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 generic, 2 fast split-K, 3 fast persistent")
    ap.add_argument("--e2e-steps", type=int, default=-1, help="-1: same as --steps")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="debug: no library event pairs around the decode kernel in the timed region")
    ap.add_argument("--mode", default="arkv", choices=["arkv", "base", "origin", "quant"],
                    help="arkv (stats-driven rho) or the paper's baselines: base, origin (rho=1), quant (rho=0)")
    ap.add_argument("--prompt-len", type=int, default=0, help="debug: override the workload's prompt length")
    ap.add_argument("--layers", type=int, default=0, help="debug: override the workload's layer count")
    ap.add_argument("--smooth", type=float, default=0.0,
                    help="lambda of the smoothed heavy-hitter scores (NEXT-4, reading R34); 0 = off")
    ap.add_argument("--sharing", default="head", choices=["head", "layer"],
                    help="token states per KV head (R20) or per layer from group-averaged scores (NEXT-3)")
    ap.add_argument("--quant", default="int4", choices=["int4", "fp8"],
                    help="Q-token format: int4 g128 asymmetric (default) or fp8 e4m3 per-token scale (NEXT-2)")
    args = ap.parse_args()
    if args.e2e_steps < 0:
        args.e2e_steps = args.steps
    wl = dict(WORKLOADS[args.workload])
    if args.prompt_len:
        wl["prompt_len"] = args.prompt_len
    if args.layers:
        wl["n_layers"] = args.layers
    wl["qmode"] = "asym"
    if args.quant == "fp8":
        wl.update(bits=8, group=wl["head_dim"], qmode="fp8")
    if args.impl == "reference":
        args.steps = min(args.steps, 128)   # each step is a bounded CPU sample (one layer-step)
        args.warmup = min(args.warmup, 4)
        line, rank = run_reference(args, wl)
    else:
        line, rank = run_arkv(args, wl)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
