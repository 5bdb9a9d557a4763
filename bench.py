#!/usr/bin/env python
"""bench.py — ARKV decode-step throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload llama3-8b-32k] [--impl arkv|reference]

A step = one decode token for every sequence of the workload through all L layers
(append -> tailor when due -> attention over O ∪ Q with HH accumulation), issued as one
arkv_decode_step call covering all layers ("layer-batched").  The prompt (prefill
statistics, ingest, prefill-end tailor) runs before the timed region.  Inputs are
synthetic (synth/, natural recipe) and resident in HBM before timing; the cache arena
(> 1 GB at configs[1]) is far larger than the 126 MB L2, so no flush is needed.

Every measured window covers THE SAME steps of the same workload on a fresh cache (same
prompt, same W warm-up steps, then the K measured steps): the device-timed window
(repeated, median reported), the per-launch kernel events (roofline), the end-to-end
window through host buffers (e2e) and the per-layer CUDA-graph window (H3).

Multi-GPU (north_star): `--gpus N` spawns N ranks itself (torchrun, one
process per GPU, NCCL) unless launched under torchrun.  The workload's units (sequence x
KV head) are partitioned sequence-major, then by KV head (parallel.shard_units): the
global problem is fixed (strong scaling).  Ranks sharing a sequence all-reduce Eq. 3's
column sums once at prefill (collective C1); the decode loop has no collective; the
outputs are all-gathered after the timed region (C2).  Time = max over ranks.

`--impl reference` times the float64 CPU oracle (oracle/) on the box's host cores on a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import copy
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs[1]: the headline configuration (1 GPU; 8 KV heads -> up to 8 GPUs)
    "llama3-8b-32k": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=1, prompt_len=32768,
                          budget=8192, window=32, bits=4, group=128, baseline_cfg=1),
    # configs[2]: batch 8 sharded over 2/4/8 GPUs by sequence
    "qwen3-8b-8k-b8": dict(n_layers=36, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=8, prompt_len=8192,
                           budget=2048, window=32, bits=4, group=128, baseline_cfg=2),
    # configs[3]
    "llama3-8b-1k-b64": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=64, prompt_len=1024,
                             budget=2048, window=32, bits=4, group=128, baseline_cfg=3),
    # configs[4]: batch 4 x 128K; at 8 GPUs each sequence spans 2 GPUs x 4 KV heads (C1 at prefill)
    "llama3-8b-128k-b4": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=4, prompt_len=131072,
                              budget=16384, window=32, bits=4, group=128, baseline_cfg=4),
    # configs[4]'s per-GPU share at 8 GPUs as a 1-GPU workload (one 128K sequence)
    "llama3-8b-128k": dict(n_layers=32, n_q_heads=32, n_kv_heads=8, head_dim=128, batch=1, prompt_len=131072,
                           budget=16384, window=32, bits=4, group=128, baseline_cfg=4),
}

METRIC = "ARKV decode tokens/s + HBM GB/s vs peak, Llama3-8B shape 32K ctx, 1/2/4/8 GPU"
POOL = 256  # distinct decode-input steps kept resident (steps beyond cycle through them)


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


def arkv_env():
    return {k: v for k, v in sorted(os.environ.items()) if k.startswith("ARKV_")}


def spawn_ranks(n: int) -> int:
    """`--gpus N` without torchrun: launch N ranks of this script on 127.0.0.1."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------------------
# inputs of this rank's shard (every sequence generated from its GLOBAL index, so ranks
# sharing a sequence hold bit-identical prompts and slice their own KV heads)
# ---------------------------------------------------------------------------------------
def shard_inputs(wl, shard, seed, dev, n_steps):
    import torch
    from synth import Shape, decode_inputs_fast, prefill_inputs_fast
    L, Hq, Hkv, d, P, W = (wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"], wl["prompt_len"],
                           wl["window"])
    G = Hq // Hkv
    h0, h1 = shard["kvh_lo"], shard["kvh_hi"]
    sh1 = Shape(batch=1, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=W)
    seqs = range(shard["seq_lo"], shard["seq_hi"])
    parts = []
    for b in seqs:
        qw, k, v = prefill_inputs_fast(sh1, seed=seed + 7919 * b, device=dev)
        parts.append((qw[:, :, h0 * G:h1 * G].contiguous(), k[:, :, h0:h1].contiguous(), v[:, :, h0:h1].contiguous()))
        del qw, k, v
    prompt = tuple(torch.cat([p[i] for p in parts]) for i in range(3))
    del parts
    pool = []
    for s in range(min(n_steps, POOL)):
        st = [decode_inputs_fast(sh1, s, seed=seed + 7919 * b, device=dev) for b in seqs]
        pool.append((torch.cat([x[0] for x in st])[:, :, h0 * G:h1 * G].contiguous(),
                     torch.cat([x[1] for x in st])[:, :, h0:h1].contiguous(),
                     torch.cat([x[2] for x in st])[:, :, h0:h1].contiguous()))
    return prompt, pool


class Run:
    """One rank's shard of the workload: fresh caches from the same resident prompt."""

    def __init__(self, args, wl, shard, dev, group):
        from paper_2603_08727_b200 import arkv as A
        self.A, self.args, self.wl, self.shard, self.dev, self.group = A, args, wl, shard, dev, group
        self.B = shard["seq_hi"] - shard["seq_lo"]
        self.Hkv = shard["kvh_hi"] - shard["kvh_lo"]
        G = wl["n_q_heads"] // wl["n_kv_heads"]
        self.Hq = G * self.Hkv
        self.total_steps = args.warmup + args.steps
        budget = wl["budget"]
        P = wl["prompt_len"]
        if args.mode == "base":            # Base: no cache limit -> every token stays bf16
            budget = P + self.total_steps + 2 * wl["window"] + 1
        self.budget = budget
        self.cfg = A.make_config(wl["n_layers"], self.Hq, self.Hkv, wl["head_dim"], batch=self.B,
                                 window=wl["window"], budget_tokens=budget, quant_bits=wl["bits"],
                                 group_size=wl["group"], max_positions=P + self.total_steps + 1,
                                 quant_mode={"asym": A.QUANT_ASYM, "fp8": A.QUANT_FP8}[wl["qmode"]],
                                 state_sharing=1 if args.sharing == "layer" else 0, smooth=args.smooth,
                                 max_prompt=P, decode_kernel=args.kernel)
        self.rho_override = None
        if args.mode == "origin":          # Base_origin: budgeted heavy hitters, all bf16
            self.rho_override = [[1.0] * wl["n_layers"] for _ in range(self.B)]
        elif args.mode == "quant":         # Base_quant: every kept eligible token quantized
            self.rho_override = [[0.0] * wl["n_layers"] for _ in range(self.B)]
        self.prompt, self.pool = shard_inputs(wl, shard, 1234, dev, self.total_steps)
        self.prefill_ms = []

    def inputs(self, s):
        return self.pool[s % len(self.pool)]

    def fresh(self):
        """A new cache after the prompt: P1 (begin) -> C1 all-reduce -> P2-P4 (finish)."""
        import torch
        import torch.distributed as dist
        cache = self.A.ArkvCache(self.cfg, self.dev)
        qw, k, v = self.prompt
        colsum = torch.zeros(self.B, self.wl["n_layers"], self.cfg.max_positions, dtype=torch.float64,
                             device=self.dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        cache.arkv_prefill_begin(qw, k, colsum=colsum)
        ev[1].record()
        if self.group is not None:
            dist.all_reduce(colsum, op=dist.ReduceOp.SUM, group=self.group)
        ev[2].record()
        stats, oq, rho = cache.arkv_prefill_finish(k, v, colsum, rho_override=self.rho_override)
        ev[3].record()
        cache.arkv_check()
        self.prefill_ms.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])))
        self.rho = rho
        return cache

    def warm(self, cache, out):
        for s in range(self.args.warmup):
            q, k, v = self.inputs(s)
            cache.arkv_decode_step(q, k, v, out=out)


def barrier(ws):
    import torch.distributed as dist
    if ws > 1:
        dist.barrier()


def max_over_ranks(x, ws, dev):
    import torch
    import torch.distributed as dist
    if ws == 1:
        return x
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_arkv(args, wl):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2603_08727_b200.parallel import sequence_group, shard_units

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL init log (transport, NVLS) on stderr
        dist.init_process_group("nccl", device_id=dev)
    Bg, Hkv_g, L, d = wl["batch"], wl["n_kv_heads"], wl["n_layers"], wl["head_dim"]
    shard = shard_units(Bg, Hkv_g, ws, rank)
    if args.emulate_shard and ws == 1:
        # one GPU runs rank 0's shard of an N-GPU partition: its step time predicts the N-GPU
        # step (the decode loop has no collective); value = the global batch's tokens/s then
        shard = shard_units(Bg, Hkv_g, args.emulate_shard, 0)
    group = sequence_group(Bg, ws, rank) if ws > 1 else None   # C1: the ranks sharing a sequence
    run = Run(args, wl, shard, dev, group)
    K, Wm = args.steps, args.warmup
    out = torch.empty(run.B, L, run.Hq, d, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    # first-launch costs of every kernel on a throwaway cache
    c = run.fresh()
    run.warm(c, out)
    del c
    run.prefill_ms.clear()
    torch.cuda.synchronize()

    # ---- device-timed windows (fresh cache each, same steps; median over repeats) ----
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ms_runs, launches, step_bytes = [], 0, 0.0
    for r in range(args.repeats):
        cache = run.fresh()
        run.warm(cache, out)
        cache.arkv_check()
        _, n0, b0 = cache.arkv_profile_read(1)
        l0 = cache.arkv_launch_count()
        barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(Wm, Wm + K):
            q, k, v = run.inputs(s)
            cache.arkv_decode_step(q, k, v, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        ms_runs.append(max_over_ranks(e0.elapsed_time(e1), ws, dev))
        _, n1, b1 = cache.arkv_profile_read(1)
        launches = cache.arkv_launch_count() - l0
        step_bytes = (b1 - b0) / (n1 - n0)
        if r == 0:
            n_o1, n_q1, pos1 = unit_counts(cache, run)
            sched_tailors = count_tailors(run, cache)
        cache.arkv_check()
        del cache
    clocks = clk.stop()
    ms = statistics.median(ms_runs)

    # ---- kernel window: CUDA event pairs around every decode-kernel launch ----
    Kk = min(K, 512)
    cache = run.fresh()
    run.warm(cache, out)
    cache.arkv_profile(True)
    for s in range(Wm, Wm + Kk):
        q, k, v = run.inputs(s)
        cache.arkv_decode_step(q, k, v, out=out)
    torch.cuda.synchronize()
    k_ms, k_cnt, k_by = cache.arkv_profile_read(0)
    cache.arkv_profile(False)
    cache.arkv_check()
    kind = cache_kernel(cache)
    arena = cache.arena_bytes
    del cache

    # ---- e2e: the same steps through host buffers (pinned), pipelined like a serving loop;
    # median of up to 3 fresh-cache windows ----
    e2e = None
    if not args.no_e2e:
        runs = [run_e2e(run, K, Wm, ws, dev) for _ in range(min(3, args.repeats))]
        e2e = sorted(runs, key=lambda r: r["value"])[len(runs) // 2]
        e2e["runs"] = [r["value"] for r in runs]

    # ---- per-layer calls captured in one CUDA graph (H3) ----
    graph = None if args.no_graph else run_graph(run, min(K, args.graph_steps), Wm, ws, dev)

    # ---- C2: all-gather of the last step's outputs; per-rank rho ----
    c2 = None
    rho_all = run.rho.reshape(-1)
    if ws > 1:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gathered = [torch.empty_like(out) for _ in range(ws)]
        dist.all_gather(gathered, out)
        torch.cuda.synchronize()
        c2 = {"bytes_per_rank": out.numel() * out.element_size(), "ms": (time.perf_counter() - t0) * 1e3,
              "what": "all_gather of the last step's [B_local, L, H_q_local, d] outputs after the timed region"}
        rr = torch.tensor(rho_all, device=dev, dtype=torch.float64)
        gl = [torch.empty_like(rr) for _ in range(ws)]
        dist.all_gather(gl, rr)
        rho_all = torch.cat(gl).cpu().numpy()

    peak, peak_src = peaks()
    read_ceiling = read_ceiling_gbs(dev) if not args.no_ceiling else None
    value = Bg * K / (ms / 1e3)
    kernel_ms = k_ms / max(k_cnt, 1)
    achieved = (k_by / max(k_cnt, 1)) / (kernel_ms / 1e3) / 1e9 if k_cnt else None
    tp = traffic_record(args, kind, "hh_window" if args.warmup + K <= wl["window"] else "steady")
    pf = np.median(np.array(run.prefill_ms), axis=0)
    P = wl["prompt_len"]
    k_pass_bytes = 2.0 * run.B * L * run.Hkv * P * d * 2  # K read once per pass (P1 algorithmic bytes)
    budget_tokens = run.B * L * run.Hkv * run.budget
    evicted = float((pos1 - n_o1 - n_q1).sum())
    per = f"{run.B} seq x {run.Hkv} KV heads per GPU"
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "tokens/s",
        "n_gpus": ws,
        "steps": K,
        "warmup": Wm,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16+int4 (fp32 accumulate)" if wl["qmode"] == "asym" else "bf16+fp8e4m3 (fp32 accumulate)",
        "data": "synthetic (synth/ natural recipe: sinks, 5% log-normal heavy hitters, recency bump, x8 outlier V channels)",
        "config": {"workload": f"{args.workload} (BASELINE.json configs[{wl['baseline_cfg']}])",
                   "layers": L, "q_heads": wl["n_q_heads"], "kv_heads": Hkv_g, "head_dim": d,
                   "global_batch": Bg, "seq_len": P, "prompt_len": P, "budget_tokens": run.budget,
                   "window": wl["window"], "mode": args.mode, "state_sharing": args.sharing, "smooth": args.smooth,
                   "quant": (f"int{wl['bits']} g{wl['group']} asym" if wl["qmode"] == "asym"
                             else f"fp8 e4m3 g{wl['group']}"), "alpha": 0.75,
                   "launch": "one arkv_decode_step per step covering all layers (layer-batched)",
                   "decode_kernel": kind,
                   "parallelism": f"batch x kv-head ({per}; C1 colsum all-reduce at prefill when a sequence spans "
                                  f"GPUs, no collective in the decode loop, C2 output all-gather after timing)",
                   "l2": "no flush: cache arena %.2f GB per GPU >> 126 MB L2" % (arena / 1e9),
                   "timed_window": f"decode steps {Wm}..{Wm + K - 1} after the prompt; every window below covers "
                                   f"these steps on a fresh cache",
                   "repeats": args.repeats, "ms_per_step_runs": [m / K for m in ms_runs],
                   "arkv_env": arkv_env(),
                   "library": os.environ.get("ARKV_LIBRARY", "paper_2603_08727_b200/libarkv.so"),
                   "emulated_shard_of": args.emulate_shard or None},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": tp.get("dram_bytes_per_launch") if tp else None,
                     "traffic_source": tp.get("source") if tp else None,
                     "kernel": "decode attention kernel (%s)" % kind, "kernel_ms_per_launch": kernel_ms,
                     "alg_bytes_per_launch": k_by / max(k_cnt, 1), "peak_source": peak_src,
                     "timing": f"CUDA event pairs around each of {k_cnt} decode-kernel launches on the launching "
                               f"stream, steps {Wm}..{Wm + Kk - 1} on a fresh cache (event records between PDL "
                               f"launches would slow the device-timed window)"},
        "step_hbm": {"alg_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms / K / 1e3) / 1e9,
                     "frac_of_peak": step_bytes / (ms / K / 1e3) / 1e9 / peak,
                     "frac_of_8tbs_nominal": step_bytes / (ms / K / 1e3) / 1e12 / 8.0,
                     "bytes": "library count over the timed steps (arkv_profile_read(1): attention + HH "
                              "accumulator traffic + tailors), per GPU"},
        "read_ceiling": {"gbs": read_ceiling, "how": "best of torch amax/sum over a 2 GiB bf16 tensor (reference only)"},
        "gpu_launches": int(launches),
        "tailors_in_timed_region": int(sched_tailors),
        "memory": {"arena_bytes": arena, "dense_bf16_bytes": run.B * L * run.Hkv * (P + run.total_steps) * 4 * d,
                   "quant_ratio": float(n_q1.sum() * run.Hkv / budget_tokens),
                   "evict_ratio": evicted / float(pos1.sum()),
                   "n_o_range": [int(n_o1.min()), int(n_o1.max())], "n_q_range": [int(n_q1.min()), int(n_q1.max())]},
        "rho": {"min": float(rho_all.min()), "median": float(statistics.median(rho_all.tolist())),
                "max": float(rho_all.max())},
        "prefill": {"stats_ms": float(pf[0]), "c1_ms": float(pf[1]), "finish_ms": float(pf[2]),
                    "stats_alg_bytes": k_pass_bytes,
                    "stats_gbs": k_pass_bytes / (pf[0] / 1e3) / 1e9,
                    "stats_frac": k_pass_bytes / (pf[0] / 1e3) / 1e9 / peak,
                    "kernel": "prefill_ws_kernel (P1: tcgen05 + TMA, two passes over K) + column sums",
                    "timing": f"CUDA events around arkv_prefill_begin / C1 / arkv_prefill_finish, median of "
                              f"{len(run.prefill_ms)} prefills (first-launch costs taken by a throwaway cache)"},
        "clocks": clocks,
        "e2e": e2e,
        "per_layer_graph": graph,
        "c2": c2,
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, run.rho[0], samples=args.cpu_steps)
    if ws > 1:
        dist.destroy_process_group()
    return line, rank


def unit_counts(cache, run):
    import numpy as np
    B, L = run.B, run.wl["n_layers"]
    n_o = np.zeros((B, L), np.int64)
    n_q = np.zeros((B, L), np.int64)
    pos = np.zeros((B, L), np.int64)
    for b in range(B):
        for l in range(L):
            n_o[b, l], n_q[b, l], pos[b, l], _ = cache.arkv_unit_counts(b, l)
    return n_o, n_q, pos


def count_tailors(run, cache):
    A, P, Wm, K = run.A, run.wl["prompt_len"], run.args.warmup, run.args.steps
    n = 0
    for b in range(run.B):
        for l in range(run.wl["n_layers"]):
            for e in A.arkv_schedule(run.cfg, P, float(run.rho[b, l]), Wm + K):
                n += Wm <= e[0] < Wm + K
    return n * run.Hkv


def run_e2e(run, K, Wm, ws, dev):
    """The public API with host buffers: every step copies that step's q/k/v host->device
    from pinned memory and its output device->host.  H2D of step s+1 and D2H of step s
    overlap step s (two copy streams)."""
    import torch
    cache = run.fresh()
    out0 = torch.empty(run.B, run.wl["n_layers"], run.Hq, run.wl["head_dim"], dtype=torch.bfloat16, device=dev)
    run.warm(cache, out0)
    stream = torch.cuda.current_stream()
    n_host = min(16, len(run.pool))
    hq = [[t.cpu().pin_memory() for t in run.inputs(Wm + i)] for i in range(n_host)]
    dq = [[torch.empty_like(t) for t in run.pool[0]] for _ in range(2)]
    hout = [torch.empty(out0.shape, dtype=out0.dtype, pin_memory=True) for _ in range(2)]
    outs = [torch.empty_like(out0) for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    computed = [torch.cuda.Event() for _ in range(2)]
    drained = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    barrier(ws)
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
    for s in range(K):
        b2 = s % 2
        if s + 1 < K:
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
    stream.wait_event(drained[(K - 1) % 2])
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1), ws, dev)
    cache.arkv_check()
    del cache
    return {"value": run.wl["batch"] * K / (e2e_ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in hq[0])),
            "d2h_bytes_per_step": int(hout[0].numel() * hout[0].element_size()),
            "pipeline": "H2D of step s+1 and D2H of step s overlap step s's compute (two copy streams); "
                        "inputs cycle through %d pinned host steps" % n_host,
            "window": f"decode steps {Wm}..{Wm + K - 1} (the device-timed steps) on a fresh cache"}


def run_graph(run, Kg, Wm, ws, dev):
    """H3: one arkv_decode_step per LAYER (a model's per-layer attention call), the Kg
    steps x L calls captured into one CUDA graph and replayed once.  The host schedule
    is data-independent, so the captured launches are exactly the eager ones."""
    import torch
    L = run.wl["n_layers"]
    cache = run.fresh()
    out = torch.empty(run.B, L, run.Hq, run.wl["head_dim"], dtype=torch.bfloat16, device=dev)
    run.warm(cache, out)
    # per-layer views of the inputs: [B][1][H][d] slices are not contiguous for B > 1
    steps = []
    for s in range(Wm, Wm + Kg):
        q, k, v = run.inputs(s)
        steps.append([(q[:, l:l + 1].contiguous(), k[:, l:l + 1].contiguous(), v[:, l:l + 1].contiguous(),
                       torch.empty(run.B, 1, run.Hq, run.wl["head_dim"], dtype=torch.bfloat16, device=dev))
                      for l in range(L)])
    torch.cuda.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
            for s in range(Kg):
                for l in range(L):
                    q, k, v, o = steps[s][l]
                    cache.arkv_decode_step(q, k, v, layer0=l, out=o, stream=side)
        torch.cuda.synchronize()
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(e0.elapsed_time(e1), ws, dev)
        cache.arkv_check()
        res = {"value": run.wl["batch"] * Kg / (ms / 1e3), "unit": "tokens/s", "ms_per_step": ms / Kg,
               "steps": Kg, "calls_per_step": L,
               "how": f"steps {Wm}..{Wm + Kg - 1}: one arkv_decode_step(layer0=l, n_layers=1) per layer, all "
                      f"{Kg * L} calls captured into one CUDA graph, replayed once (CUDA events)"}
    except Exception as ex:  # reported, not fatal: the layer-batched window is the headline
        res = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    del cache
    return res


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
    return {0: "generic", 1: "split-K (chunked pipeline, cost-balanced LPT splits)", 2: "persistent",
            3: "auto (split-K chunked pipeline with cost-balanced LPT splits; persistent at >= 32 units per SM)"}[
        A.lib().arkv_cache_info(cache.handle, 1)]


def traffic_record(args, kind, window):
    """ncu DRAM bytes per launch of the decode kernel (profiles/ncu_traffic.json), with the
    capture it came from; the library cannot read DRAM counters in-process.  window:
    "hh_window" when the timed steps all lie in the first heavy-hitter window after the prompt
    (caches at their fullest, logit stores), else "steady"."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if args.mode != "arkv" or not os.path.exists(tp):
        return None
    try:
        rec = json.load(open(tp)).get(args.workload, {}).get(kind)
        if isinstance(rec, dict) and window in rec:
            rec = rec[window]
        return rec if isinstance(rec, dict) and "dram_bytes_per_launch" in rec else None
    except Exception:
        return None


def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [os.cpu_count() or 1])
    except Exception:
        return os.cpu_count() or 1


def _oracle_slice(wl, rho_seq):
    """The oracle on one layer (median rho) x all KV heads of one sequence after the
    prompt, advanced untimed to 8 steps before the first decode tailor (R12, R14)."""
    import numpy as np
    import oracle as O
    from synth import Shape, decode_inputs_fast, prefill_inputs_fast
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
    # first decode tailor of this unit (data-independent schedule, oracle's own rule)
    dec = [e for e in O.schedule(P, 4096, r, cfg) if e[0] >= 0]
    t_first = dec[0][0] if dec else 8
    s0 = max(0, t_first - 7)
    step_in = lambda s: [f(x[:, li:li + 1]) for x in decode_inputs_fast(sh1, s, seed=1234, device="cpu")]  # noqa: E731
    for s in range(s0):
        ora.decode_step(*step_in(s))
    return ora, step_in, s0, li, r


def cpu_baseline(wl, rho_seq, samples=8):
    """The float64 oracle as it stands: one layer x all KV heads, `samples` decode steps
    that end with the unit's first decode tailor, timed with all BLAS threads and again
    single-threaded (threadpoolctl); tokens/s extrapolated to all L layers."""
    from threadpoolctl import threadpool_limits
    ora, step_in, s0, li, r = _oracle_slice(wl, rho_seq)
    ora1 = copy.deepcopy(ora)
    inputs = [step_in(s) for s in range(s0, s0 + samples)]

    def timed(o):
        t0 = time.perf_counter()
        for x in inputs:
            o.decode_step(*x)
        return (time.perf_counter() - t0) / samples

    threads = _oracle_threads()
    per_all = timed(ora)
    with threadpool_limits(limits=1):
        per_one = timed(ora1)
    L = wl["n_layers"]
    sample = (f"layer {li} (rho={r:.3f}) x {wl['n_kv_heads']} KV heads, decode steps {s0}..{s0 + samples - 1} "
              f"(the last one runs the unit's first decode tailor) after a {wl['prompt_len']}-token prompt; float64 "
              f"numpy; tokens/s extrapolated to {L} layers")
    return {"value": wl["batch"] / (per_all * L), "unit": "tokens/s", "cores": int(threads), "kind": "oracle",
            "sample": sample, "extrapolated": True,
            "single_thread": {"value": wl["batch"] / (per_one * L), "cores": 1}}


def run_reference(args, wl):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only).  A step is one
    decode step of one layer x all KV heads of one sequence (a bounded sample); tokens/s
    is extrapolated to the workload (L layers, whole batch)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return None, rank
    rho_seq = [0.2 + 0.8 * l / max(wl["n_layers"] - 1, 1) for l in range(wl["n_layers"])]
    ora, step_in, s0, li, r = _oracle_slice(wl, rho_seq)
    for s in range(s0, s0 + args.warmup):
        ora.decode_step(*step_in(s))
    inputs = [step_in(s) for s in range(s0 + args.warmup, s0 + args.warmup + args.steps)]
    t0 = time.perf_counter()
    for x in inputs:
        ora.decode_step(*x)
    el = time.perf_counter() - t0
    per_sample = el / args.steps
    L = wl["n_layers"]
    value = wl["batch"] / (per_sample * L)
    sample = (f"each step: one decode step of layer {li} of {L} (rho={r:.3f}) x {wl['n_kv_heads']} KV heads of one "
              f"sequence, float64 numpy oracle; tokens/s extrapolated x {L} layers x batch {wl['batch']}")
    threads = _oracle_threads()
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_sample * 1e3,
            "ms_per_step_note": "measured per sampled layer-step; a full step is x%d layers" % L,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{args.workload} (BASELINE.json configs[{wl['baseline_cfg']}])"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": int(threads), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}, 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--repeats", type=int, default=5, help="device-timed windows (fresh cache each); median")
    ap.add_argument("--impl", default="arkv", choices=["arkv", "reference"])
    ap.add_argument("--workload", default="llama3-8b-32k", choices=sorted(WORKLOADS))
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 generic, 2 fast split-K, 3 fast persistent")
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--graph-steps", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ceiling", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--emulate-shard", type=int, default=0,
                    help="measurement: on 1 GPU, run rank 0's shard of an N-GPU partition (its step time)")
    ap.add_argument("--allow-tuning-library", action="store_true",
                    help="measurement only: accept ARKV_LIBRARY (an A/B tuning build); the line says so")
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
    ws, rank, _ = dist_env()
    if args.impl == "arkv" and "ARKV_LIBRARY" in os.environ and not args.allow_tuning_library:
        # a measurement build (libarkv_tuning.so) is not the product: no bench line from it
        print(json.dumps({"error": "ARKV_LIBRARY is set: bench.py measures the product libarkv.so only",
                          "arkv_env": arkv_env()}), flush=True)
        sys.exit(2)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if ws != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    wl = dict(WORKLOADS[args.workload])
    if args.prompt_len:
        wl["prompt_len"] = args.prompt_len
    if args.layers:
        wl["n_layers"] = args.layers
    wl["qmode"] = "asym"
    if args.quant == "fp8":
        wl.update(bits=8, group=wl["head_dim"], qmode="fp8")
    if args.impl == "reference":
        args.steps = min(args.steps, 64)    # each step is a bounded CPU sample (one layer-step)
        args.warmup = min(args.warmup, 4)
        line, rank = run_reference(args, wl)
    else:
        line, rank = run_arkv(args, wl)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
