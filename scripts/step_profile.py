"""Diagnostic: per-step device time of the first decode steps at a workload (HH window vs
steady state).  Each step is bracketed by CUDA events and, separately, the decode kernel's
own event pair (arkv_profile).  Not a bench number (events between steps stop PDL overlap).

    python scripts/step_profile.py [--workload llama3-8b-32k] [--steps 120]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_08727_b200 import arkv as A  # noqa: E402
from synth import Shape, decode_inputs_fast, prefill_inputs_fast  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama3-8b-32k")
    ap.add_argument("--steps", type=int, default=120)
    ap.add_argument("--rho", type=float, default=None, help="override every layer's rho (0: Base_quant-like)")
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    B, L, Hq, Hkv, d, P = (wl["batch"], wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"],
                           wl["prompt_len"])
    dev = torch.device("cuda", 0)
    cfg = A.make_config(L, Hq, Hkv, d, batch=B, window=wl["window"], budget_tokens=wl["budget"],
                        quant_bits=wl["bits"], group_size=wl["group"], max_positions=P + args.steps + 1, max_prompt=P)
    cache = A.ArkvCache(cfg, dev)
    sh = Shape(batch=B, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=wl["window"])
    qw, k, v = prefill_inputs_fast(sh, seed=1234, device=dev)
    ov = None if args.rho is None else [[args.rho] * L for _ in range(B)]
    _, _, rho = cache.arkv_prefill_stats(qw, k, v, rho_override=ov)
    del qw, k, v
    pool = [decode_inputs_fast(sh, s, seed=1234, device=dev) for s in range(args.steps)]
    out = torch.empty(B, L, Hq, d, dtype=torch.bfloat16, device=dev)
    sched = [A.arkv_schedule(cfg, P, float(rho[b, l]), args.steps) for b in range(B) for l in range(L)]
    tail = np.zeros(args.steps, int)
    for ev in sched:
        for e in ev:
            if e[0] < args.steps:
                tail[e[0]] += Hkv
    # warm-up of first-launch costs on a throwaway cache would change state; instead the
    # first 2 steps are reported but excluded from the summaries
    step_ms, kern_ms = [], []
    for s in range(args.steps):
        q, kk, vv = pool[s]
        cache.arkv_profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cache.arkv_decode_step(q, kk, vv, out=out)
        e1.record()
        torch.cuda.synchronize()
        km, kc, _ = cache.arkv_profile_read(0)
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(km)
    cache.arkv_profile(False)
    cache.arkv_check()
    W = wl["window"]
    for s in range(args.steps):
        print(f"step {s:4d} tailored_units {tail[s]:4d} step_ms {step_ms[s]:.4f} decode_kernel_ms {kern_ms[s]:.4f}")
    first_tailor = int(np.nonzero(tail)[0][0]) if tail.any() else args.steps
    hh = [i for i in range(2, min(first_tailor, args.steps))]
    post = [i for i in range(first_tailor + 1, args.steps) if tail[i] == 0]
    f = lambda xs, arr: float(np.median([arr[i] for i in xs])) if xs else float("nan")  # noqa: E731
    print(f"first decode tailor at step {first_tailor}; window W={W}")
    print(f"HH-window steps (2..{first_tailor - 1}): step {f(hh, step_ms):.4f} ms, kernel {f(hh, kern_ms):.4f} ms")
    print(f"post-tailor steps w/o tailor: step {f(post, step_ms):.4f} ms, kernel {f(post, kern_ms):.4f} ms")


if __name__ == "__main__":
    main()
