"""Diagnostic (tuning build only): per-CTA start/end times of the split-K decode kernel at
chosen decode steps (HH window and post-tailor) — wave shape, per-SM busy time, the tail,
and CTA time per byte by the unit's Quantized share.  Not a bench number.

    python -m paper_2603_08727_b200.build --tuning
    ARKV_LIBRARY=paper_2603_08727_b200/libarkv_tuning.so python scripts/cta_timeline.py --at 10 40
"""
import argparse
import ctypes
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
    ap.add_argument("--at", type=int, nargs="+", default=[10, 40])
    ap.add_argument("--mode", default="arkv")
    ap.add_argument("--dump", default=".")
    ap.add_argument("--per-layer", action="store_true",
                    help="one call per layer; the recorded call is layer L/2 of each --at step, also timed with events")
    args = ap.parse_args()
    wl = bench.WORKLOADS[args.workload]
    B, L, Hq, Hkv, d, P = (wl["batch"], wl["n_layers"], wl["n_q_heads"], wl["n_kv_heads"], wl["head_dim"],
                           wl["prompt_len"])
    steps = max(args.at) + 1
    dev = torch.device("cuda", 0)
    cfg = A.make_config(L, Hq, Hkv, d, batch=B, window=wl["window"], budget_tokens=wl["budget"],
                        quant_bits=wl["bits"], group_size=wl["group"], max_positions=P + steps + 1, max_prompt=P)
    cache = A.ArkvCache(cfg, dev)
    lib = A.lib()
    fn = lib.arkv_debug_cta_times
    fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    print("occupancy (blocks/SM): chunk kernel", lib.arkv_debug_occupancy(0), "ring kernel", lib.arkv_debug_occupancy(1))
    sh = Shape(batch=B, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=wl["window"])
    qw, k, v = prefill_inputs_fast(sh, seed=1234, device=dev)
    rho_ov = None
    if args.mode == "quant":
        rho_ov = [[0.0] * L for _ in range(B)]
    _, _, rho = cache.arkv_prefill_stats(qw, k, v, rho_override=rho_ov)
    del qw, k, v
    out = torch.empty(B, L, Hq, d, dtype=torch.bfloat16, device=dev)
    n_max = 16384
    buf = (ctypes.c_ulonglong * (8 * n_max))()
    for s in range(steps):
        q, kk, vv = decode_inputs_fast(sh, s, seed=1234, device=dev)
        rec = s in args.at
        if rec:
            torch.cuda.synchronize()
            fn(1, None, 0)
        if args.per_layer:
            lr = L // 2
            for l in range(L):
                ql, kl, vl = q[:, l:l + 1].contiguous(), kk[:, l:l + 1].contiguous(), vv[:, l:l + 1].contiguous()
                if rec and l == lr:
                    torch.cuda.synchronize()
                    fn(1, None, 0)
                    clr = lib.arkv_debug_cta_clear
                    clr()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    cache.arkv_decode_step(ql, kl, vl, layer0=l, out=out[:, l:l + 1])
                    e1.record()
                    torch.cuda.synchronize()
                    print(f"   layer call {l} at step {s}: {e0.elapsed_time(e1) * 1e3:.1f} us (events)")
                    fn(0, ctypes.cast(buf, ctypes.c_void_p), n_max)
                    break
                cache.arkv_decode_step(ql, kl, vl, layer0=l, out=out[:, l:l + 1].contiguous())
            if rec:
                for l in range(lr + 1, L):
                    ql, kl, vl = q[:, l:l + 1].contiguous(), kk[:, l:l + 1].contiguous(), vv[:, l:l + 1].contiguous()
                    cache.arkv_decode_step(ql, kl, vl, layer0=l, out=out[:, l:l + 1].contiguous())
        else:
            cache.arkv_decode_step(q, kk, vv, out=out)
        if rec:
            torch.cuda.synchronize()
            if not args.per_layer:
                fn(0, ctypes.cast(buf, ctypes.c_void_p), n_max)
            r = np.frombuffer(buf, dtype=np.uint64).reshape(n_max, 8).copy()
            fn(0, None, 0)
            valid = r[:, 1] > 0
            r = r[valid]
            t0 = r[:, 0].astype(np.int64)
            t1 = r[:, 1].astype(np.int64)
            base = t0.min()
            t0 -= base
            t1 -= base
            sm = (r[:, 2] >> np.uint64(32)).astype(np.int64)
            uid = (r[:, 2] & np.uint64(0xFFFFFFFF)).astype(np.int64)
            n_ot = (r[:, 3] >> np.uint64(32)).astype(np.int64)
            n_qt = (r[:, 3] & np.uint64(0xFFFFFFFF)).astype(np.int64)
            tf = r[:, 4].astype(np.int64) - base
            tw = r[:, 5:8].astype(np.int64) - base
            np.savez(os.path.join(args.dump, f"cta_step{s}.npz"), t0=t0, t1=t1, sm=sm, uid=uid, n_ot=n_ot, n_qt=n_qt,
                     tf=tf, tw=tw)
            print(f"   per CTA (us): fill (start -> first item) {np.mean(tf - t0) / 1e3:.2f}, warp finish spread "
                  f"(last - first warp) {np.mean(tw.max(1) - tw.min(1)) / 1e3:.2f}, merge (last warp -> end) "
                  f"{np.mean(t1 - tw.max(1)) / 1e3:.2f}, duration {np.mean(t1 - t0) / 1e3:.2f}")
            span = t1.max()
            dur = t1 - t0
            by = n_ot * 16384 + n_qt * 4608
            print(f"== step {s}: {len(r)} CTAs, kernel span {span / 1e3:.1f} us, "
                  f"bytes {by.sum() / 1e6:.1f} MB -> {by.sum() / span:.0f} GB/s over the span")
            if len(r) < 400:
                print(f"   CTA durations (us): min {dur.min() / 1e3:.1f} median {np.median(dur) / 1e3:.1f} max {dur.max() / 1e3:.1f}; "
                      f"fill mean {np.mean(r[:, 4].astype(np.int64) - base - t0) / 1e3:.1f}")
            busy = np.zeros(sm.max() + 1)
            last = np.zeros(sm.max() + 1)
            for i in range(len(r)):
                busy[sm[i]] += dur[i]
                last[sm[i]] = max(last[sm[i]], t1[i])
            print(f"   per-SM busy (CTA-time / 2 slots): mean {busy.mean() / 2e3:.1f} us, "
                  f"min {busy.min() / 2e3:.1f}, max {busy.max() / 2e3:.1f}; SM last end: "
                  f"min {last.min() / 1e3:.1f} us, median {np.median(last) / 1e3:.1f}")
            qshare = (n_qt * 4608) / np.maximum(by, 1)
            for lo, hi in [(0, 0.1), (0.1, 0.3), (0.3, 0.6), (0.6, 0.9), (0.9, 1.01)]:
                m = (qshare >= lo) & (qshare < hi) & (by > 0)
                if m.any():
                    print(f"   Q share [{lo:.1f},{hi:.1f}): {m.sum():4d} CTAs, mean dur {dur[m].mean() / 1e3:6.1f} us, "
                          f"mean bytes {by[m].mean() / 1e6:.2f} MB, {by[m].sum() / dur[m].sum():.0f} GB/s per CTA")
            # timeline: active CTAs over time
            ts = np.linspace(0, span, 21)
            act = [int(((t0 <= t) & (t1 > t)).sum()) for t in ts]
            print("   active CTAs at 5% steps:", act)
            starts = np.sort(t0)
            print(f"   CTA starts: 25% {starts[len(starts) // 4] / 1e3:.1f} us, 50% {starts[len(starts) // 2] / 1e3:.1f}, "
                  f"last {starts[-1] / 1e3:.1f}; ends: first {np.sort(t1)[0] / 1e3:.1f}")
    cache.arkv_check()


if __name__ == "__main__":
    main()
