"""Diagnostic: per-layer output error vs the oracle on lattice / natural inputs for the
three decode kernels (generic, split-K (+cluster HH), persistent) and both quant formats."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from paper_2603_08727_b200 import arkv as A
from synth import (Shape, prefill_inputs_lattice, decode_inputs_lattice, prefill_inputs_fast, decode_inputs_fast)

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
Hq, Hkv = (32, 8) if P > 4096 else (8, 2)
BUD = P // 4
KERNELS = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 3]
QUANTS = sys.argv[4].split(",") if len(sys.argv) > 4 else ["asym", "fp8"]
sh = Shape(batch=1, n_layers=4, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=128, prompt_len=P, window=32)
for recipe in ("lattice", "natural"):
    pf = prefill_inputs_lattice if recipe == "lattice" else prefill_inputs_fast
    df = decode_inputs_lattice if recipe == "lattice" else decode_inputs_fast
    for quant in QUANTS:
        for kernel in KERNELS:
            bits = 8 if quant == "fp8" else 4
            cfg = A.make_config(4, Hq, Hkv, 128, budget_tokens=BUD, max_positions=P + steps + 1, max_prompt=P,
                                decode_kernel=kernel, quant_bits=bits,
                                quant_mode=A.QUANT_FP8 if quant == "fp8" else A.QUANT_ASYM)
            gpu = A.ArkvCache(cfg)
            qw, k, v = pf(sh, seed=3, device="cuda")
            _, _, rho = gpu.arkv_prefill_stats(qw, k, v)
            ocfg = O.Cfg(n_layers=4, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=128, window=32, budget_tokens=BUD,
                         quant_bits=bits, quant_mode=quant)
            ora = O.OracleARKV(ocfg)
            f = lambda t: t.double().cpu().numpy()  # noqa: E731
            ora.prefill(f(qw), f(k), f(v), rho_override=rho)
            errs = np.zeros((steps, 4))
            for s in range(steps):
                q, kn, vn = df(sh, s, seed=3, device="cuda")
                out = gpu.arkv_decode_step(q, kn, vn, out_fp32=True).double().cpu().numpy()
                ref = ora.decode_step(f(q), f(kn), f(vn))
                for l in range(4):
                    errs[s, l] = np.abs(out[:, l] - ref[:, l]).max()
            gpu.arkv_check()
            st = [ (gpu.arkv_export_unit(0, l, 0)["state"] == ora.export(0, l, 0)["state"]).all() for l in range(4)]
            print(f"{recipe:8s} {quant:5s} kernel {kernel}: rho {np.round(rho[0], 3)} max|err| per layer "
                  f"{np.round(errs.max(0), 5)} states_equal {st}", flush=True)
