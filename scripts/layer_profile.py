"""Diagnostic: per-layer decode calls (a model's attention call per layer) — decode-kernel
time per call (library event pairs) vs the whole call, eager launches.  Not a bench number."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2603_08727_b200 import arkv as A  # noqa: E402
from synth import Shape, decode_inputs_fast, prefill_inputs_fast  # noqa: E402

wl = bench.WORKLOADS["llama3-8b-32k"]
B, L, Hq, Hkv, d, P = 1, 32, 32, 8, 128, 32768
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 80
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda", 0)
cfg = A.make_config(L, Hq, Hkv, d, budget_tokens=8192, max_positions=P + steps + 1, max_prompt=P, decode_kernel=kernel)
cache = A.ArkvCache(cfg, dev)
sh = Shape(batch=1, n_layers=L, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d, prompt_len=P, window=32)
qw, k, v = prefill_inputs_fast(sh, seed=1234, device=dev)
cache.arkv_prefill_stats(qw, k, v)
del qw, k, v
pool = []
for s in range(steps):
    q, kk, vv = decode_inputs_fast(sh, s, seed=1234, device=dev)
    pool.append([(q[:, l:l + 1].contiguous(), kk[:, l:l + 1].contiguous(), vv[:, l:l + 1].contiguous()) for l in range(L)])
out = torch.empty(1, 1, Hq, d, dtype=torch.bfloat16, device=dev)
call_ms, kern_ms = [], []
for s in range(steps):
    cache.arkv_profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L):
        q, kk, vv = pool[s][l]
        cache.arkv_decode_step(q, kk, vv, layer0=l, out=out)
    e1.record()
    torch.cuda.synchronize()
    km, kc, _ = cache.arkv_profile_read(0)
    call_ms.append(e0.elapsed_time(e1) / L)
    kern_ms.append(km / max(kc, 1))
cache.arkv_check()
hh = slice(2, 30)
post = slice(40, steps)
print(f"per-layer call (eager, event pairs around every decode kernel): HH steps call {np.median(call_ms[hh]) * 1e3:.1f} us "
      f"kernel {np.median(kern_ms[hh]) * 1e3:.1f} us; later steps call {np.median(call_ms[post]) * 1e3:.1f} us "
      f"kernel {np.median(kern_ms[post]) * 1e3:.1f} us")
