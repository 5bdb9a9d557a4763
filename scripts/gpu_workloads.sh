#!/bin/bash
# Both fast kernels on every bench workload (run under gpurun)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/wl
for W in qwen3-8b-8k-b8 llama3-8b-1k-b64 llama3-8b-128k; do for K in 2 3; do
  timeout 600 python bench.py --workload $W --kernel $K --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/wl/$W-$K.json 2>gpurun_out/wl/$W-$K.err
  python -c "
import json; d=json.load(open('gpurun_out/wl/$W-$K.json')); print('$W k=$K', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/wl/$W-$K.err
done; done
