#!/bin/bash
# Step-time shares: bench with HH accumulation / combine launches skipped (timing only)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/skip
for SK in 0 2 5 7; do
  ARKV_TIMING_SKIP=$SK timeout 300 python bench.py --kernel 2 --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/skip/b$SK.json 2>gpurun_out/skip/b$SK.err
  python -c "
import json; d=json.load(open('gpurun_out/skip/b$SK.json')); print('skip=$SK', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])" || tail -2 gpurun_out/skip/b$SK.err
done
for M in origin quant; do for K in 2 3; do
  timeout 300 python bench.py --kernel $K --mode $M --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/skip/m$M$K.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/skip/m$M$K.json')); print('mode=$M kernel=$K', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])"
done; done
