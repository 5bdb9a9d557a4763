#!/bin/bash
# Step-time shares: bench with tailor / HH accumulation launches skipped (timing only)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/skip
for K in 2 3; do for SK in 0 1 2 3; do
  ARKV_TIMING_SKIP=$SK timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/skip/b$K$SK.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/skip/b$K$SK.json')); print('kernel=$K skip=$SK', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done; done
