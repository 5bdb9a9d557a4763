#!/bin/bash
# Step-time breakdown: bench with/without the kernel event pairs, and ncu launch lists
# for the split-K (2) and persistent (3) decode kernels (run under gpurun).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/bd
for K in 2 3; do
  for EV in "" "--no-kernel-events"; do
    timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 $EV > gpurun_out/bd/b$K$EV.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/bd/b$K$EV.json')); print('kernel=$K $EV', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'])"
  done
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/bd/launches_k$K.csv \
     python bench.py --kernel $K --steps 60 --warmup 4 --no-cpu-baseline --e2e-steps 0 --no-ceiling > /dev/null 2>&1
  echo "ncu k$K exit=$?"
done
