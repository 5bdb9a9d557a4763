#!/bin/bash
# Step anatomy at configs[1]: ncu launch list of the bench command + timing with parts skipped
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/bd
for SK in 0 1 2 4 7; do
  ARKV_TIMING_SKIP=$SK timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/bd/s$SK.json 2>gpurun_out/bd/s$SK.err
  python -c "
import json; d=json.load(open('gpurun_out/bd/s$SK.json')); print('skip=$SK', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'launches', d['gpu_launches'])" || tail -2 gpurun_out/bd/s$SK.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv \
   --log-file gpurun_out/bd/launches.csv python bench.py --steps 1024 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1
echo "ncu exit=$?"
