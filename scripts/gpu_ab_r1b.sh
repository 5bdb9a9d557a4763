#!/bin/bash
# GPU tests + A/B of the fused HH combine (ARKV_FUSE_HH) at configs[1]
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/ab/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 gpurun_out/ab/gpu_tests.log
for F in 1 0 1; do
  ARKV_FUSE_HH=$F timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/ab/f$F.json 2>gpurun_out/ab/f$F.err
  python -c "
import json; d=json.load(open('gpurun_out/ab/f$F.json')); print('fuse_hh=$F', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'], 'launches', d['gpu_launches'])" || tail -2 gpurun_out/ab/f$F.err
done
