#!/bin/bash
# GPU test suite + A/B bench of the two fast kernels at configs[1] (run under gpurun)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/chk
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/chk/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -2 gpurun_out/chk/gpu_tests.log
for K in 2 3; do
  timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/chk/b$K.json 2>gpurun_out/chk/b$K.err
  python -c "
import json; d=json.load(open('gpurun_out/chk/b$K.json')); print('kernel=$K', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/chk/b$K.err
done
for M in quant; do for K in 2 3; do
  timeout 300 python bench.py --kernel $K --mode $M --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/chk/m$M$K.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/chk/m$M$K.json')); print('mode=$M kernel=$K', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])"
done; done
