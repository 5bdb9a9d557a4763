#!/bin/bash
# A/B of the two fast decode kernels at configs[1] (run under gpurun)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/ab
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "persistent or gqa_groups or mid_config and 2-4" > gpurun_out/ab/tests.log 2>&1
echo "tests exit=$?"; tail -1 gpurun_out/ab/tests.log
for K in 2 3; do
  timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab/b$K.json 2>gpurun_out/ab/b$K.err
  python -c "
import json; d=json.load(open('gpurun_out/ab/b$K.json')); print('kernel=$K', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" || tail -3 gpurun_out/ab/b$K.err
done
