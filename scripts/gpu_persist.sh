#!/bin/bash
# Persistent decode kernel: parity tests, then A/B against the split-K kernel (run under gpurun).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/persist
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "persistent or gqa_groups or batch_and_spare or mid_config" \
  > gpurun_out/persist/tests.log 2>&1
echo "tests exit=$?"; tail -3 gpurun_out/persist/tests.log
for K in 2 3; do for rep in 1 2; do
  timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/persist/b$K$rep.json 2>gpurun_out/persist/b$K$rep.err
  python -c "
import json; d=json.load(open('gpurun_out/persist/b$K$rep.json')); print('kernel=$K', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" || tail -5 gpurun_out/persist/b$K$rep.err
done; done
