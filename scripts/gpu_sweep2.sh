#!/bin/bash
# Split count and pipeline shape sweep of the split-K fast kernel at configs[1]
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/sw2
for S in 2 3 4 5; do
  ARKV_SPLITS=$S timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/sw2/s$S.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw2/s$S.json')); print('S=$S', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
for C in 4,2 6,2 4,3 8,1; do
  ARKV_FAST_CFG=$C timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/sw2/c$C.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw2/c$C.json')); print('cfg=$C', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
