#!/bin/bash
# Pipeline shapes of the split-K decode kernel (ARKV_FAST_CFG=C,SPW) in ARKV and Base_quant modes
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/cfg
for CF in 4,1 3,2 2,2 2,3 4,1; do for M in arkv quant; do
  ARKV_FAST_CFG=$CF timeout 300 python bench.py --mode $M --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/cfg/$M.json 2>gpurun_out/cfg/err
  python -c "
import json; d=json.load(open('gpurun_out/cfg/$M.json')); print('cfg=$CF $M', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 gpurun_out/cfg/err
done; done
