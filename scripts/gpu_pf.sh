#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/pfx
for P in 0 2 4 8 0 4; do
  ARKV_PREFETCH=$P timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/pfx/b$P.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pfx/b$P.json')); print('prefetch=$P', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
