#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/ab4
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/ab4/t.log 2>&1; echo "t exit=$?"; tail -1 gpurun_out/ab4/t.log
for K in 2 3 2 3; do
  timeout 300 python bench.py --kernel $K --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/ab4/b$K.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab4/b$K.json')); print('k=$K', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
