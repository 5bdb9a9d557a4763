#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/ab3
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "persistent or gqa" > gpurun_out/ab3/t.log 2>&1; echo "t exit=$?"; tail -1 gpurun_out/ab3/t.log
for O in 1 1; do
  ARKV_ITEM_ORDER=$O timeout 300 python bench.py --kernel 3 --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/ab3/b$O.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab3/b$O.json')); print('k3 order=$O', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
