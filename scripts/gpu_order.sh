#!/bin/bash
# A/B: item order of the split-K fast kernel (ARKV_ITEM_ORDER 0/1/2)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/order
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "mid_config and 2-4-128" > gpurun_out/order/t.log 2>&1; echo "t exit=$?"
ARKV_ITEM_ORDER=1 timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "mid_config and 2-4-128 or full_size" > gpurun_out/order/t1.log 2>&1; echo "t1 exit=$?"
for O in 0 1 2 0 1 2; do
  ARKV_ITEM_ORDER=$O timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/order/b$O.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/order/b$O.json')); print('order=$O', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
done
