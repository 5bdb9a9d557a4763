#!/bin/bash
# spin combine (per-unit split flags instead of a grid-wide wait): GPU tests + A/B bench
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/spin; mkdir -p $O
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "toy or mid_config or smoothed or cuda_graph or full_size_configs1" > $O/t.log 2>&1; echo "tests exit=$?"; tail -1 $O/t.log
for R in 1 2; do for S in 1 0; do
  ARKV_SPIN_COMBINE=$S timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('spin=$S tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel=%.4f'%d['roofline']['kernel_ms_per_launch'])" || tail -2 $O/b.err
done; done
