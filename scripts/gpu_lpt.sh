#!/bin/bash
# split-K launch order: layers largest first (ARKV_LPT=1, default) vs layer order
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/lpt; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/t.log 2>&1; echo "tests exit=$?"; tail -1 $O/t.log
for R in 1 2; do for L in 1 0; do
  ARKV_LPT=$L timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('lpt=$L tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 $O/b.err
done; done
for L in 1 0; do
  ARKV_LPT=$L timeout 300 python bench.py --workload qwen3-8b-8k-b8 --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/q.json 2>$O/q.err
  python -c "
import json; d=json.load(open('$O/q.json')); print('qwen lpt=$L tok/s=%.0f'%d['value'], 'kernel=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 $O/q.err
done
