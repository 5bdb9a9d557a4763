#!/bin/bash
# select kernel with the shared-memory key cache: GPU tests, tailor launch lists (prefill +
# decode), bench A/B (ARKV_SELECT_NOCACHE)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/sel; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/t.log 2>&1; echo "gpu tests exit=$?"; tail -1 $O/t.log
for NC in 0; do
  if [ $NC = 1 ]; then export ARKV_SELECT_NOCACHE=1; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tailor --csv --log-file $O/l$NC.csv python bench.py --steps 300 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1
  python scripts/ncu_summary.py launches $O/l$NC.csv $O/l$NC.md | tail -3
  timeout 300 python scripts/prefill_time.py 2>&1 | tail -1 | cut -c1-110
  timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('nocache=$NC tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'])" || tail -2 $O/b.err
done
