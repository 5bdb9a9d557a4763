#!/bin/bash
# tailor move kernel: parity tests + prefill finish timing + launch list of the prefill tailor
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/mv; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu -x > $O/t.log 2>&1
echo "gpu tests exit=$?"; tail -1 $O/t.log
for R in 1 2; do timeout 300 python scripts/prefill_time.py 2>&1 | tail -1 | cut -c1-120; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tailor --csv --log-file $O/launches.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/l.md | tail -4
timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err
python -c "
import json; d=json.load(open('$O/b.json')); print('tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'], d['prefill']['stats_ms'], d['prefill']['finish_ms'])" || tail -2 $O/b.err
