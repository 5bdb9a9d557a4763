#!/bin/bash
# GPU tests + configs[1] bench (1024 steps, x2) + launch list of the tailor/combine kernels
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/q; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 $O/gpu_tests.log
for R in 1 2; do
timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling $EXTRA > $O/b.json 2>$O/b.err
python -c "
import json; d=json.load(open('$O/b.json')); print('tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 $O/b.err
done
B="python bench.py --steps 400 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|persist" -c 3000 --csv \
   --log-file $O/launches.csv $B > /dev/null 2>&1; echo "ncu list exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md | tail -8
