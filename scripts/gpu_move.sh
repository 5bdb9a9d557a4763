#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/mv
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/mv/t.log 2>&1; echo "gpu tests exit=$?"; tail -3 gpurun_out/mv/t.log
python scripts/prefill_time.py > gpurun_out/mv/pf.json 2>gpurun_out/mv/pf.err; cat gpurun_out/mv/pf.json; tail -2 gpurun_out/mv/pf.err
ARKV_MOVE_GENERIC=1 python scripts/prefill_time.py > gpurun_out/mv/pf_generic.json 2>&1; cat gpurun_out/mv/pf_generic.json
timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/mv/b.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/mv/b.json')); print('bench', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|tailor" --csv --log-file gpurun_out/mv/launches.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tailor_move" -c 1 -o gpurun_out/mv/prof_move python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu full exit=$?"
