#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/shb
for SH in head layer; do
timeout 600 python bench.py --sharing $SH --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/shb/b$SH.json 2>gpurun_out/shb/b$SH.err
python -c "
import json; d=json.load(open('gpurun_out/shb/b$SH.json')); print('$SH', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/shb/b$SH.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tailor_select" -c 40 --csv --log-file gpurun_out/shb/sel_layer.csv python bench.py --sharing layer --steps 100 --warmup 4 --no-cpu-baseline --e2e-steps 0 --no-ceiling --no-kernel-events > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tailor_select" -c 40 --csv --log-file gpurun_out/shb/sel_head.csv python bench.py --steps 100 --warmup 4 --no-cpu-baseline --e2e-steps 0 --no-ceiling --no-kernel-events > /dev/null 2>&1
echo done
