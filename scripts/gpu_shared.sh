#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/sh
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/sh/t.log 2>&1; echo "gpu tests exit=$?"; tail -3 gpurun_out/sh/t.log; grep -E "^FAILED|^E  " gpurun_out/sh/t.log | head -10
for SH in head layer; do
timeout 600 python bench.py --sharing $SH --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/sh/b$SH.json 2>gpurun_out/sh/b$SH.err
python -c "
import json; d=json.load(open('gpurun_out/sh/b$SH.json')); print('$SH', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'])" || tail -3 gpurun_out/sh/b$SH.err
done
