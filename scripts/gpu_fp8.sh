#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/fp8
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/fp8/t.log 2>&1; echo "gpu tests exit=$?"; tail -3 gpurun_out/fp8/t.log; grep -E "^FAILED|^E  " gpurun_out/fp8/t.log | head -10
for K in 2 3; do
timeout 600 python bench.py --quant fp8 --kernel $K --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/fp8/b$K.json 2>gpurun_out/fp8/b$K.err
python -c "
import json; d=json.load(open('gpurun_out/fp8/b$K.json')); print('fp8 k$K', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.3f'%d['roofline']['frac'], d['config']['quant'], d['config']['decode_kernel'], d['memory'])" || tail -5 gpurun_out/fp8/b$K.err
done
