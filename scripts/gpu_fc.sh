#!/bin/bash
# fused (last split CTA) vs separate combine with the 3x2 kernel
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/fc; mkdir -p $O
for F in 0 1 0 1; do
ARKV_FUSE_COMBINE=$F timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err
python -c "
import json; d=json.load(open('$O/b.json')); print('fuse=$F tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 $O/b.err
done
