#!/bin/bash
# A/B of a compile-time switch: $1 = extra nvcc flags of variant B (variant A = default).
# Alternates the two libraries over 3 rounds of configs[1] (ARKV mode) and Base_quant mode.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/abb
python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/libA.so
ARKV_NVCC_FLAGS="$1" python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/libB.so
echo "B flags: $1"
for R in 1 2 3; do for V in A B; do
  cp /tmp/lib$V.so paper_2603_08727_b200/libarkv.so
  for M in arkv quant; do
    timeout 300 python bench.py --mode $M --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/abb/$V$M$R.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/abb/$V$M$R.json')); print('$V $M r$R', 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])"
  done
done; done
cp /tmp/libA.so paper_2603_08727_b200/libarkv.so
