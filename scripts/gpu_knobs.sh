#!/bin/bash
# Runtime knobs of the 3x2 split-K kernel at configs[1] + ncu source captures (arkv, quant)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/kn
B="timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling"
one() {
  python -c "
import json; d=json.load(open('gpurun_out/kn/$1.json')); print('$1', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 gpurun_out/kn/$1.err
}
$B > gpurun_out/kn/base.json 2>gpurun_out/kn/base.err; one base
for QG in 1 2; do ARKV_QGROUP=$QG $B > gpurun_out/kn/qg$QG.json 2>gpurun_out/kn/qg$QG.err; one qg$QG; done
for IO in 0 2; do ARKV_ITEM_ORDER=$IO $B > gpurun_out/kn/io$IO.json 2>gpurun_out/kn/io$IO.err; one io$IO; done
for PF in 1 2; do ARKV_PREFETCH=$PF $B > gpurun_out/kn/pf$PF.json 2>gpurun_out/kn/pf$PF.err; one pf$PF; done
ARKV_INTERLEAVE=1 $B > gpurun_out/kn/il.json 2>gpurun_out/kn/il.err; one il
for M in quant arkv; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o gpurun_out/kn/prof_$M \
  python bench.py --mode $M --steps 200 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1; echo "ncu $M exit=$?"
done
