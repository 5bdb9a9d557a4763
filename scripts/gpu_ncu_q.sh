#!/bin/bash
# ncu --set full (with source) of the decode kernel in ARKV mode and Base_quant mode
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/nq
for M in quant arkv; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o gpurun_out/nq/prof_$M \
  python bench.py --mode $M --steps 200 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1; echo "ncu $M exit=$?"
done
