#!/bin/bash
# Round 2: pipeline shape (consumers x stages per warp) with self-refill, batched and small calls.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_cfg; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph --allow-tuning-library"
summ() { python -c "import json; d=json.load(open('$1')); print('$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'])" || tail -2 ${1%.json}.err; }
for c in 32 42 22 23 62 43; do
  ARKV_LIBRARY=$T ARKV_FAST_CFG=$c timeout 600 $B > $O/n1_c$c.json 2>$O/n1_c$c.err; summ $O/n1_c$c.json "N=1 cfg=$c"
  ARKV_LIBRARY=$T ARKV_FAST_CFG=$c timeout 600 $B --emulate-shard 8 > $O/n8_c$c.json 2>$O/n8_c$c.err; summ $O/n8_c$c.json "N=8 cfg=$c"
done
