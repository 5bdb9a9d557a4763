#!/bin/bash
# Round 2: split count with self-refill (emulated shards and the default).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_ssweep2; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph --allow-tuning-library"
run() { ARKV_LIBRARY=$T ARKV_SPLITS=$2 timeout 600 $B --emulate-shard $1 > $O/n$1_s$2.json 2>$O/n$1_s$2.err
  python -c "import json; d=json.load(open('$O/n$1_s$2.json')); print('N=$1 S=$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'])" || tail -2 $O/n$1_s$2.err; }
for s in 6 8 9 12 16 19 24 28; do run 8 $s; done
for s in 4 6 9 12; do run 4 $s; done
for s in 2 3 4 5; do run 1 $s; done
