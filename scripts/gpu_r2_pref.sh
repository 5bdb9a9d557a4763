#!/bin/bash
# Round 2: L2 prefetch depth for small calls (emulated N-GPU shards) and the batched default.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_pref; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
B="python bench.py --steps 256 --warmup 8 --repeats 2 --no-cpu-baseline --no-ceiling --no-e2e --allow-tuning-library"
run() { ARKV_LIBRARY=$T ARKV_PREFETCH=$2 timeout 600 $B --emulate-shard $1 $3 > $O/n$1_p$2.json 2>$O/n$1_p$2.err
  python -c "import json; d=json.load(open('$O/n$1_p$2.json')); g=d['per_layer_graph']; print('N=$1 prefetch=$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'], 'graph', g.get('ms_per_step') if g else None)" || tail -2 $O/n$1_p$2.err; }
for p in 0 2 4 8 16 64; do run 8 $p --no-graph; done
for p in 0 4 16; do run 1 $p "--graph-steps 64"; done
for p in 0 4 16; do run 2 $p --no-graph; done
