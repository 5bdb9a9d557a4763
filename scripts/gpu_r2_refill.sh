#!/bin/bash
# Round 2: self-refill (each consumer warp loads its own items) vs the in-order producer.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_refill; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --allow-tuning-library"
summ() { python -c "import json; d=json.load(open('$1')); g=d['per_layer_graph']; print('$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'], 'graph', g.get('ms_per_step') if g else None)" || tail -2 ${1%.json}.err; }
for r in 1 0; do
  ARKV_LIBRARY=$T ARKV_SELF_REFILL=$r timeout 600 $B --graph-steps 64 > $O/n1_r$r.json 2>$O/n1_r$r.err; summ $O/n1_r$r.json "N=1 refill=$r"
  ARKV_LIBRARY=$T ARKV_SELF_REFILL=$r timeout 600 $B --no-graph --emulate-shard 8 > $O/n8_r$r.json 2>$O/n8_r$r.err; summ $O/n8_r$r.json "N=8 refill=$r"
  ARKV_LIBRARY=$T ARKV_SELF_REFILL=$r timeout 600 $B --no-graph --emulate-shard 4 > $O/n4_r$r.json 2>$O/n4_r$r.err; summ $O/n4_r$r.json "N=4 refill=$r"
  ARKV_LIBRARY=$T ARKV_SELF_REFILL=$r timeout 600 $B --no-graph --steps 20 --warmup 5 --repeats 5 > $O/hh_r$r.json 2>$O/hh_r$r.err; summ $O/hh_r$r.json "20-step refill=$r"
done
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -2 $O/gpu_tests.log
