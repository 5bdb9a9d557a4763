#!/bin/bash
# product (round-2 merges, defaults 0) GPU tests; A/B vs the warp merges with the prefetched
# first batch (tuning build, -DARKV_HH_LANE_MERGE=1 -DARKV_COMBINE_WARP_MERGE=1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4_ab3; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for n in 2 4 8; do
  timeout 300 python bench.py --steps 512 --emulate-shard $n > $O/e${n}_p.json 2>/dev/null
  ARKV_LIBRARY=$T timeout 300 python bench.py --steps 512 --emulate-shard $n --allow-tuning-library > $O/e${n}_t.json 2>/dev/null
done
timeout 300 python bench.py > $O/def_p.json 2>/dev/null
ARKV_LIBRARY=$T timeout 300 python bench.py --allow-tuning-library > $O/def_t.json 2>/dev/null
python -c "
import json
for k in ['e2','e4','e8','def']:
  p=json.load(open('$O/'+k+'_p.json')); t=json.load(open('$O/'+k+'_t.json'))
  print(k, 'round-2 merge', round(p['ms_per_step'],4), 'warp merge+prefetch', round(t['ms_per_step'],4))"
