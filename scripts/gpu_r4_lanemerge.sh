#!/bin/bash
# A/B: HH combine's split merge by the whole warp (product) vs lane-per-head (tuning build,
# -DARKV_HH_LANE_MERGE=0); then GPU tests and bench lines of the product build.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4_lanemerge; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
for i in 1 2 3; do
  timeout 600 python scripts/step_profile.py --steps 40 > $O/p_$i.txt 2>&1; echo "lane-merge"; tail -2 $O/p_$i.txt | head -1
  ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 40 > $O/t_$i.txt 2>&1; echo "per-head"; tail -2 $O/t_$i.txt | head -1
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; tail -c 300 $O/bench20.json | head -c 300; echo
ARKV_LIBRARY=$T timeout 600 python bench.py --steps 20 --warmup 5 --allow-tuning-library > $O/bench20_perhead.json 2> $O/bench20_perhead.err
python -c "import json;[print(f, json.load(open('$O/'+f))['value']) for f in ['bench20.json','bench20_perhead.json']]"
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; python -c "import json;print('default', json.load(open('$O/bench.json'))['value'])"
