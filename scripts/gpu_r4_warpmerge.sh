#!/bin/bash
# A/B: split merges by the whole warp in the combine and the HH combine (product) vs the
# lane-per-(head, dim) merges of HEAD (tuning build, -DARKV_HH_LANE_MERGE=0
# -DARKV_COMBINE_WARP_MERGE=0): default bench lines (steady state) and 20-step lines.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4_warpmerge; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
for i in 1 2 3; do
  timeout 600 python bench.py > $O/def_p$i.json 2>/dev/null
  ARKV_LIBRARY=$T timeout 600 python bench.py --allow-tuning-library > $O/def_t$i.json 2>/dev/null
  timeout 600 python bench.py --steps 20 --warmup 5 > $O/b20_p$i.json 2>/dev/null
  ARKV_LIBRARY=$T timeout 600 python bench.py --steps 20 --warmup 5 --allow-tuning-library > $O/b20_t$i.json 2>/dev/null
done
python - <<'PY'
import json
O='gpurun_out/r4_warpmerge'
for k in ['def','b20']:
  for v in ['p','t']:
    xs=[json.load(open(f'{O}/{k}_{v}{i}.json')) for i in (1,2,3)]
    print(k, 'warp-merge' if v=='p' else 'head', [round(x['value'],1) for x in xs], [round(x['roofline']['kernel_ms_per_launch']*1e3,2) for x in xs])
PY
