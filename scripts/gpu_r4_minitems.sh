#!/bin/bash
# small calls: per-CTA work cap (ARKV_MIN_ITEMS, tuning build = product defaults) vs the
# per-layer CUDA-graph mode and the emulated 8-GPU shard (32 units per call)
cd $GRAFT_REPO_ROOT
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r4_mi; mkdir -p $O
for mi in ${MI_LIST:-20 8 4 20 8 4}; do
  ARKV_MIN_ITEMS=$mi ARKV_LIBRARY=$T timeout 600 python bench.py --steps 64 --allow-tuning-library > $O/def_$mi.json 2>/dev/null
  ARKV_MIN_ITEMS=$mi ARKV_LIBRARY=$T timeout 600 python bench.py --steps 256 --emulate-shard 8 --allow-tuning-library > $O/e8_$mi.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/def_$mi.json')); e=json.load(open('$O/e8_$mi.json'))
print('min_items $mi', 'default', round(d['value']), 'per-layer-graph ms/step', round(d['per_layer_graph']['ms_per_step'],4), 'emul8', round(e['value']), round(e['ms_per_step'],4))"
done
