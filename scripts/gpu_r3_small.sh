#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_small; mkdir -p $O
for mi in 20 10 6 3; do
ARKV_LIBRARY=$T ARKV_MIN_ITEMS=$mi timeout 600 python bench.py --steps 64 --warmup 5 --repeats 3 --emulate-shard 8 --allow-tuning-library > $O/emul8_$mi.json 2> $O/emul8_$mi.err; python -c "
import json;d=json.loads(open('$O/emul8_$mi.json').read().strip().splitlines()[-1]);print('emul8 min_items $mi',round(d['value']),d['ms_per_step'],round(d['roofline']['frac'],3),d.get('per_layer_graph',{}).get('ms_per_step'))"
done
for mi in 20 10 6; do
ARKV_LIBRARY=$T ARKV_MIN_ITEMS=$mi timeout 600 python bench.py --steps 64 --warmup 5 --repeats 3 --allow-tuning-library > $O/n1_$mi.json 2> $O/n1_$mi.err; python -c "
import json;d=json.loads(open('$O/n1_$mi.json').read().strip().splitlines()[-1]);print('n1 min_items $mi',round(d['value']),d['ms_per_step'],round(d['roofline']['frac'],3),d.get('per_layer_graph',{}).get('ms_per_step'))"
done
