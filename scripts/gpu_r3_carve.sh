#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_carve; mkdir -p $O
mkdir -p $O/tl; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/tl > $O/tl/cta.txt 2>&1; grep -E "==|active" $O/tl/cta.txt
for i in 1 2; do env ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$i.txt" 2>&1; tail -2 "$O/sp_$i.txt"; done
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; python -c "
import json;d=json.loads(open('$O/bench20.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'],d['e2e']['value'])"
