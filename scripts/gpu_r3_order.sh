#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_order; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
for cfg in "ARKV_CHUNKS=0" "ARKV_CHUNKS=1" "ARKV_EXACT_WAVES=3" "ARKV_QCOST=50" "ARKV_QCOST=75" "ARKV_CHUNKS=0" "ARKV_CHUNKS=1"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
mkdir -p $O/c1; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/c1 > $O/c1/cta.txt 2>&1; grep -E "==|per CTA|active" $O/c1/cta.txt
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20_$i.json 2> $O/bench20_$i.err; python -c "
import json;d=json.loads(open('$O/bench20_$i.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'])"; done
