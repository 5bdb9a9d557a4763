#!/bin/bash
# cost-balanced split-K launch list: parity, CTA timeline, A/B of the split rule
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r3_chunks; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 > $O/cta.txt 2>&1; tail -22 $O/cta.txt
for cfg in "ARKV_CHUNKS=0" "ARKV_CHUNKS=2" "ARKV_CHUNKS=1" "ARKV_WAVES=40" "ARKV_WAVES=50" "ARKV_QCOST=80" "ARKV_CTA_COST=0"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > $O/sp_$cfg.txt 2>&1; echo "$cfg"; tail -2 $O/sp_$cfg.txt
done
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; python -c "
import json;d=json.loads(open('$O/bench20.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'])"
