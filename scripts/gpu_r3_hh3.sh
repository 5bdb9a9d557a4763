#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_hh3; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
for i in 1 2; do timeout 600 python scripts/step_profile.py --steps 70 > $O/sp$i.txt 2>&1; tail -2 $O/sp$i.txt; done
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench20_$i.json 2> $O/bench20_$i.err; python -c "
import json;d=json.loads(open('$O/bench20_$i.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'],d['e2e']['value'])"; done
