#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_trim; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 600 python scripts/step_profile.py --steps 60 --rho 0 > $O/spq.txt 2>&1; echo rho0; tail -2 $O/spq.txt
for i in 1 2; do timeout 600 python scripts/step_profile.py --steps 70 > $O/sp$i.txt 2>&1; tail -2 $O/sp$i.txt; done
B="python bench.py --steps 1024 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 $B --mode quant > $O/quant.json 2>$O/quant.err; python -c "import json; d=json.load(open('$O/quant.json')); print('quant', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3))"
timeout 900 $B > $O/arkv.json 2>$O/arkv.err; python -c "import json; d=json.load(open('$O/arkv.json')); print('arkv', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3))"
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; python -c "
import json;d=json.loads(open('$O/bench20.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'],d['e2e']['value'])"
