#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_bulk; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 600 python scripts/step_profile.py --steps 60 > $O/bulk.txt 2>&1; echo bulk; tail -2 $O/bulk.txt
ARKV_LIBRARY=$T ARKV_HH_BULK=0 timeout 600 python scripts/step_profile.py --steps 60 > $O/stg.txt 2>&1; echo stg; tail -2 $O/stg.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ceiling > $O/bench20.json 2>$O/bench20.err
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -3 $O/gpu_tests.log
