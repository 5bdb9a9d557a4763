#!/bin/bash
# Round 2: HH combine without empty blocks + ex2.approx: tests, HH step time, ncu of the combine.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_hh2; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -3 $O/gpu_tests.log
timeout 600 python scripts/step_profile.py --steps 80 > $O/steps.txt 2>&1; tail -2 $O/steps.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ceiling > $O/bench20.json 2>$O/bench20.err
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['ms_per_step_runs'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode|combine" -c 60 --csv --log-file $O/launches.csv python scripts/step_profile.py --steps 30 > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null; cat $O/ncu_launches.md | tail -5
