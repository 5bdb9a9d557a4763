#!/bin/bash
# Round 2: HH-window step cost breakdown (per-step events + ncu launch list of steps 0..60).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_hh; mkdir -p $O
timeout 600 python scripts/step_profile.py --steps 120 > $O/steps.txt 2>&1; echo "steps exit=$?"; tail -3 $O/steps.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ceiling > $O/bench20.json 2>$O/bench20.err; echo "bench20 exit=$?"
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc" -c 400 --csv \
   --log-file $O/launches.csv python scripts/step_profile.py --steps 60 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null; cat $O/ncu_launches.md
