#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_move; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 600 python scripts/prefill_time.py --reps 5 > $O/prefill.txt 2>&1; tail -4 $O/prefill.txt
BL="python bench.py --steps 400 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tailor_move_frag -s 0 -c 1 -o $O/prof_move $BL > /dev/null 2>&1; echo "ncu move exit=$?"
python scripts/ncu_summary.py report $O/prof_move.ncu-rep $O/prof_move.json > /dev/null 2>&1; python scripts/ncu_lines.py $O/prof_move.ncu-rep 20 > $O/prof_move_lines.txt 2>&1
python -c "
import json; d=json.load(open('$O/prof_move.json'))[0]; print(d['gpu__time_duration.sum'], d['smsp__issue_active.avg.pct_of_peak_sustained_active'], d['smsp__inst_executed.sum'])"
head -8 $O/prof_move_lines.txt
