#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/mvn; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tailor_move -c 1 -o $O/prof_move python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py report $O/prof_move.ncu-rep $O/prof_move.json > /dev/null
ncu -i $O/prof_move.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
rm -f $O/prof_move.ncu-rep
