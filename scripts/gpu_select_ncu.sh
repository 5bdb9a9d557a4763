#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/seln; mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tailor_select -s 4 -c 1 -o $O/prof_sel python bench.py --steps 120 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py report $O/prof_sel.ncu-rep $O/prof_sel.json > /dev/null
ncu -i $O/prof_sel.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
rm -f $O/prof_sel.ncu-rep
