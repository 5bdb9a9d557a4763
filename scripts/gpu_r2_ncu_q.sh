#!/bin/bash
# Round 2: ncu --set full with source of the decode kernel in quant mode (Q-tile path), in
# the default mode, and of the HH combine.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_ncu_q; mkdir -p $O
B="python bench.py --steps 64 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 40 -c 1 -o $O/quant $B --mode quant > /dev/null 2>&1; echo "ncu quant exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 120 -c 1 -o $O/arkv $B > /dev/null 2>&1; echo "ncu arkv exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_combine_hh -s 10 -c 1 -o $O/combine_hh $B > /dev/null 2>&1; echo "ncu hh exit=$?"
for r in quant arkv combine_hh; do
  python scripts/ncu_summary.py report $O/$r.ncu-rep $O/$r.json > /dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_sass.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
done
ls -la $O
rm -f $O/*.ncu-rep
