#!/bin/bash
# Round 2: ncu of the decode kernel in an emulated 8-GPU shard (32 units per call), and of
# the prefill-end tailor kernels.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_ncu_small; mkdir -p $O
B="python bench.py --steps 64 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 60 -c 1 -o $O/n8 $B --emulate-shard 8 > /dev/null 2>&1; echo "ncu n8 exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tailor_move_frag|tailor_select" -c 2 -o $O/prefill_tailor $B > /dev/null 2>&1; echo "ncu prefill exit=$?"
for r in n8 prefill_tailor; do
  python scripts/ncu_summary.py report $O/$r.ncu-rep $O/$r.json > /dev/null
  ncu -i $O/$r.ncu-rep --page source --csv --print-source sass > $O/${r}_sass.csv 2>/dev/null
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file $O/launches_n8.csv $B --emulate-shard 8 --steps 16 > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/launches_n8.csv $O/ncu_launches_n8.md > /dev/null; cat $O/ncu_launches_n8.md | tail -8
rm -f $O/*.ncu-rep
