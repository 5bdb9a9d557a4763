#!/bin/bash
# Round-1 (second session) artefacts: smoke, default bench line, reference arm, ncu launch
# list of the bench command, --set full of the decode kernel (summarised on the box).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/final2; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit=$?"; cat $O/bench.json
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $O/reference.json 2> $O/reference.err; echo "ref exit=$?"; cat $O/reference.json
B="python bench.py --steps 400 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv \
   --log-file $O/launches.csv $B > /dev/null 2>&1; echo "ncu list exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o $O/prof_decode_fast $B > /dev/null 2>&1; echo "ncu decode exit=$?"
python scripts/ncu_summary.py report $O/prof_decode_fast.ncu-rep $O/prof_decode_fast.json > /dev/null
ncu -i $O/prof_decode_fast.ncu-rep --page source --csv --print-source sass > $O/prof_decode_fast_sass.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none -k regex:"tailor_move|tailor_select|tailor_scan|combine" -s 20 -c 4 -o $O/prof_tailor $B > /dev/null 2>&1; echo "ncu tailor exit=$?"
python scripts/ncu_summary.py report $O/prof_tailor.ncu-rep $O/prof_tailor.json > /dev/null
rm -f $O/prof_tailor.ncu-rep
ls -la $O
