#!/bin/bash
# Round-end artefacts (run under gpurun): default bench line, reference arm, smoke,
# ncu launch list of the bench command and --set full captures of the top kernels.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke exit=$?"
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench exit=$?"; cat gpurun_out/final/bench.json
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/final/reference.json 2> gpurun_out/final/reference.err; echo "ref exit=$?"; cat gpurun_out/final/reference.json
B="python bench.py --steps 200 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv \
   --log-file gpurun_out/final/launches.csv $B > /dev/null 2>&1; echo "ncu list exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o gpurun_out/final/prof_decode_fast $B > /dev/null 2>&1; echo "ncu decode exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_persist_kernel -s 150 -c 1 -o gpurun_out/final/prof_decode_persist python bench.py --kernel 3 --steps 200 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events > /dev/null 2>&1; echo "ncu persist exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tailor_move|tailor_select|prefill_tc" -c 4 -o gpurun_out/final/prof_tailor_prefill $B > /dev/null 2>&1; echo "ncu tailor/prefill exit=$?"
