#!/bin/bash
# Prefill kernel: parity tests, event timing (tcgen05 vs mma.sync), ncu launch list
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/pf
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pf/t.log 2>&1; echo "gpu tests exit=$?"; tail -1 gpurun_out/pf/t.log
python scripts/prefill_time.py > gpurun_out/pf/tc.json 2>gpurun_out/pf/tc.err; cat gpurun_out/pf/tc.json; tail -2 gpurun_out/pf/tc.err
ARKV_PREFILL_TC=0 python scripts/prefill_time.py > gpurun_out/pf/mma.json 2>&1; cat gpurun_out/pf/mma.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill" --csv --log-file gpurun_out/pf/launches.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prefill_tc" -c 2 -o gpurun_out/pf/prof_prefill python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu full exit=$?"
