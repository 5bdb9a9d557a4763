#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/pf2
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pf2/t.log 2>&1; echo "gpu tests exit=$?"; tail -1 gpurun_out/pf2/t.log
python scripts/prefill_time.py > gpurun_out/pf2/tc.json 2>gpurun_out/pf2/tc.err; cat gpurun_out/pf2/tc.json; tail -2 gpurun_out/pf2/tc.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prefill|tailor" --csv --log-file gpurun_out/pf2/launches.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
