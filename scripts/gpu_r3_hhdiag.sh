#!/bin/bash
# HH-window diagnosis: per-step kernel time with and without the HH logit stores (tuning build)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r3_hhdiag; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 70 > $O/store.txt 2>&1; echo store; tail -3 $O/store.txt
ARKV_LIBRARY=$T ARKV_HH_NOSTORE=1 timeout 600 python scripts/step_profile.py --steps 70 > $O/nostore.txt 2>&1; echo nostore; tail -3 $O/nostore.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; tail -c 600 $O/bench20.json
