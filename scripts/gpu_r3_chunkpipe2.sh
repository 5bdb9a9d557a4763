#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_chunkpipe2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
for cfg in "ARKV_FAST_PIPE=2" "ARKV_FAST_PIPE=4"; do
  env ARKV_LIBRARY=$T ARKV_PERSIST_QSHARE=101 $cfg timeout 600 python scripts/step_profile.py --steps 40 --rho 0 > "$O/spq_$cfg.txt" 2>&1; echo "rho0 split-K $cfg"; tail -2 "$O/spq_$cfg.txt"
done
env ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 40 --rho 0 > "$O/spq_persist.txt" 2>&1; echo "rho0 auto(persistent)"; tail -2 "$O/spq_persist.txt"
for cfg in "ARKV_FAST_PIPE=2" "ARKV_FAST_PIPE=4" "ARKV_FAST_PIPE=2" "ARKV_FAST_PIPE=4"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
