#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_rpt; mkdir -p $O
for cfg in "ARKV_HH_RPT=8" "ARKV_HH_RPT=4" "ARKV_HH_RPT=8" "ARKV_HH_RPT=4"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 40 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt" | head -1
done
