#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_persist; mkdir -p $O
for cfg in "ARKV_CHUNKS=0" "ARKV_DECODE_PERSIST=1" "ARKV_CHUNKS=0 ARKV_SPLITS=2"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
