#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_occ; mkdir -p $O
ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 --dump $O > $O/cta.txt 2>&1; grep -E "occupancy|==|active" $O/cta.txt
