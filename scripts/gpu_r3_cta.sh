#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r3_cta; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 > $O/arkv.txt 2>&1; cat $O/arkv.txt | tail -30
