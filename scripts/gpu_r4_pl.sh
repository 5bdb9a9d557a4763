#!/bin/bash
# per-layer call timeline (tuning build = product defaults): where a ~34 MB layer call's time goes
cd $GRAFT_REPO_ROOT
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r4_pl; mkdir -p $O
ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --per-layer --at 8 40 --dump $O > $O/cta.txt 2>&1; tail -60 $O/cta.txt
