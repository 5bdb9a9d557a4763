#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_ncu_q; mkdir -p $O
timeout 600 python scripts/step_profile.py --steps 60 --rho 0 > $O/sp.txt 2>&1; tail -2 $O/sp.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_chunk_kernel --launch-skip 45 --launch-count 1 -o $O/quant -f python scripts/step_profile.py --steps 48 --rho 0 > $O/ncu1.log 2>&1; tail -1 $O/ncu1.log
mkdir -p $O/pl; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --per-layer --at 8 40 --dump $O/pl > $O/pl/cta.txt 2>&1; cat $O/pl/cta.txt | grep -v "Q share"
