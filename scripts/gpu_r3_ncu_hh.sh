#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_ncu_hh; mkdir -p $O
timeout 600 python scripts/step_profile.py --steps 70 > $O/sp.txt 2>&1; tail -2 $O/sp.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_combine_hh --launch-skip 8 --launch-count 1 -o $O/combine_hh -f python scripts/step_profile.py --steps 12 > $O/ncu1.log 2>&1; tail -2 $O/ncu1.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:decode_fast_kernel --launch-skip 8 --launch-count 1 -o $O/decode_hh -f python scripts/step_profile.py --steps 12 > $O/ncu2.log 2>&1; tail -2 $O/ncu2.log
