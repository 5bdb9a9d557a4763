#!/bin/bash
# Round 2: per-layer call cost breakdown.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_layer; mkdir -p $O
timeout 600 python scripts/layer_profile.py 80 0 > $O/layer_split.txt 2>&1; cat $O/layer_split.txt | tail -2
timeout 600 python scripts/layer_profile.py 80 3 > $O/layer_persist.txt 2>&1; cat $O/layer_persist.txt | tail -2
timeout 900 ncu --set full --clock-control none -k regex:decode_fast_kernel -s 1500 -c 1 -o $O/prof_layer python scripts/layer_profile.py 60 0 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py report $O/prof_layer.ncu-rep $O/prof_layer.json > /dev/null; rm -f $O/prof_layer.ncu-rep; cat $O/prof_layer.json | head -60
