#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_wave; mkdir -p $O
for cfg in "ARKV_DECODE_NOPDL=0" "ARKV_DECODE_NOPDL=1" "ARKV_FAST_PIPE=2"; do
mkdir -p "$O/$cfg"; env $cfg ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump "$O/$cfg" > "$O/$cfg/cta.txt" 2>&1; echo $cfg; grep -E "==|active" "$O/$cfg/cta.txt"
done
nvidia-smi -q | grep -iE "mig|compute mode|persistence" | head
