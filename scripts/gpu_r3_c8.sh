#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_c8; mkdir -p $O
for cfg in "ARKV_FAST_PIPE=4" "ARKV_FAST_PIPE=8 ARKV_CTAS_PER_SM=1 ARKV_EXACT_WAVES=4" "ARKV_FAST_PIPE=8 ARKV_CTAS_PER_SM=1 ARKV_EXACT_WAVES=3" "ARKV_FAST_PIPE=8 ARKV_CTAS_PER_SM=1 ARKV_EXACT_WAVES=2"; do
mkdir -p "$O/$cfg"; env $cfg ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump "$O/$cfg" > "$O/$cfg/cta.txt" 2>&1; echo "$cfg"; grep -E "==|active" "$O/$cfg/cta.txt"
env $cfg ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 70 > "$O/$cfg/sp.txt" 2>&1; tail -2 "$O/$cfg/sp.txt"
done
