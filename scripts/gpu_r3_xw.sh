#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3_xw; mkdir -p $O
for fl in "-DARKV_CHUNK_XWARPS=0" "-DARKV_CHUNK_XWARPS=1" "-DARKV_CHUNK_MINB=1"; do
ARKV_NVCC_FLAGS="$fl" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
mkdir -p "$O/$fl"; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump "$O/$fl" > "$O/$fl/cta.txt" 2>&1; echo "$fl"; grep -E "==|active" "$O/$fl/cta.txt"
ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 70 > "$O/$fl/sp.txt" 2>&1; tail -2 "$O/$fl/sp.txt"
done
