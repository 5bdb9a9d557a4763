#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3_chunkb; mkdir -p $O
for cb in 12288 9216; do
ARKV_NVCC_FLAGS="-DARKV_CHUNK_BYTES=$cb" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
mkdir -p $O/$cb; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/$cb > $O/$cb/cta.txt 2>&1; echo "chunk $cb"; grep -E "==|active" $O/$cb/cta.txt
for i in 1 2; do ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 70 > $O/$cb/sp$i.txt 2>&1; tail -2 $O/$cb/sp$i.txt; done
done
