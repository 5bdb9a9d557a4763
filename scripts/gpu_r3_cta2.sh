#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
for c in 0 1; do
O=gpurun_out/r3_cta2/chunks$c; mkdir -p $O
ARKV_CHUNKS=$c ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 4 8 20 40 60 --dump $O > $O/cta.txt 2>&1; grep "==" $O/cta.txt
done
O=gpurun_out/r3_cta2/s6; mkdir -p $O
ARKV_CHUNKS=0 ARKV_SPLITS=6 ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O > $O/cta.txt 2>&1; grep "==" $O/cta.txt
O=gpurun_out/r3_cta2/s2; mkdir -p $O
ARKV_CHUNKS=0 ARKV_SPLITS=2 ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O > $O/cta.txt 2>&1; grep "==" $O/cta.txt
