#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_pl; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
for mi in 20 8 4; do
mkdir -p $O/m$mi; ARKV_MIN_ITEMS=$mi ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --per-layer --at 8 40 --dump $O/m$mi > $O/m$mi/cta.txt 2>&1; echo "min_items $mi"; grep -E "layer call|==|CTA durations|per CTA" $O/m$mi/cta.txt
done
