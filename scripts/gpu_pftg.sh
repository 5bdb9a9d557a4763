#!/bin/bash
# prefill epilogue: tile groups (default) vs column groups (ARKV_PF_TILE_GROUPS=0)
cd $GRAFT_REPO_ROOT
O=gpurun_out/pftg; mkdir -p $O
ARKV_NVCC_FLAGS="-DARKV_PF_TILE_GROUPS=0" python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib0.so
python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib1.so
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "prefill or toy or mid_config or full_size_configs1 or determinism or smoothed" > $O/t.log 2>&1
echo "tests (tile groups) exit=$?"; tail -1 $O/t.log
for R in 1 2; do for V in 0 1; do
  cp /tmp/lib$V.so paper_2603_08727_b200/libarkv.so
  timeout 300 python scripts/prefill_time.py > $O/p$V.log 2>&1; echo "tile groups $V: $(tail -1 $O/p$V.log | cut -c1-110)"
done; done
cp /tmp/lib1.so paper_2603_08727_b200/libarkv.so
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:prefill_ws --csv --log-file $O/l.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/l.csv $O/l.md | tail -3
