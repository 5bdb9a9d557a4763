#!/bin/bash
# warp-specialised tcgen05 prefill: 16 vs 8 epilogue warps (build switch), parity tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/pf2; mkdir -p $O
ARKV_NVCC_FLAGS="-DARKV_PF_EPI_WARPS=8" python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib8.so
python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib16.so
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "prefill or toy or mid_config or full_size_configs1" > $O/t.log 2>&1
echo "prefill tests (16 warps) exit=$?"; tail -2 $O/t.log
for V in 8 16 8 16; do
  cp /tmp/lib$V.so paper_2603_08727_b200/libarkv.so
  timeout 300 python scripts/prefill_time.py > $O/p$V.log 2>&1; echo "epi warps $V: $(tail -1 $O/p$V.log | cut -c1-120)"
done
cp /tmp/lib16.so paper_2603_08727_b200/libarkv.so
timeout 600 ncu --set full --clock-control none -k regex:prefill_ws -c 2 -o $O/prof_pfws python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py report $O/prof_pfws.ncu-rep $O/prof_pfws.json > /dev/null; rm -f $O/prof_pfws.ncu-rep
