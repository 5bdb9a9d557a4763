#!/bin/bash
# prefill: FMA-pipe exponentials every Nth element (build switch ARKV_PF_POLY_EVERY)
cd $GRAFT_REPO_ROOT
O=gpurun_out/pf4; mkdir -p $O
for N in 0 3 8; do
  ARKV_NVCC_FLAGS="-DARKV_PF_POLY_EVERY=$N" python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib$N.so
done
python -m paper_2603_08727_b200.build --force > /dev/null 2>&1 && cp paper_2603_08727_b200/libarkv.so /tmp/lib4.so
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "prefill or toy or mid_config or full_size_configs1 or determinism" > $O/t.log 2>&1
echo "prefill tests (poly 4) exit=$?"; tail -1 $O/t.log
for R in 1 2; do for N in 0 3 4 8; do
  cp /tmp/lib$N.so paper_2603_08727_b200/libarkv.so
  timeout 300 python scripts/prefill_time.py > $O/p$N.log 2>&1; echo "poly every $N: $(tail -1 $O/p$N.log | cut -c1-110)"
done; done
cp /tmp/lib4.so paper_2603_08727_b200/libarkv.so
