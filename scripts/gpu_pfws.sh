#!/bin/bash
# warp-specialised tcgen05 prefill: prefill parity tests, timing vs the first tcgen05 kernel
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/pf; mkdir -p $O
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "prefill or toy or mid_config or full_size_configs1" > $O/t.log 2>&1
echo "prefill tests exit=$?"; tail -5 $O/t.log
for V in 1 2 1 2; do
  ARKV_PREFILL_TC=$V timeout 300 python scripts/prefill_time.py > $O/p$V.log 2>&1; echo "variant $V"; tail -4 $O/p$V.log
done
