#!/bin/bash
# compute-sanitizer (memcheck, racecheck) over the session-2 kernels: warp-specialised
# prefill (TMA + tcgen05), fused combine + HH, 3x2 decode ring, smoothed scores, move kernel
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/san2; mkdir -p $O; rm -f $O/summary.txt
SEL="toy_config or mid_config and 2-4-128-asym or smoothed and 0.5-2-head or prefill_statistics_natural or persistent_kernel_mid and 128 or batch_and_spare"
for TOOL in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 \
     python -m pytest tests/test_parity_gpu.py -q -p no:randomly -m gpu -k "$SEL" > $O/$TOOL.log 2>&1
  echo "$TOOL exit=$?" | tee -a $O/summary.txt
  grep -E "ERROR SUMMARY|passed|failed|Error" $O/$TOOL.log | tail -5 | tee -a $O/summary.txt
done
