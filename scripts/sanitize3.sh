#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the session-3 kernels: chunked
# split-K decode pipeline with the cost-balanced launch order, HH combine, cp.async move
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/san3; mkdir -p $O; rm -f $O/summary.txt
SEL="toy_config or mid_config and 2-4-128-asym or mid_config and fp8 or gqa_groups and 1-8 or batch_and_spare or smoothed and 0.5-2-head"
for TOOL in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 \
     python -m pytest tests/test_parity_gpu.py -q -p no:randomly -m gpu -k "$SEL" > $O/$TOOL.log 2>&1
  echo "$TOOL exit=$?" | tee -a $O/summary.txt
  grep -E "ERROR SUMMARY|passed|failed|Error" $O/$TOOL.log | tail -5 | tee -a $O/summary.txt
done
