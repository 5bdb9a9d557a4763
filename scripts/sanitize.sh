#!/bin/bash
# compute-sanitizer over the toy + mid-size GPU parity tests (run under gpurun).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/san
rm -f gpurun_out/san/summary.txt
SEL="toy_config or mid_config and 2-4-128-asym or batch_and_spare or no_prefill_tailor or sharded_prefill or persistent_kernel_mid and 128 or gqa_groups and 1-8"
for TOOL in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 --error-exitcode 9 \
     python -m pytest tests/test_parity_gpu.py -q -p no:randomly -m gpu -k "$SEL" > gpurun_out/san/$TOOL.log 2>&1
  echo "$TOOL exit=$?" | tee -a gpurun_out/san/summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/$TOOL.log | tail -3 | tee -a gpurun_out/san/summary.txt
done
# synccheck with the mma.sync prefill instead of the tcgen05 one (tool coverage of tcgen05)
ARKV_PREFILL_MMA=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --error-exitcode 9 \
   python -m pytest tests/test_parity_gpu.py -q -p no:randomly -m gpu -k "sharded_prefill" > gpurun_out/san/synccheck_notc.log 2>&1
echo "synccheck (ARKV_PREFILL_MMA=1, sharded_prefill) exit=$?" | tee -a gpurun_out/san/summary.txt
grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/synccheck_notc.log | tail -3 | tee -a gpurun_out/san/summary.txt
