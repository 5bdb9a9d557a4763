#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/pf3; mkdir -p $O
python -m paper_2603_08727_b200.build > /dev/null 2>&1
timeout 300 python -m pytest tests/test_parity_gpu.py -q -m gpu -x -k "prefill or toy or mid_config or full_size_configs1 or determinism" > $O/t.log 2>&1
echo "prefill tests exit=$?"; tail -2 $O/t.log
for V in 1 x 1 x; do
  ARKV_PREFILL_TC=$V timeout 300 python scripts/prefill_time.py > $O/p$V.log 2>&1; echo "variant $V: $(tail -1 $O/p$V.log | cut -c1-130)"
done
for W in qwen3-8b-8k-b8 llama3-8b-128k; do timeout 300 python scripts/prefill_time.py --workload $W 2>&1 | tail -1 | cut -c1-150; done
timeout 600 ncu --set full --clock-control none -k regex:prefill_ws -c 2 -o $O/prof_pfws python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py report $O/prof_pfws.ncu-rep $O/prof_pfws.json > /dev/null; rm -f $O/prof_pfws.ncu-rep
