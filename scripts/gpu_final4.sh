#!/bin/bash
# Round-1 end-of-session artefacts: GPU tests, smoke, default bench line, reference arm,
# other workloads, ncu launch list of the bench command, --set full of the decode kernel and
# of the two prefill passes (summarised on the box).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/final4; mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -1 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?"
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit=$?"; cat $O/bench.json
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > $O/reference.json 2> $O/reference.err; echo "ref exit=$?"
for W in qwen3-8b-8k-b8 llama3-8b-1k-b64 llama3-8b-128k; do
  timeout 600 python bench.py --workload $W --steps 512 --warmup 8 --no-cpu-baseline --no-ceiling > $O/wl_$W.json 2>$O/wl_$W.err
  python -c "
import json; d=json.load(open('$O/wl_$W.json')); print('$W', 'tok/s=%.0f'%d['value'], 'e2e=%.0f'%d['e2e']['value'], 'kernel=%s'%d['config']['decode_kernel'], 'frac=%.4f'%d['roofline']['frac'], 'prefill_stats_ms=%.3f'%d['prefill']['stats_ms'])" || tail -2 $O/wl_$W.err
done
timeout 600 python bench.py --quant fp8 --steps 1024 --warmup 8 --no-cpu-baseline --no-ceiling > $O/fp8.json 2>$O/fp8.err
python -c "
import json; d=json.load(open('$O/fp8.json')); print('fp8', 'tok/s=%.0f'%d['value'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 $O/fp8.err
B="python bench.py --steps 400 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling --no-kernel-events"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv \
   --log-file $O/launches.csv $B > /dev/null 2>&1; echo "ncu list exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o $O/prof_decode_fast $B > /dev/null 2>&1; echo "ncu decode exit=$?"
python scripts/ncu_summary.py report $O/prof_decode_fast.ncu-rep $O/prof_decode_fast.json > /dev/null
rm -f $O/prof_decode_fast.ncu-rep
timeout 900 ncu --set full --clock-control none -k regex:"prefill_ws|tailor_move" -c 3 -o $O/prof_prefill $B > /dev/null 2>&1; echo "ncu prefill exit=$?"
python scripts/ncu_summary.py report $O/prof_prefill.ncu-rep $O/prof_prefill.json > /dev/null
rm -f $O/prof_prefill.ncu-rep
ls $O
