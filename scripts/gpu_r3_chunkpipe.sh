#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_chunkpipe; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
for cfg in "ARKV_FAST_PIPE=2" "ARKV_FAST_PIPE=3" "ARKV_FAST_PIPE=4" "ARKV_FAST_PIPE=2"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
for cfg in "ARKV_FAST_PIPE=2" "ARKV_FAST_PIPE=3" "ARKV_FAST_PIPE=4"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python bench.py --steps 256 --warmup 5 --mode quant --allow-tuning-library > "$O/quant_$cfg.json" 2> "$O/quant_$cfg.err"; python -c "
import json;d=json.loads(open('$O/quant_$cfg.json').read().strip().splitlines()[-1]);print('quant $cfg',d['value'],d['ms_per_step'],d['roofline']['frac'])"
done
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; python -c "
import json;d=json.loads(open('$O/bench20.json').read().strip().splitlines()[-1]);print('bench20',d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['kernel_ms_per_launch'],d['e2e']['value'])"
