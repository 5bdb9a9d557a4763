#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_tune; mkdir -p $O
for cfg in "ARKV_QCOST=62" "ARKV_QCOST=45" "ARKV_QCOST=35" "ARKV_QCOST=62 ARKV_EXACT_WAVES=3" "ARKV_QCOST=45 ARKV_EXACT_WAVES=3"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
mkdir -p $O/tl; ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/tl > $O/tl/cta.txt 2>&1; grep -E "==|per CTA|active" $O/tl/cta.txt
for n in 8 2; do
for p in 2 4; do
ARKV_LIBRARY=$T ARKV_FAST_PIPE=$p timeout 600 python bench.py --steps 64 --warmup 5 --repeats 3 --emulate-shard $n --allow-tuning-library > $O/emul${n}_p$p.json 2> $O/emul${n}_p$p.err; python -c "
import json;d=json.loads(open('$O/emul${n}_p$p.json').read().strip().splitlines()[-1]);print('emul $n pipe $p',d['value'],d['ms_per_step'],d['roofline']['frac'],d.get('per_layer_graph',{}).get('ms_per_step'))"
done; done
