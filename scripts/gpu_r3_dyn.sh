#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_dyn; mkdir -p $O
ARKV_LIBRARY=$T ARKV_DYN_ITEMS=1 timeout 900 python -m pytest tests -m gpu -x -q -k "toy or mid_config or gqa or full_size_configs1_sampled or graph" > $O/tests_dyn.log 2>&1; tail -2 $O/tests_dyn.log
for c in 0 1; do
  mkdir -p $O/d$c
  ARKV_CHUNKS=0 ARKV_DYN_ITEMS=$c ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/d$c > $O/d$c/cta.txt 2>&1; grep -E "==|per CTA" $O/d$c/cta.txt
done
for cfg in "ARKV_CHUNKS=0 ARKV_DYN_ITEMS=0" "ARKV_CHUNKS=0 ARKV_DYN_ITEMS=1" "ARKV_CHUNKS=0 ARKV_DYN_ITEMS=1 ARKV_SPLITS=4" "ARKV_CHUNKS=0 ARKV_DYN_ITEMS=1 ARKV_SPLITS=6"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
