#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_exact; mkdir -p $O
for cfg in "ARKV_CHUNKS=0" "ARKV_CHUNKS=2" "ARKV_CHUNKS=1 ARKV_EXACT_WAVES=2" "ARKV_CHUNKS=1 ARKV_EXACT_WAVES=3" "ARKV_CHUNKS=1 ARKV_EXACT_WAVES=4" "ARKV_CHUNKS=2 ARKV_SPLITS=2" "ARKV_CHUNKS=2 ARKV_SPLITS=4" "ARKV_CHUNKS=0"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
mkdir -p $O/e3; ARKV_CHUNKS=1 ARKV_EXACT_WAVES=3 ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/e3 > $O/e3/cta.txt 2>&1; grep -E "==|per CTA|active" $O/e3/cta.txt
mkdir -p $O/m2; ARKV_CHUNKS=2 ARKV_LIBRARY=$T timeout 600 python scripts/cta_timeline.py --at 8 40 --dump $O/m2 > $O/m2/cta.txt 2>&1; grep -E "==|per CTA|active" $O/m2/cta.txt
