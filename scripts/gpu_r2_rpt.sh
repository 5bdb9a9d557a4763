#!/bin/bash
# Round 2: HH combine 256 x 8 vs 512 x 4 rows per block (A/B, same box); tests.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_rpt; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
for rep in 1 2; do
timeout 600 python scripts/step_profile.py --steps 50 > $O/rpt8_$rep.txt 2>&1; echo "rpt8"; tail -2 $O/rpt8_$rep.txt | head -1
ARKV_LIBRARY=$T ARKV_HH_RPT=4 timeout 600 python scripts/step_profile.py --steps 50 > $O/rpt4_$rep.txt 2>&1; echo "rpt4"; tail -2 $O/rpt4_$rep.txt | head -1
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ceiling > $O/bench20.json 2>$O/bench20.err
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 1800 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -2 $O/gpu_tests.log
