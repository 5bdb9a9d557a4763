#!/bin/bash
# Round 2: L2 residency hints for the HH logits (A/B) + GPU tests.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_l2; mkdir -p $O
timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_hints.txt 2>&1; echo "steps exit=$?"; tail -3 $O/steps_hints.txt
ARKV_LIBRARY=$PWD/paper_2603_08727_b200/libarkv_tuning.so ARKV_L2_HINTS=0 timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_nostream.txt 2>&1; echo "steps exit=$?"; tail -3 $O/steps_nostream.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ceiling > $O/bench20.json 2>$O/bench20.err; echo "bench20 exit=$?"
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 600 python bench.py --steps 2048 --warmup 8 --no-cpu-baseline --no-ceiling > $O/bench2048.json 2>$O/bench2048.err; echo "bench2048 exit=$?"
python -c "import json; d=json.load(open('$O/bench2048.json')); print('bench2048', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc" -c 120 --csv \
   --log-file $O/launches.csv python scripts/step_profile.py --steps 40 > /dev/null 2>&1; echo "ncu exit=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -5 $O/gpu_tests.log
