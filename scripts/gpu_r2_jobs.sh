#!/bin/bash
# Round 2: tailor job-array size (kernel parameter bytes) vs decode step; acc prefetch A/B; prefill.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_jobs; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
B="python bench.py --steps 1024 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
summ() { python -c "import json; d=json.load(open('$1')); print('$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'], 'P1 %.3f finish %.3f' % (d['prefill']['stats_ms'], d['prefill']['finish_ms']))" || tail -2 ${1%.json}.err; }
timeout 600 $B > $O/jobs256.json 2>$O/jobs256.err; summ $O/jobs256.json "product (jobs 256, acc prefetch)"
timeout 600 $B --steps 20 --warmup 5 > $O/jobs256_20.json 2>$O/jobs256_20.err; summ $O/jobs256_20.json "product 20 steps"
timeout 600 python scripts/step_profile.py --steps 80 > $O/steps.txt 2>&1; tail -2 $O/steps.txt
ARKV_NVCC_FLAGS="-DARKV_MAX_JOBS=96" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
ARKV_LIBRARY=$T timeout 600 $B --allow-tuning-library > $O/jobs96.json 2>$O/jobs96.err; summ $O/jobs96.json "jobs 96"
ARKV_LIBRARY=$T ARKV_ACC_PREFETCH=0 timeout 600 $B --allow-tuning-library --steps 20 --warmup 5 > $O/nopref_20.json 2>$O/nopref_20.err; summ $O/nopref_20.json "jobs96 no acc prefetch 20 steps"
ARKV_LIBRARY=$T timeout 600 $B --allow-tuning-library --steps 20 --warmup 5 > $O/pref_20.json 2>$O/pref_20.err; summ $O/pref_20.json "jobs96 acc prefetch 20 steps"
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -3 $O/gpu_tests.log
