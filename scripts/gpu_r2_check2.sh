#!/bin/bash
# Round 2: GPU tests (lattice full-size, non-finite, stats) + new bench (default and driver-like).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_check2; mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2>$O/bench20.err; echo "bench20 exit=$?"; tail -3 $O/bench20.err
python -c "import json; d=json.load(open('$O/bench20.json')); print('bench20', d['value'], d['ms_per_step'], d['e2e']['value'], d['per_layer_graph'], d['step_hbm'], d['roofline']['frac'], d['cpu_baseline'])"
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -15 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2>$O/bench.err; echo "bench exit=$?"; tail -3 $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'], d['per_layer_graph'], d['step_hbm'], d['roofline']['frac'], d['config']['ms_per_step_runs'])"
timeout 900 python bench.py --impl reference --steps 8 --warmup 2 > $O/reference.json 2>$O/reference.err; echo "ref exit=$?"; cat $O/reference.json; tail -3 $O/reference.err
