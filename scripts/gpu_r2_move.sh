#!/bin/bash
# Round 2: move kernels with a 1-D grid of exactly the jobs' tiles; tests; prefill timing; ncu.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_move; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -3 $O/gpu_tests.log
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 $B > $O/bench.json 2>$O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); print('bench', d['value'], d['ms_per_step'], 'P1', d['prefill']['stats_ms'], 'finish', d['prefill']['finish_ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"tailor|prefill" -c 12 --csv --log-file $O/launches.csv $B --steps 8 > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null; cat $O/ncu_launches.md | tail -8
