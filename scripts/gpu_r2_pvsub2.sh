#!/bin/bash
# Round 2: PV subnormal fix for fp8 + full GPU tests + per-layer graph launch list.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_pvsub2; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -4 $O/gpu_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|persist" -c 2000 --csv \
   --log-file $O/launches_graph.csv python bench.py --steps 16 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --graph-steps 16 > /dev/null 2>&1; echo "ncu exit=$?"
python scripts/ncu_summary.py launches $O/launches_graph.csv $O/ncu_launches_graph.md > /dev/null; cat $O/ncu_launches_graph.md
