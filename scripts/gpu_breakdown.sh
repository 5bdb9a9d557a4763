#!/bin/bash
# ncu launch lists (our kernels only) for the split-K (2) and persistent (3) decode kernels
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/bd
for K in 2 3; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 2000 --csv \
     --log-file gpurun_out/bd/launches_k$K.csv \
     python bench.py --kernel $K --steps 200 --warmup 4 --no-cpu-baseline --e2e-steps 0 --no-ceiling --no-kernel-events > /dev/null 2>&1
  echo "ncu k$K exit=$?"
done
