#!/bin/bash
# Persistent decode kernel with 3 consumers x 2 stages: GPU tests + workloads, split vs persistent
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/p2
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/p2/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 gpurun_out/p2/gpu_tests.log
one() {
  python -c "
import json; d=json.load(open('gpurun_out/p2/$1.json')); print('$1', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 gpurun_out/p2/$1.err
}
B="timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling"
for K in 2 3; do $B --kernel $K > gpurun_out/p2/k$K.json 2>gpurun_out/p2/k$K.err; one k$K; done
for K in 2 3; do $B --kernel $K --mode quant > gpurun_out/p2/q$K.json 2>gpurun_out/p2/q$K.err; one q$K; done
B5="timeout 300 python bench.py --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling"
for W in qwen3-8b-8k-b8 llama3-8b-1k-b64 llama3-8b-128k; do
  $B5 --workload $W --kernel 3 > gpurun_out/p2/${W}_k3.json 2>gpurun_out/p2/${W}_k3.err; one ${W}_k3
done
