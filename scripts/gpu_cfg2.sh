#!/bin/bash
# 3x2 pipeline default: GPU tests, split-count sweep, other workloads, fp8
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/cfg2
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/cfg2/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 gpurun_out/cfg2/gpu_tests.log
run() {  # name, env..., args
  local n=$1; shift
  env "$@" > /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cfg2/$n.json')); print('$n', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'frac=%.4f'%d['roofline']['frac'])" || tail -2 gpurun_out/cfg2/$n.err
}
B="timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling"
for S in 2 3 4 5; do ARKV_SPLITS=$S $B > gpurun_out/cfg2/s$S.json 2>gpurun_out/cfg2/s$S.err; run s$S true; done
$B > gpurun_out/cfg2/auto.json 2>gpurun_out/cfg2/auto.err; run auto true
$B --quant fp8 > gpurun_out/cfg2/fp8.json 2>gpurun_out/cfg2/fp8.err; run fp8 true
ARKV_FAST_CFG=4,1 $B --quant fp8 > gpurun_out/cfg2/fp8_41.json 2>gpurun_out/cfg2/fp8_41.err; run fp8_41 true
B5="timeout 300 python bench.py --steps 512 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling"
for W in qwen3-8b-8k-b8 llama3-8b-1k-b64 llama3-8b-128k; do
  $B5 --workload $W > gpurun_out/cfg2/$W.json 2>gpurun_out/cfg2/$W.err; run $W true
  ARKV_FAST_CFG=4,1 $B5 --workload $W > gpurun_out/cfg2/${W}_41.json 2>gpurun_out/cfg2/${W}_41.err; run ${W}_41 true
  $B5 --workload $W --kernel 3 > gpurun_out/cfg2/${W}_k3.json 2>gpurun_out/cfg2/${W}_k3.err; run ${W}_k3 true
done
