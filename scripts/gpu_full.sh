#!/bin/bash
# Full GPU test suite + compute-sanitizer pass (run under gpurun)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/full/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 gpurun_out/full/gpu_tests.log
bash scripts/sanitize.sh
