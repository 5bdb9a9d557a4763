#!/bin/bash
# Re-entry check of HEAD on a B200: GPU test suite, smoke, default bench line.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
mkdir -p gpurun_out/r1b
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r1b/gpu_tests.log 2>&1
echo "gpu tests exit=$?"; tail -3 gpurun_out/r1b/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b/smoke.log 2>&1; echo "smoke exit=$?"
timeout 900 python bench.py > gpurun_out/r1b/bench.json 2> gpurun_out/r1b/bench.err; echo "bench exit=$?"; cat gpurun_out/r1b/bench.json
