set -x
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1200 python -m pytest tests -m gpu -x -q -p no:randomly 2>&1 | tail -40 > gpurun_out/gpu_tests_4.log
timeout 900 python bench.py --steps 512 --warmup 8 --no-cpu-baseline > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
timeout 900 python bench.py --steps 512 --warmup 8 --no-cpu-baseline --kernel 1 > gpurun_out/bench_r1b_generic.json 2>> gpurun_out/bench_r1b.err
