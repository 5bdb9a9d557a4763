cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1500 python -m pytest tests -m gpu -q -p no:randomly -k "full_size" 2>&1 | tail -15 > gpurun_out/gpu_tests_h.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err
