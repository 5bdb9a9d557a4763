cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1200 python -m pytest tests -m gpu -x -q -p no:randomly 2>&1 | tail -3
timeout 900 python bench.py --cpu-steps 2 > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err
tail -2 gpurun_out/bench_r1e.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|prefill" -c 600 --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 64 --warmup 4 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
