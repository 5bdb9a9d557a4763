cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1200 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -15 > gpurun_out/gpu_tests_g.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke_g.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err
B="python bench.py --steps 64 --warmup 4 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|prefill" -c 600 --csv --log-file gpurun_out/launches_r1g.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 40 -c 1 -o gpurun_out/prof_decode_fast_r1g2 $B > /dev/null 2>&1
