set -x
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1200 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -30 > gpurun_out/gpu_tests_3.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 512 --warmup 8 --cpu-steps 2 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 24 --warmup 4 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 10 -c 2 -o gpurun_out/prof_decode_r1a python bench.py --steps 16 --warmup 4 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
