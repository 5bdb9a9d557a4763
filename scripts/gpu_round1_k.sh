cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1800 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -15 > gpurun_out/gpu_tests_k.log
for TC in 1 0; do ARKV_PREFILL_TC=$TC timeout 600 python bench.py --no-cpu-baseline --steps 1024 > gpurun_out/bench_r1k_tc$TC.json 2> gpurun_out/bench_r1k_tc$TC.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|prefill" -c 600 --csv --log-file gpurun_out/launches_r1k.csv python bench.py --steps 64 --warmup 4 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
