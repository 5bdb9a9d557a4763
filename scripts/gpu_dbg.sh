cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
for args in "--prompt-len 32768 --layers 8" "--prompt-len 9000"; do
  echo "== $args"
  ARKV_DEBUG_SYNC=1 timeout 300 python bench.py --steps 16 --warmup 2 --no-cpu-baseline --e2e-steps 0 $args 2>&1 | grep -E "arkv:|ms_per_step" | cut -c 1-200
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:randomly 2>&1 | tail -3
timeout 900 python bench.py --steps 512 --warmup 8 --cpu-steps 2 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err
tail -2 gpurun_out/bench_r1c.err
