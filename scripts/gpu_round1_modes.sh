cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/r1m
timeout 900 python bench.py > gpurun_out/r1m/default.json 2> gpurun_out/r1m/default.err
for M in base origin quant arkv; do
  timeout 600 python bench.py --mode $M --steps 1024 --no-cpu-baseline --no-ceiling > gpurun_out/r1m/mode_$M.json 2> gpurun_out/r1m/mode_$M.err
done
timeout 900 python bench.py --workload qwen3-8b-8k-b8 --steps 512 --no-cpu-baseline --no-ceiling > gpurun_out/r1m/wl_qwen.json 2> gpurun_out/r1m/wl_qwen.err
timeout 900 python bench.py --workload llama3-8b-1k-b64 --steps 192 --no-cpu-baseline --no-ceiling > gpurun_out/r1m/wl_b64.json 2> gpurun_out/r1m/wl_b64.err
timeout 900 python bench.py --workload llama3-8b-128k --steps 512 --no-cpu-baseline --no-ceiling > gpurun_out/r1m/wl_128k.json 2> gpurun_out/r1m/wl_128k.err
ls -la gpurun_out/r1m
