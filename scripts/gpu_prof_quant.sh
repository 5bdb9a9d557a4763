cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 100 -c 1 -o gpurun_out/prof_quant python bench.py --mode quant --steps 120 --warmup 4 --e2e-steps 0 --no-cpu-baseline --no-ceiling > /dev/null 2>&1
ls -la gpurun_out/prof_quant.ncu-rep
