cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
B="python bench.py --steps 200 --warmup 4 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 150 -c 1 -o gpurun_out/prof_decode_fast_r1j $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tailor_move -s 40 -c 1 -o gpurun_out/prof_move_r1j $B > /dev/null 2>&1
timeout 300 python bench.py --steps 2048 --warmup 8 > gpurun_out/bench_r1j.json 2> gpurun_out/bench_r1j.err
