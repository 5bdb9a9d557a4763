cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
B="python bench.py --steps 40 --warmup 4 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|prefill" -c 400 --csv --log-file gpurun_out/launches_r1d.csv $B > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 8 -c 1 -o gpurun_out/prof_decode_fast_r1d $B > gpurun_out/ncu_full1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_pass -c 2 -o gpurun_out/prof_prefill_r1d $B > gpurun_out/ncu_full2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tailor_move|tailor_select" -c 2 -o gpurun_out/prof_tailor_r1d $B > gpurun_out/ncu_full3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:decode_combine -s 8 -c 1 -o gpurun_out/prof_combine_r1d $B > gpurun_out/ncu_full4.log 2>&1
ls -la gpurun_out/*.ncu-rep
