#!/bin/bash
# In-situ L2 behaviour of the HH step (no cache flush between kernels; application replay)
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_l2; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 900 ncu --metrics $M --cache-control none --clock-control none --replay-mode application -k regex:"decode_combine_hh|decode_chunk" --launch-skip 14 --launch-count 4 --csv python scripts/step_profile.py --steps 12 > $O/l2.csv 2> $O/l2.err; echo "exit=$?"
grep -E "decode_combine_hh|decode_chunk" $O/l2.csv | cut -c1-400 | head -40
