#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_fuse; mkdir -p $O
ARKV_LIBRARY=$T ARKV_FUSE_COMBINE=1 timeout 900 python -m pytest tests -m gpu -x -q -k "toy or mid_config or gqa or full_size_configs1_sampled or graph or batch" > $O/tests.log 2>&1; tail -1 $O/tests.log
for cfg in "ARKV_FUSE_COMBINE=0" "ARKV_FUSE_COMBINE=1" "ARKV_FUSE_COMBINE=0" "ARKV_FUSE_COMBINE=1"; do
  env ARKV_LIBRARY=$T $cfg timeout 600 python scripts/step_profile.py --steps 70 > "$O/sp_$cfg.txt" 2>&1; echo "$cfg"; tail -2 "$O/sp_$cfg.txt"
done
B="python bench.py --steps 512 --warmup 40 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --allow-tuning-library"
for f in 0 1 0 1; do ARKV_LIBRARY=$T ARKV_FUSE_COMBINE=$f timeout 900 $B > $O/b_$f.json 2>$O/b_$f.err; python -c "import json; d=json.loads(open('$O/b_$f.json').read().strip().splitlines()[-1]); print('fuse $f', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3), d['per_layer_graph']['ms_per_step'])"; done
for f in 0 1; do ARKV_LIBRARY=$T ARKV_FUSE_COMBINE=$f timeout 900 $B --emulate-shard 8 > $O/e8_$f.json 2>$O/e8_$f.err; python -c "import json; d=json.loads(open('$O/e8_$f.json').read().strip().splitlines()[-1]); print('emul8 fuse $f', round(d['value']), d['ms_per_step'], round(d['roofline']['frac'],3), d['per_layer_graph']['ms_per_step'])"; done
