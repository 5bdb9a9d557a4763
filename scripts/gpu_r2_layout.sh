#!/bin/bash
# Round 2: [row][G] HH logits + split cap by items per CTA: tests, HH step time, per-layer sweep.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_layout; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 2400 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -4 $O/gpu_tests.log
timeout 600 python scripts/step_profile.py --steps 100 > $O/steps.txt 2>&1; echo "steps"; tail -2 $O/steps.txt
B="python bench.py --steps 256 --warmup 8 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --graph-steps 64"
for mi in 4 8 12 24 48; do
  ARKV_LIBRARY=$T ARKV_MIN_ITEMS=$mi timeout 600 $B > $O/mi_$mi.json 2>$O/mi_$mi.err
  python -c "import json; d=json.load(open('$O/mi_$mi.json')); print('min_items $mi', 'batched %.4f ms' % d['ms_per_step'], 'graph %s' % d['per_layer_graph'].get('ms_per_step'))" 2>/dev/null || tail -2 $O/mi_$mi.err
done
timeout 600 $B --kernel 3 > $O/persist.json 2>$O/persist.err
python -c "import json; d=json.load(open('$O/persist.json')); print('persistent', 'batched %.4f ms' % d['ms_per_step'], 'graph %s' % d['per_layer_graph'].get('ms_per_step'))" || tail -2 $O/persist.err
