cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
for cfg in "1 0" "1 1" "3 0" "3 1" "2 0"; do
  set -- $cfg
  for S in 3 6; do
  ARKV_SPLITS=$S ARKV_QGROUP=$1 ARKV_INTERLEAVE=$2 timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('qg=$1 il=$2 S=$S', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))"
  done
done
