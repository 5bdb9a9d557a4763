cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
for M in 0 1; do for rep in 1 2; do
  ARKV_PRODUCER=$M timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('mode=$M', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))"
done; done
