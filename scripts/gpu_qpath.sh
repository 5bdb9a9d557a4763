cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 1200 python -m pytest tests -m gpu -q -p no:randomly -x 2>&1 | tail -3
for M in arkv quant origin; do for CFG in 4,1 6,2; do
  ARKV_FAST_CFG=$CFG timeout 300 python bench.py --mode $M --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 --no-ceiling > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('$M cfg=$CFG', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))"
done; done
