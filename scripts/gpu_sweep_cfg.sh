cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 600 python -m pytest tests -m gpu -q -p no:randomly -k "mid_config or determinism" 2>&1 | tail -2
for CFG in 4,1 4,2 6,2 4,3 8,1; do for S in 2 3 5; do
  ARKV_FAST_CFG=$CFG ARKV_SPLITS=$S timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('cfg=$CFG S=$S', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))" 2>&1 | tail -1
done; done
