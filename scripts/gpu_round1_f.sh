cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
for F in 1 0; do for S in 2 3 4; do
  ARKV_SPLITS=$S ARKV_FUSE_COMBINE=$F timeout 300 python bench.py --steps 1024 --warmup 8 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); print('fuse=$F S=$S', 'tok/s=%.0f'%d['value'], 'ms/step=%.4f'%d['ms_per_step'], 'kernel_ms=%.4f'%d['roofline']['kernel_ms_per_launch'], 'kGB/s=%.0f frac=%.3f'%(d['roofline']['achieved'], d['roofline']['frac']))"
done; done
ARKV_SPLITS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 60 -c 1 -o gpurun_out/prof_decode_fast_r1g python bench.py --steps 80 --warmup 4 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
