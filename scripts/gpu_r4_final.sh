#!/bin/bash
# session 4 final: GPU tests, smoke, bench lines (default, driver window), emulated shards
cd $GRAFT_REPO_ROOT
O=gpurun_out/r4_final; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err
for n in 2 4 8; do timeout 600 python bench.py --steps 512 --emulate-shard $n > $O/emul_n$n.json 2>/dev/null; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference.json 2> $O/reference.err
python - <<'PY'
import json
O='gpurun_out/r4_final'
for f in ['bench','bench20','emul_n2','emul_n4','emul_n8','reference']:
    try:
        d=json.load(open(f'{O}/{f}.json')); print(f, round(d['value'],1), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('per_layer_graph') or {}).get('ms_per_step'), (d.get('clocks') or {}))
    except Exception as e: print(f, 'ERR', e)
PY
