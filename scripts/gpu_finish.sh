#!/bin/bash
# launch list of the prefill path (P1-P4) at configs[1]; bench smoke of the new prefill block
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/fin; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python scripts/prefill_time.py --reps 1 > /dev/null 2>&1; echo "ncu exit=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/fin/launches.csv')))
st = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[st]; ix = {k: j for j, k in enumerate(h)}
agg = collections.OrderedDict()
for r in rows[st + 1:]:
    if len(r) < len(h): continue
    key = (r[ix['ID']], r[ix['Kernel Name']].split('(')[0])
    v = float(r[ix['Metric Value']].replace(',', '')); u = r[ix['Metric Unit']]
    m = r[ix['Metric Name']]
    if m == 'gpu__time_duration.sum': v = v / 1e3 if u == 'ns' else (v * 1e3 if u == 'ms' else v)
    else: v = v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1) / 1e6
    agg.setdefault(key, {})[m] = v
for (i, n), d in agg.items():
    print(f"{n[:40]:40s} {d.get('gpu__time_duration.sum', 0):9.1f} us  R {d.get('dram__bytes_read.sum', 0):9.1f} MB  W {d.get('dram__bytes_write.sum', 0):8.1f} MB")
PY
timeout 300 python bench.py --steps 64 --warmup 4 --no-cpu-baseline --e2e-steps 0 --no-ceiling > $O/b.json 2>$O/b.err; echo "bench exit=$?"
python -c "import json; d=json.load(open('$O/b.json')); print(d['prefill'])" || tail -3 $O/b.err
