#!/bin/bash
# Round 2 artefacts: GPU tests, smoke, default bench line, driver-like 20-step line, reference
# arm, emulated shards, ncu launch list of the bench command, --set full of the decode kernel.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_final; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -2 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; echo "bench20 exit=$?"
timeout 900 python bench.py --impl reference --steps 8 --warmup 2 > $O/reference.json 2> $O/reference.err; echo "ref exit=$?"
python - <<'PY'
import json
for f in ("bench", "bench20"):
    d = json.load(open(f"gpurun_out/r2_final/{f}.json"))
    print(f, "value=%.0f" % d["value"], "ms=%.4f" % d["ms_per_step"], "e2e=%.0f" % d["e2e"]["value"],
          "kernel_frac=%.3f" % d["roofline"]["frac"], "step_frac=%.3f" % d["step_hbm"]["frac_of_peak"],
          "graph=%s" % d["per_layer_graph"].get("ms_per_step"), "cpu=%s" % d.get("cpu_baseline", {}).get("value"),
          "clk=%s" % d["clocks"])
d = json.load(open("gpurun_out/r2_final/reference.json")); print("reference", d["value"], d["ms_per_step"])
PY
for n in 2 4 8; do timeout 600 python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-graph --emulate-shard $n > $O/emul_n$n.json 2>$O/emul_n$n.err; python -c "import json; d=json.load(open('$O/emul_n$n.json')); print('emulated N=$n', 'ms/step %.4f' % d['ms_per_step'], 'tok/s %.0f' % d['value'])"; done
BL="python bench.py --steps 400 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv --log-file $O/launches.csv $BL > /dev/null 2>&1; echo "ncu list exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast_kernel -s 150 -c 1 -o $O/prof_decode_fast $BL > /dev/null 2>&1; echo "ncu decode exit=$?"
python scripts/ncu_summary.py report $O/prof_decode_fast.ncu-rep $O/prof_decode_fast.json > /dev/null
rm -f $O/prof_decode_fast.ncu-rep
cat $O/ncu_launches.md | head -14
