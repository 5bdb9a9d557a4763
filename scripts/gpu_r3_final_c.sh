#!/bin/bash
# Round 2 session 3 artefacts, part B: default bench line, driver-like 20-step line, reference
# arm, ncu launch list of the bench command.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_final_c; mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2> $O/bench20.err; echo "bench20 exit=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench20b.json 2> $O/bench20b.err; echo "bench20b exit=$?"
timeout 900 python bench.py --impl reference --steps 8 --warmup 2 > $O/reference.json 2> $O/reference.err; echo "ref exit=$?"
python - <<'PY'
import json
for f in ("bench", "bench20", "bench20b"):
    d = json.loads(open(f"gpurun_out/r3_final_c/{f}.json").read().strip().splitlines()[-1])
    print(f, "value=%.0f" % d["value"], "ms=%.4f" % d["ms_per_step"], "e2e=%.0f" % d["e2e"]["value"],
          "kernel_frac=%.3f" % d["roofline"]["frac"], "traffic=%s" % d["roofline"]["traffic"], "step_frac=%.3f" % d["step_hbm"]["frac_of_peak"],
          "graph=%s" % d["per_layer_graph"].get("ms_per_step"), "cpu=%s" % d.get("cpu_baseline", {}).get("value"),
          "prefill=%s/%s" % (d["prefill"]["stats_ms"], d["prefill"]["finish_ms"]), "clk=%s" % d["clocks"])
d = json.loads(open("gpurun_out/r3_final_c/reference.json").read().strip().splitlines()[-1]); print("reference", d["value"], d["ms_per_step"])
PY
BL="python bench.py --steps 400 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|tailor|combine|hh_acc|prefill|persist" -c 3000 --csv --log-file $O/launches.csv $BL > /dev/null 2>&1; echo "ncu list exit=$?"
python scripts/ncu_summary.py launches $O/launches.csv $O/ncu_launches.md > /dev/null
cat $O/ncu_launches.md | head -16
