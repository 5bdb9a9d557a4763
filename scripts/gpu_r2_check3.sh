#!/bin/bash
# Round 2: GPU tests + bench lines after the PV exact unpack / HH cleanup.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_check3; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -6 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench20.json 2>$O/bench20.err; echo "bench20 exit=$?"; tail -2 $O/bench20.err
timeout 900 python bench.py > $O/bench.json 2>$O/bench.err; echo "bench exit=$?"; tail -2 $O/bench.err
python - <<'PY'
import json
for f in ("bench20", "bench"):
    d = json.load(open(f"gpurun_out/r2_check3/{f}.json"))
    print(f, "value=%.0f" % d["value"], "ms=%.4f" % d["ms_per_step"], "e2e=%.0f" % d["e2e"]["value"],
          "frac=%.3f" % d["roofline"]["frac"], "step_frac=%.3f" % d["step_hbm"]["frac_of_peak"],
          "graph=%s" % d["per_layer_graph"].get("value"), "clk=%s" % d["clocks"])
PY
