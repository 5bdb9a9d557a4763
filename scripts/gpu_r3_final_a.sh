#!/bin/bash
# Round 2 session 3 artefacts, part A: GPU tests, smoke, ncu --set full of the decode kernel
# (HH-window step and steady step of the bench command), of the HH combine and of the
# prefill-end tailor move; emulated shards.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_final; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -1 $O/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit=$?"; tail -1 $O/smoke.log
BL="python bench.py --steps 400 --warmup 4 --repeats 1 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_chunk_kernel -s 8 -c 1 -o $O/prof_decode_hh $BL > /dev/null 2>&1; echo "ncu decode hh exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_chunk_kernel -s 150 -c 1 -o $O/prof_decode_steady $BL > /dev/null 2>&1; echo "ncu decode steady exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_combine_hh -s 8 -c 1 -o $O/prof_combine_hh $BL > /dev/null 2>&1; echo "ncu combine_hh exit=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tailor_move_frag -s 0 -c 1 -o $O/prof_move $BL > /dev/null 2>&1; echo "ncu move exit=$?"
for f in prof_decode_hh prof_decode_steady prof_combine_hh prof_move; do python scripts/ncu_summary.py report $O/$f.ncu-rep $O/$f.json > /dev/null 2>&1; python scripts/ncu_lines.py $O/$f.ncu-rep 30 > $O/${f}_lines.txt 2>&1; done
python - <<'PY'
import json
for f in ("prof_decode_hh", "prof_decode_steady", "prof_combine_hh", "prof_move"):
    try:
        d = json.load(open(f"gpurun_out/r3_final/{f}.json"))[0]
        print(f, d["kernel"][:40], d["gpu__time_duration.sum"], "rd", d["dram__bytes_read.sum"], "wr", d["dram__bytes_write.sum"], "issue", d["smsp__issue_active.avg.pct_of_peak_sustained_active"])
    except Exception as e:
        print(f, "missing", e)
PY
for n in 2 4 8; do timeout 600 python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-graph --emulate-shard $n > $O/emul_n$n.json 2>$O/emul_n$n.err; python -c "import json; d=json.load(open('$O/emul_n$n.json')); print('emulated N=$n', 'ms/step %.4f' % d['ms_per_step'], 'tok/s %.0f' % d['value'])"; done
