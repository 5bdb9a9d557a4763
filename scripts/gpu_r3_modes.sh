#!/bin/bash
# Round 2 (session 3, chunk pipeline): the paper's baselines through the same kernels (NEXT-1) + workloads, with the auto
# kernel choice; default bench line.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r3_modes; mkdir -p $O
B="python bench.py --steps 1024 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
summ() { python -c "import json; d=json.load(open('$1')); print('$2', 'tok/s %.0f' % d['value'], 'ms/step %.4f' % d['ms_per_step'], 'kernel frac %.3f' % d['roofline']['frac'], 'step frac %.3f' % d['step_hbm']['frac_of_peak'], d['config']['decode_kernel'][:12])" || tail -2 ${1%.json}.err; }
for m in arkv base origin quant; do timeout 900 $B --mode $m > $O/mode_$m.json 2>$O/mode_$m.err; summ $O/mode_$m.json "mode $m"; done
timeout 900 $B --quant fp8 > $O/fp8.json 2>$O/fp8.err; summ $O/fp8.json "fp8"
for w in qwen3-8b-8k-b8 llama3-8b-1k-b64 llama3-8b-128k; do timeout 900 $B --workload $w --steps 512 > $O/wl_$w.json 2>$O/wl_$w.err; summ $O/wl_$w.json "wl $w"; done
