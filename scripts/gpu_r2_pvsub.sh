#!/bin/bash
# Round 2: PV on subnormal codes (probability scale 2^-24): parity, A/B vs exact unpack,
# quant mode, per-layer split sweep.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_pvsub; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 2400 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1; echo "gpu tests exit=$?"; tail -4 $O/gpu_tests.log
timeout 900 python scripts/diag_lattice.py 3 32768 2,3 asym > $O/diag32k.txt 2>&1; cat $O/diag32k.txt
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --graph-steps 64"
summ() { python -c "import json,sys; d=json.load(open('$1')); print('$2', 'ms/step %.4f' % d['ms_per_step'], 'kernel frac %.3f' % d['roofline']['frac'], 'kernel ms %.4f' % d['roofline']['kernel_ms_per_launch'], 'graph', d['per_layer_graph'].get('ms_per_step'))" 2>/dev/null || tail -2 ${1%.json}.err; }
timeout 600 $B > $O/sub_arkv.json 2>$O/sub_arkv.err; summ $O/sub_arkv.json "pvsub arkv"
timeout 600 $B --mode quant --no-graph > $O/sub_quant.json 2>$O/sub_quant.err; summ $O/sub_quant.json "pvsub quant(split)"
timeout 600 $B --mode quant --no-graph --kernel 3 > $O/sub_quant_p.json 2>$O/sub_quant_p.err; summ $O/sub_quant_p.json "pvsub quant(persist)"
ARKV_NVCC_FLAGS="-DARKV_PV_SUB=0" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
ARKV_LIBRARY=$T timeout 600 $B --allow-tuning-library > $O/exact_arkv.json 2>$O/exact_arkv.err; summ $O/exact_arkv.json "exact arkv"
ARKV_LIBRARY=$T timeout 600 $B --allow-tuning-library --mode quant --no-graph > $O/exact_quant.json 2>$O/exact_quant.err; summ $O/exact_quant.json "exact quant(split)"
python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
for mi in 4 8 24 48 1000; do
  ARKV_LIBRARY=$T ARKV_MIN_ITEMS=$mi timeout 600 $B --allow-tuning-library --no-graph --graph-steps 64 > $O/mi_$mi.json 2>$O/mi_$mi.err
  ARKV_LIBRARY=$T ARKV_MIN_ITEMS=$mi timeout 600 $B --allow-tuning-library > $O/mi_$mi.json 2>$O/mi_$mi.err; summ $O/mi_$mi.json "min_items $mi"
done
