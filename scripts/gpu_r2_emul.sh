#!/bin/bash
# Round 2: emulated N-GPU shards on one GPU (per-GPU step time of the batch x KV-head partition).
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_emul; mkdir -p $O
B="python bench.py --steps 512 --warmup 8 --repeats 3 --no-cpu-baseline --no-ceiling --no-e2e --no-graph"
for wl in llama3-8b-32k qwen3-8b-8k-b8; do
for n in 1 2 4 8; do
  timeout 900 $B --workload $wl --emulate-shard $n > $O/${wl}_n$n.json 2>$O/${wl}_n$n.err
  python -c "import json; d=json.load(open('$O/${wl}_n$n.json')); print('$wl N=$n', 'ms/step %.4f' % d['ms_per_step'], 'tok/s %.0f' % d['value'], 'kernel frac %.3f' % d['roofline']['frac'], d['config']['parallelism'][:40])" || tail -3 $O/${wl}_n$n.err
done
done
timeout 900 $B --workload llama3-8b-128k-b4 --emulate-shard 8 --steps 256 > $O/128k_n8.json 2>$O/128k_n8.err
python -c "import json; d=json.load(open('$O/128k_n8.json')); print('128k-b4 N=8', 'ms/step %.4f' % d['ms_per_step'], 'tok/s %.0f' % d['value'], 'kernel frac %.3f' % d['roofline']['frac'])" || tail -3 $O/128k_n8.err
