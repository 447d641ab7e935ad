set -u
O=gpurun_out/g
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "graph or compress or merge_parity" > $O/t.log 2>&1; tail -n 3 $O/t.log
for w in resnet50 bert_large gpt2_xl; do
 for gf in "" "--no-graphs"; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 20 $gf --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot --no-union > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print('$w $gf', round(d['ms_per_step'],4), round(d['gate_bj5']['frac'],3), d['gpu_launches'], {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()})" || tail -n 5 $O/b.err
 done
done
