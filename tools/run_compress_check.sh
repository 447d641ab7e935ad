set -u
O=gpurun_out/cc
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "compress or full_size or graph or readme or files or multi_rank or merge or exchange" > $O/t.log 2>&1; tail -n 3 $O/t.log
for w in resnet50 gpt2_xl resnet50 gpt2_xl; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 10 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot --no-union > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print('$w', round(d['ms_per_step'],4), d['per_step_ms']['p50'], round(d['gate_bj5']['frac'],3), {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}, d['spec'])" || tail -n 5 $O/b.err
done
