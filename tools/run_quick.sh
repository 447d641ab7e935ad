# quick GPU check (not product): parity tests + short benches of two workloads
set -u
O=gpurun_out/q
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -n 3 $O/gpu_tests.log
for w in resnet50 gpt2_xl; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 10 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/$w.json 2> $O/$w.err
  python -c "import json;d=json.load(open('$O/$w.json'));print('$w', round(d['ms_per_step'],4), {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}, d['gate_bj5']['frac'])"
done
