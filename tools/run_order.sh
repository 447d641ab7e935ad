set -u
O=gpurun_out/or
mkdir -p $O
for w in resnet50 gpt2_xl resnet50 gpt2_xl; do
 for pf in "" "--persist-first"; do
  timeout 600 python bench.py --workload $w --steps 40 --warmup 10 $pf --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot --no-union > $O/b.json 2> $O/b.err
  python -c "import json;d=json.load(open('$O/b.json'));print('$w $pf', round(d['ms_per_step'],4), d['per_step_ms'], round(d['gate_bj5']['frac'],3))" || tail -n 5 $O/b.err
 done
done
