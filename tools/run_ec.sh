# early-clear check (not product; needs tools/ab/early_clear.patch applied): parity tests + bench A/B with and without the overlapped clear
set -u
O=gpurun_out/ec_${1:-x}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "early_clear or merge_parity or exchange_world1 or graph_replay or gpt2_xl_full" > $O/tests.log 2>&1; tail -n 3 $O/tests.log
B="--steps 50 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot --no-union"
for w in gpt2_xl resnet50; do
  for v in "1" "2" "4" "off"; do
    if [ $v = off ]; then X="--no-early-clear"; else X=""; export LOWDIFF_CLEAR_CTAS=$v; fi
    timeout 600 python bench.py --workload $w $B $X > $O/$w$v.json 2> $O/$w$v.err
    python -c "import json;d=json.load(open('$O/$w$v.json'));print('$w $v', round(d['ms_per_step'],4), d['per_step_ms']['p50'], {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}, round(d['gate_bj5']['frac'],3))"
  done
done
