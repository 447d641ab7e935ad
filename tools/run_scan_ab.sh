# scan A/B (not product): compress parity subset, then the GPT-2 XL / ResNet-50 step with variants
# tools/run_scan_ab.sh TAG v1 v2 ... ("default" = in-tree build)
set -u
TAG=$1; shift
O=gpurun_out/sab_$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "compress or full_size or graph_replay" > $O/tests.log 2>&1; tail -n 2 $O/tests.log
B="--steps 50 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot --no-union --trace-calls 0"
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/tools/variants/$v/liblowdiff.so; fi
  for w in gpt2_xl resnet50; do
    timeout 600 python bench.py --workload $w $B > $O/$w.$v.json 2> $O/$w.$v.err
    python -c "import json;d=json.load(open('$O/$w.$v.json'));print('$v $w', round(d['ms_per_step'],4), d['per_step_ms']['p50'], {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items() if k in ('scan','select','emit','merge')})"
  done
done; done
