# kernel variants (not product): compress chain timings with each build
set -u
for v in default tools/variants/pf16 tools/variants/pf12 tools/variants/pf10 default tools/variants/pf16; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/$v/liblowdiff.so; fi
  timeout 600 python bench.py --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --no-recovery > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));print('$v', round(d['ms_per_step'],4), d['per_step_ms']['p50'], {k: round(x['ms_per_launch'],4) for k,x in d['kernels'].items()})"
done
