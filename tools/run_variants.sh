# kernel variants (not product): compress chain timings with each build
set -u
for v in default tools/variants/sw2 tools/variants/sw8 tools/variants/sw16 default; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/$v/liblowdiff.so; fi
  timeout 600 python bench.py --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --no-recovery > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));print('$v', round(d['ms_per_step'],4), {k: round(x['ms_per_launch'],4) for k,x in d['kernels'].items()})"
done
