# kernel variants (not product): replay timings with each build
set -u
for v in default tools/variants/sgd12 tools/variants/sgd16; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/$v/liblowdiff.so; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));r=d['recovery'];print('$v', round(r['ms'],2), 'sgd', round(r['sgd']['ms'],2))"
done
