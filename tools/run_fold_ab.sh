# find-fold A/B (not product): GPU suite on the default build, then default vs tools/variants/prefold
set -u
timeout 1200 python -m pytest tests -m gpu -x -q -k "smoke" > gpurun_out/scan_tests.log 2>&1; tail -n 3 gpurun_out/scan_tests.log
for v in default tools/variants/prefold default tools/variants/prefold; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/$v/liblowdiff.so; fi
  timeout 600 python bench.py --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --no-recovery > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));print('$v gpt', round(d['ms_per_step'],4), d['per_step_ms']['p50'], d['roofline']['frac'], {k: round(x['ms_per_launch'],4) for k,x in d['kernels'].items()})"
  timeout 600 python bench.py --workload resnet50 --steps 50 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --no-recovery > gpurun_out/var.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/var.json'));print('$v res', round(d['ms_per_step'],4), d['per_step_ms']['p50'], d['roofline']['frac'])"
done
