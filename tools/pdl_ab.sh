set -u
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_tests.log 2>&1; tail -n 3 gpurun_out/pdl_tests.log
for p in 0 1 0 1; do
  LOWDIFF_PDL=$p timeout 300 python bench.py --workload resnet50 --steps 50 --warmup 20 --no-cpu --no-writer --no-replica --no-snapshot --no-recovery --no-full --no-update --no-e2e > gpurun_out/pdl_res_$p.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pdl_res_$p.json').read().strip().splitlines()[-1]);print('res pdl=$p',d['ms_per_step'],d['per_step_ms']['p50'],d['gate_bj5']['frac'])"
  LOWDIFF_PDL=$p timeout 300 python bench.py --steps 20 --warmup 8 --no-cpu --no-writer --no-replica --no-snapshot --no-recovery --no-full --no-update --no-e2e > gpurun_out/pdl_gpt_$p.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/pdl_gpt_$p.json').read().strip().splitlines()[-1]);print('gpt pdl=$p',d['ms_per_step'],d['per_step_ms']['p50'])"
done
