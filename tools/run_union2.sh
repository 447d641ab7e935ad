set -u
O=gpurun_out/u2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_union.py -x -q > $O/t.log 2>&1; tail -n 3 $O/t.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/b.json 2> $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));u=d['union'];print({k:(u[k]['ms'],u[k]['entries'],round(u[k]['algorithmic_gbs'])) for k in ('shard0','all')})"
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_union.py -x -q -k "compact_parity and (True-0.9-3 or False-0.0-8)" > $O/san.log 2>&1; tail -n 2 $O/san.log
