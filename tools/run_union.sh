set -u
O=gpurun_out/u
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_union.py -x -q > $O/union_tests.log 2>&1; tail -n 15 $O/union_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -n 3 $O/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/bench_union.json 2> $O/bench_union.err
python -c "import json;d=json.load(open('$O/bench_union.json'));print(json.dumps(d['union'],indent=1))"
tail -n 3 $O/bench_union.err
