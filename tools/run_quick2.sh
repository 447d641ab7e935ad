set -u
O=gpurun_out/q2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -n 3 $O/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union > $O/bench.json 2> $O/bench.err
python -c "import json;d=json.load(open('$O/bench.json'));r=d['recovery'];print('replay', r['ms'], r['replay_kernel_ms'], r['value'])"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:^replay_kernel -s 1 -c 1 -o $O/replay python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --replay-steps 10 > $O/ncu.out 2>&1; tail -n 1 $O/ncu.out
