set -u
O=gpurun_out/rp
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "replay or ieee or density_one or recovery or union or fused or sharded" > $O/tests.log 2>&1; tail -n 3 $O/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union > $O/bench.json 2> $O/bench.err
python -c "import json;d=json.load(open('$O/bench.json'));r=d['recovery'];print('replay', r['ms'], r['replay_kernel_ms'], r['value'], 'sgd', r['sgd']['ms'])"
tail -n 2 $O/bench.err
