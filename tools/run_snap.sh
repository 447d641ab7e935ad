set -u
O=gpurun_out/sn
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "snapshot" > $O/t.log 2>&1; tail -n 2 $O/t.log
timeout 600 python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-union > $O/b.json 2> $O/b.err
python -c "import json;d=json.load(open('$O/b.json'));print(json.dumps(d['snapshot'],indent=0))" || tail -n 5 $O/b.err
