set -u
timeout 900 python -m pytest tests -m gpu -x -q -k "recover or recovery or replica or sharded or union" > gpurun_out/rf_t.log 2>&1; tail -n 3 gpurun_out/rf_t.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-union --no-snapshot --recovery-files 100 > gpurun_out/rf.json 2> gpurun_out/rf.err
python -c "import json;d=json.load(open('gpurun_out/rf.json'));print(d['recovery_files'])" || tail -n 5 gpurun_out/rf.err
