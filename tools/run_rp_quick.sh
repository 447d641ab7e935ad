# replay quick check (not product): replay parity tests + 100-step probes at world 1 and 8
set -u
O=gpurun_out/rq_${1:-x}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "replay or recover or selftest or ieee or fused or sharded or replica or union" > $O/tests.log 2>&1; tail -n 2 $O/tests.log
for rep in 1 2; do
  timeout 300 python tools/replay_probe.py 100 1 2>&1 | tail -1
  timeout 300 python tools/replay_probe.py 100 8 2>&1 | tail -1
done
