# round-start validation (not product): full GPU suite, smoke, default bench line
set -u
O=gpurun_out/v_${1:-x}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -n 3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench exit $?
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['ms_per_step'], d.get('roofline'), d.get('clocks'))"
