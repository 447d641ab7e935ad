# replay check (not product): replay-related GPU tests (incl. the paired-Adam self-test) + the bench's
# recovery legs (100-step GPT-2 XL replay at N=1 and the C4-shape 8-rank leg)
set -u
O=gpurun_out/rp_${1:-x}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -k "replay or ieee or selftest or density_one or recovery or recover or union or fused or sharded or replica" > $O/tests.log 2>&1; tail -n 3 $O/tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union > $O/bench.json 2> $O/bench.err
python -c "import json;d=json.load(open('$O/bench.json'));r=d['recovery'];print('replay', {k: r[k] for k in r if k not in ('sgd','c4_shape')}); print('sgd', r['sgd']); print('c4', r.get('c4_shape'))"
tail -n 2 $O/bench.err
