# compute-sanitizer memcheck / racecheck on small GPU cases (not product)
set -u
O=gpurun_out/san
mkdir -p $O
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_memcheck.log 2>&1; tail -n 3 $O/smoke_memcheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_union.py -x -q -k "compact_parity and (True-0.9-3 or False-0.0-8 or True-0.0-1) or persist_files_and_recover and 2-3" > $O/union_memcheck.log 2>&1; tail -n 3 $O/union_memcheck.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "compress_mlp or compress_resnet50 or multi_rank_recovery or drift_reversal or merge_parity or graph or corruption" > $O/parity_memcheck.log 2>&1; tail -n 3 $O/parity_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "multi_rank_recovery or compress_resnet50_speculation" > $O/race.log 2>&1; tail -n 3 $O/race.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_union.py -x -q -k "compact_parity and True-0.9-3" > $O/race_union.log 2>&1; tail -n 3 $O/race_union.log
