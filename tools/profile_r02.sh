#!/bin/bash
# Round-2 profiling pass on a GPU box (run under gpurun from the repo root); outputs in gpurun_out/.
# Not part of the product.  1) GPU tests, 2) the default bench line (and ResNet-50),
# 3) the ncu launch list of a short bench command, 4) ncu --set full of the top kernels
# (one launch each, steady state: call 21 of the step loop).
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r02}
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/${TAG}_gpu_tests.log 2>&1; tail -n 3 $OUT/${TAG}_gpu_tests.log
fi
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; tail -2 $OUT/${TAG}_bench.err
timeout 300 python bench.py --workload resnet50 --steps 200 --no-cpu --no-snapshot --no-replica --no-full \
    > $OUT/${TAG}_bench_resnet50.json 2> $OUT/${TAG}_bench_resnet50.err
[ "${SKIP_NCU:-0}" = 1 ] && exit 0
SHORT="python bench.py --steps 4 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-c4-shape --replay-steps 10"
# our kernels only (the gradient generator's launches are torch's), steady state
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k "regex:^(small|scan|refill|chunk_prep|find|digit|count|tile_start|merge|update|replay|materialize|union)" \
    -s 300 -c 200 --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 12 --warmup 24 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-c4-shape --replay-steps 10 \
    > $OUT/${TAG}_launches.out 2>&1
tail -2 $OUT/${TAG}_launches.out
# per call: 1 scan, 1 chunk_prep, 1 refill, 2 find, 1 digit, 1 count_emit -> skip 20 = call 21
for ks in scan_kernel:20 count_emit_kernel:20 chunk_prep_kernel:20 digit_kernel:20 merge_kernel:20 update_kernel:4 replay_kernel:1; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$k -s $skip -c 1 -o $OUT/${TAG}_prof_$k $SHORT \
      > $OUT/${TAG}_p_$k.out 2>&1
  tail -1 $OUT/${TAG}_p_$k.out
done
