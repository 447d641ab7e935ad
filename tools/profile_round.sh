#!/bin/bash
# One profiling pass on a GPU box (run under gpurun from the repo root); outputs in gpurun_out/.
# Not part of the product.  1) the bench line, 2) the ncu launch list of a short bench command,
# 3) ncu --set full of the top kernels (one launch each, steady state).
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/p_gpu_tests.log 2>&1; tail -n 2 $OUT/p_gpu_tests.log
python bench.py --steps 20 --warmup 8 > $OUT/p_bench.json 2> $OUT/p_bench.err
tail -2 $OUT/p_bench.err
SHORT="python bench.py --steps 4 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --replay-steps 10"
# our kernels only (the gradient generator's launches are torch's), steady state: skip the first 400
# (~23 calls: the EF residual and the speculative band settle over the first ~10, see tools/spec_ratio.py)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k "regex:^(small|scan|chunk_prep|find|digit|count|tile_start|merge|update|replay|materialize|union)" \
    -s 400 -c 200 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 12 --warmup 24 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --replay-steps 10 \
    > $OUT/p_launches.out 2>&1
tail -2 $OUT/p_launches.out
# skips land on call 21 of the step loop (3 scan / chunk_prep launches per call: main + 2 refill levels)
for ks in scan_kernel:63 merge1_kernel:21 update_kernel:4 replay_kernel:1 count_emit_kernel:21 chunk_prep_kernel:63 union_tile_kernel:2; do
  k=${ks%%:*}; skip=${ks##*:}
  ncu --set full --clock-control none --import-source on -k regex:^$k -s $skip -c 1 -o $OUT/prof_$k $SHORT \
      > $OUT/p_$k.out 2>&1
  tail -1 $OUT/p_$k.out
done
