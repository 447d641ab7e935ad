# launch lists (not product) of our kernels for two workloads, steady state
set -u
O=gpurun_out/ll
mkdir -p $O
K="regex:^(small|scan|chunk_prep|find|digit|count|tile_start|merge|update|replay|materialize|union)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 300 -c 40 --csv --log-file $O/resnet.csv \
  python bench.py --workload resnet50 --steps 30 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/resnet.out 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 150 -c 40 --csv --log-file $O/gpt2.csv \
  python bench.py --steps 12 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/gpt2.out 2>&1
