set -u
O=gpurun_out/r3
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:^(small|scan|chunk_prep|find|digit|count|layer_scan|emit|tile_start|merge|update|replay|materialize)" -s 300 -c 60 --csv --log-file $O/launches_resnet.csv \
  python bench.py --workload resnet50 --steps 30 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/ncu_resnet.out 2>&1
tail -n 2 $O/ncu_resnet.out
