set -u
O=gpurun_out/r3
mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery > $O/snap_gpt2.json 2> $O/snap_gpt2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 60 --csv --log-file $O/launches_resnet.csv \
  python bench.py --workload resnet50 --steps 30 --warmup 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery --no-snapshot > $O/ncu_resnet.out 2>&1
tail -2 $O/*.err $O/ncu_resnet.out
