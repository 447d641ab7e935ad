set -u
O=gpurun_out/r2
mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-recovery > $O/snap_gpt2.json 2> $O/snap_gpt2.err
for w in resnet50 bert_large; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 20 --no-cpu --no-writer --no-replica --no-snapshot > $O/$w.json 2> $O/$w.err
done
for ppm in 1000 2500 5000; do
  timeout 600 python bench.py --ppm $ppm --steps 20 --warmup 8 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --replay-steps 100 > $O/gpt2_$ppm.json 2> $O/gpt2_$ppm.err
done
tail -n 3 $O/*.err
