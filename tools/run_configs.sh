# Config lines for profiles/ (not product): C2 ResNet-50, C3 BERT-large, the C4 density sweep, and
# the peer-exchange GPT-2 XL line (NEXT-1 fused update)
set -u
O=gpurun_out/cfg_${1:-r02}
mkdir -p $O
for w in resnet50 bert_large; do
  timeout 600 python bench.py --workload $w --steps 200 --no-cpu --no-writer --no-replica --no-snapshot > $O/$w.json 2> $O/$w.err
done
for ppm in 1000 2500 5000; do
  timeout 600 python bench.py --ppm $ppm --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union > $O/gpt2_$ppm.json 2> $O/gpt2_$ppm.err
done
timeout 600 python bench.py --exchange peer --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-recovery > $O/gpt2_peer.json 2> $O/gpt2_peer.err
tail -n 2 $O/*.err
