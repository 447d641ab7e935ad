set -u
O=gpurun_out/bc
mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 5 --exchange peer --no-cpu --no-e2e --no-writer --no-replica --no-full --no-snapshot --no-union --no-recovery > $O/peer.json 2> $O/peer.err
python -c "import json;d=json.load(open('$O/peer.json'));print('peer', round(d['ms_per_step'],4), {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()}, d['update'])" || tail -n 5 $O/peer.err
timeout 900 python bench.py > $O/default.json 2> $O/default.err
python -c "
import json;d=json.load(open('$O/default.json'))
print('default', round(d['value'],1), round(d['ms_per_step'],4), d['per_step_ms'], d['clocks'], d['gpu_launches'])
print(d['recovery']['ms'], d['recovery']['sgd'])
print(d['cpu_baseline'])" || tail -n 5 $O/default.err
