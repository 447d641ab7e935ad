# level-1 drop variants (not product): per-call compress ms over 62 calls, 2 and 8 rotating buffers
set -u
for v in default tools/variants/l1_22 tools/variants/l1_23; do
  if [ "$v" = default ]; then unset LOWDIFF_LIB; else export LOWDIFF_LIB=$PWD/$v/liblowdiff.so; fi
  for nb in 2 8; do
    PYTHONPATH=. CALLS=62 timeout 600 python tools/spec_ratio.py $nb > gpurun_out/l1.txt
    python -c "
import sys
ms=[float(l.split()[-1]) for l in open('gpurun_out/l1.txt')][8:]
print('$v nb=$nb sum(8..61) %.2f ms  max %.2f  calls>4ms %d' % (sum(ms), max(ms), sum(m > 4 for m in ms)))"
  done
  timeout 600 python bench.py --steps 20 --no-cpu --no-e2e --no-writer --no-replica --no-full --no-update --no-snapshot --no-union --no-recovery > gpurun_out/l1b.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/l1b.json'));print('$v bench', round(d['ms_per_step'],4), d['per_step_ms']['p50'])"
done
