"""Per-call phase breakdown of lowdiff_compress's select kernel (diagnostic; needs a GPU).

python tools/phase_probe.py [workload] [calls] [ppm]: compresses D4 gradients (4 buffers in rotation,
like bench.py) and prints, per call, the select kernel's phase durations (us) and the refill trace."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2_xl"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ppm = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
sizes = table(wl)
psi = sum(sizes)
ctx = ld.Context(sizes, density_ppm=ppm)
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model=wl, device="cuda") for i in range(4)]
r = torch.zeros(psi, device="cuda")
send = torch.empty(2 * ctx.K, dtype=torch.int32, device="cuda")
names = ["hist0", "plan", "rs1", "pl1", "rs2", "pl2", "d1", "f1", "d2", "f2", "count", "-", "-", "-", "emit"]
print("call  total_us  " + " ".join("%6s" % n for n in names) + "   lvl1 lvl2 direct cand/K")
for t in range(calls):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.compress(grads[t % 4], r, send)
    e1.record()
    torch.cuda.synchronize()
    ph = ctx.compress_phases()
    _, lev, cand, thr = ctx.compress_trace()
    st = ctx.stats()
    d = []
    last = ph[0]
    for i in range(1, 16):
        if ph[i] == 0:
            d.append(0.0)
            continue
        d.append((ph[i] - last) / 1e3)
        last = ph[i]
    print("%4d %9.1f  " % (t, e0.elapsed_time(e1) * 1e3) + " ".join("%6.1f" % x for x in d[:15]) +
          "   %4d %4d %6d %5.2f" % ((lev == 1).sum(), (lev == 2).sum(), st["direct_segments"],
                                 cand.astype(np.float64).sum() / ctx.K))
