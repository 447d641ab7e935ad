"""Correlate per-step device time of compress+exchange with the compress trace (not part of the product).

python tools/spike_probe.py [workload] [steps] [mode]: per step the device time of compress and of
exchange (events around each, synchronised per step), refill levels, DIRECT segments and the
candidates / K ratio; prints the slowest steps and a summary split by 'had a refill'."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
graphs = (sys.argv[3] if len(sys.argv) > 3 else "graphs") == "graphs"
sizes = table(wl)
psi = sum(sizes)
dev = torch.device("cuda", 0)
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model=wl, device=dev) for i in range(4)]
ctx = ld.Context(sizes, density_ppm=10000, optim=ld.ADAM)
K = ctx.K
r = torch.zeros(psi, device=dev)
dense = torch.empty(psi, device=dev)
send = torch.empty(2 * K, dtype=torch.int32, device=dev)
ctx.set_graphs(graphs)
rows = []
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for t in range(30 + steps):
    torch.cuda.synchronize()
    ev[0].record()
    ctx.compress(grads[t % 4], r, send)
    ev[1].record()
    ctx.exchange(send, None, dense)
    ev[2].record()
    torch.cuda.synchronize()
    _, lev, cand, _ = ctx.compress_trace()
    st = ctx.stats()
    if t >= 30:
        rows.append((t, ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3, int((lev == 1).sum()),
                     int((lev == 2).sum()), st["direct_segments"], float(cand.sum()) / K))
a = np.array(rows)
print(f"{wl} graphs={graphs}: compress us p50 {np.median(a[:, 1]):.0f} mean {a[:, 1].mean():.0f} max {a[:, 1].max():.0f};"
      f" exchange us p50 {np.median(a[:, 2]):.0f} mean {a[:, 2].mean():.0f} max {a[:, 2].max():.0f}")
miss = (a[:, 3] + a[:, 4]) > 0
for name, m in (("refill", miss), ("no refill", ~miss)):
    if m.any():
        print(f"  {name}: {m.sum()} steps, compress p50 {np.median(a[m, 1]):.0f} mean {a[m, 1].mean():.0f} us")
dirty = a[:, 5] > 0
for name, m in (("direct>0", dirty & ~miss), ("clean", ~dirty & ~miss)):
    if m.any():
        print(f"  {name}: {m.sum()} steps, compress p50 {np.median(a[m, 1]):.0f} mean {a[m, 1].mean():.0f} us")
print("  slowest: step compress_us exchange_us lvl1 lvl2 direct cand/K")
for row in sorted(rows, key=lambda x: -x[1])[:12]:
    print("   %4d %8.0f %8.0f %4d %4d %6d %6.2f" % row)
print("  fastest:")
for row in sorted(rows, key=lambda x: x[1])[:5]:
    print("   %4d %8.0f %8.0f %4d %4d %6d %6.2f" % row)
