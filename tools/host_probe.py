"""Host-side enqueue cost vs device step time of the bench loop (not part of the product).

python tools/host_probe.py [workload] [steps] -> per-step host enqueue time (perf_counter around
step()) and device time (events), p10/p50/p90/max, and the same with persist off / graphs off."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
sizes = table(wl)
psi = sum(sizes)
dev = torch.device("cuda", 0)
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model=wl, device=dev) for i in range(4)]


def run(persist=True, graphs=True, sync_every=0):
    ctx = ld.Context(sizes, density_ppm=10000, ckpt_dir="/tmp/hp", batch_size=4, ring_slots=8, write_files=False,
                     optim=ld.ADAM)
    K = ctx.K
    r = torch.zeros(psi, device=dev)
    dense = torch.empty(psi, device=dev)
    sends = [torch.empty(2 * K, dtype=torch.int32, device=dev) for _ in range(2)]
    scal = [ld.derive_step_scalars(t, 1e-3) for t in range(1, 30 + steps + 2)]
    ctx.set_graphs(graphs)
    it = [0]

    def step():
        t = it[0]
        sd = sends[t % 2]
        ctx.compress(grads[t % 4], r, sd)
        ctx.exchange(sd, None, dense)
        if persist:
            ctx.batch_persist(t + 1, scal[t], sd)
        it[0] += 1

    for _ in range(30):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    host = []
    ev[0].record()
    for i in range(steps):
        h0 = time.perf_counter()
        step()
        host.append((time.perf_counter() - h0) * 1e6)
        ev[i + 1].record()
        if sync_every and (i + 1) % sync_every == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    dt = np.array([ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(steps)])
    host = np.array(host)
    q = lambda a: "p10 %.0f p50 %.0f p90 %.0f max %.0f mean %.1f" % (np.percentile(a, 10), np.percentile(a, 50),
                                                                     np.percentile(a, 90), a.max(), a.mean())
    print(f"persist={persist} graphs={graphs} sync_every={sync_every}\n  host us: {q(host)}\n  dev  us: {q(dt)}",
          flush=True)
    ctx.close()


run()
run(persist=False)
run(graphs=False)
run(sync_every=1)
run()
