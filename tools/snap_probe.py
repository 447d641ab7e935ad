"""Probe: slowdown of an HBM-bound proxy backward while gradient buckets stream D2H (not product).

  python tools/snap_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import table  # noqa: E402

sizes = table("gpt2_xl")
psi = sum(sizes)
plan = ld.bucket_plan(sizes, 4 << 20)
offs = [0]
for n in sizes:
    offs.append(offs[-1] + n)
g = torch.randn(psi, device="cuda")
scratch = torch.empty(max(offs[f + c] - offs[f] for f, c in plan), device="cuda")
host = torch.empty(psi, pin_memory=True)
side = torch.cuda.Stream()
ctx = ld.Context(sizes, density_ppm=10000)


def run(mode, reps=20, it=[10]):
    it[0] += 1
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    e0.record()
    if mode == "one_big":
        with torch.cuda.stream(side):
            host.copy_(g, non_blocking=True)
    for f, c in plan:
        a, b = offs[f], offs[f + c]
        for _ in range(reps):
            torch.mul(g[a:b], 1.0, out=scratch[:b - a])
        if mode == "torch_d2h":
            ev = torch.cuda.Event()
            ev.record()
            side.wait_event(ev)
            with torch.cuda.stream(side):
                host[a:b].copy_(g[a:b], non_blocking=True)
        elif mode == "lowdiff":
            ctx.snapshot_layer(it[0], f, c, g[a:b])
    e1.record()
    torch.cuda.current_stream().wait_stream(side)
    if mode == "lowdiff":
        ctx.wait_persist()
    e2.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), e0.elapsed_time(e2)


for mode in ["alone", "torch_d2h", "lowdiff", "one_big", "alone", "lowdiff", "torch_d2h"]:
    r = [run(mode) for _ in range(3)]
    print(f"{mode:10s} backward {min(x[0] for x in r):8.2f} ms   all done {min(x[1] for x in r):8.2f} ms", flush=True)
for reps in (0, 1, 5):
    for mode in ["alone", "lowdiff"]:
        r = [run(mode, reps) for _ in range(3)]
        print(f"reps={reps} {mode:10s} backward {min(x[0] for x in r):8.2f} ms   all done {min(x[1] for x in r):8.2f} ms",
              flush=True)
