"""Candidates admitted per call relative to K (not product): GPT-2 XL bench inputs, 40 steps (the
stats are per call)."""
import os
import sys

import torch
import paper_2509_04084_b200 as ld
from inputs import gradient, table
sizes = table("gpt2_xl")
psi = sum(sizes)
ctx = ld.Context(sizes, density_ppm=10000)
K = ctx.K
NB = int(sys.argv[1]) if len(sys.argv) > 1 else 2   # distinct gradient buffers, used in rotation
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model="gpt2_xl", device="cuda") for i in range(NB)]
r = torch.zeros(psi, device="cuda")
send = torch.empty(2 * K, dtype=torch.int32, device="cuda")
for t in range(int(os.environ.get("CALLS", "40"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.compress(grads[t % NB], r, send)
    e1.record()
    torch.cuda.synchronize()
    st = ctx.stats()
    print(t, "hits", st["spec_hits"], "misses", st["spec_misses"], "cand/K", round(st["spec_candidates"] / K, 3), "ms", round(e0.elapsed_time(e1), 3))
