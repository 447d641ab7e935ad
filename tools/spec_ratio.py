"""Candidates admitted per call relative to K (not product): GPT-2 XL bench inputs, 40 steps (the
stats are per call)."""
import torch
import paper_2509_04084_b200 as ld
from inputs import gradient, table
sizes = table("gpt2_xl")
psi = sum(sizes)
ctx = ld.Context(sizes, density_ppm=10000)
K = ctx.K
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model="gpt2_xl", device="cuda") for i in range(2)]
r = torch.zeros(psi, device="cuda")
send = torch.empty(2 * K, dtype=torch.int32, device="cuda")
for t in range(40):
    ctx.compress(grads[t % 2], r, send)
    torch.cuda.synchronize()
    st = ctx.stats()
    print(t, "hits", st["spec_hits"], "misses", st["spec_misses"], "cand/K", round(st["spec_candidates"] / K, 3))
