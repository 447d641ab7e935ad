"""Diagnostic (not part of the product): per-iteration behaviour of lowdiff_compress on a model
table -- speculative-band candidates per k, hits/misses, and per-kernel device times.

  python tools/spec_probe.py [model] [ppm] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "gpt2_xl"
ppm = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 25
sizes = table(model)
psi = sum(sizes)
ctx = ld.Context(sizes, density_ppm=ppm)
K_large = sum(ctx.layer_k(l)[0] for l, n in enumerate(sizes) if n > 16384)
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model=model, device="cuda") for i in range(2)]
r = torch.zeros(psi, device="cuda")
send = torch.empty(2 * ctx.K, dtype=torch.int32, device="cuda")
print(f"{model} psi={psi} K={ctx.K} K_large={K_large}")
for it in range(iters):
    ctx.prof_enable(True)
    ctx.compress(grads[it % 2], r, send)
    t = {n: ctx.prof_read(n)[0] for n in ("small_layer", "scan", "select", "emit")}
    st = ctx.stats()
    print(f"it {it:3d} cand/K_large {st['spec_candidates'] / max(1, K_large):6.3f} hits {st['spec_hits']:4d} "
          f"misses {st['spec_misses']:4d} | " + " ".join(f"{k} {v:.3f}" for k, v in t.items()) + " ms")
ctx.close()
