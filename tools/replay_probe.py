"""Replay timing / ncu driver (diagnostic): n steps of GPT-2 XL blocks at 1% (world ranks' blocks per
step over this rank's 1/world range, like bench.py's recovery leg)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
optim = ld.SGD if (len(sys.argv) > 3 and sys.argv[3] == "sgd") else ld.ADAM
sizes = table("gpt2_xl")
psi = sum(sizes)
ctx = ld.Context(sizes, density_ppm=10000)
K = ctx.K
g = [gradient(sizes, q, 0, dist="D4", alpha=0.5, model="gpt2_xl", device="cuda") for q in range(2)]
r = torch.zeros(psi, device="cuda")
blk = torch.empty((world, 2 * K), dtype=torch.int32, device="cuda")
for q in range(world):   # distinct blocks per rank (the residual evolves)
    ctx.compress(g[q % 2], r, blk[q])
diffs = blk.reshape(1, -1).expand(n, -1).contiguous()
lo, hi = 0, psi // world
p = torch.randn(hi - lo, device="cuda") * 0.02
m = torch.zeros(hi - lo, device="cuda")
v = torch.zeros(hi - lo, device="cuda")
sc = [ld.derive_step_scalars(t, 1e-3) for t in range(1, n + 1)]
ctx.replay_range(optim, world, n, diffs, sc, lo, hi, p, m, v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.replay_range(optim, world, n, diffs, sc, lo, hi, p, m, v)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"replay n={n} world={world} {'sgd' if optim == ld.SGD else 'adam'}: {ms:.2f} ms, "
      f"{n * (hi - lo) / ms / 1e9:.3f} T param-steps/s")
