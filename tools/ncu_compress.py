"""Drive lowdiff_compress for ncu (diagnostic): N calls on D4 gradients (4 buffers in rotation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_04084_b200 as ld  # noqa: E402
from inputs import gradient, table  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2_xl"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 24
sizes = table(wl)
ctx = ld.Context(sizes, density_ppm=10000)
grads = [gradient(sizes, 0, i, dist="D4", alpha=0.5, model=wl, device="cuda") for i in range(4)]
r = torch.zeros(sum(sizes), device="cuda")
send = torch.empty(2 * ctx.K, dtype=torch.int32, device="cuda")
for t in range(calls):
    ctx.compress(grads[t % 4], r, send)
torch.cuda.synchronize()
print("done", ctx.stats()["spec_misses"])
