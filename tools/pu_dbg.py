import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2509_04084_b200 as ld
from inputs import gradient, table
world, optim = int(sys.argv[1]), (ld.SGD if sys.argv[2] == "sgd" else ld.ADAM)
sizes = table("resnet50"); psi = sum(sizes)
ctxs = [ld.Context(sizes, density_ppm=10000, world=world, rank=q, optim=optim) for q in range(world)]
slots = [c.peer_alloc(2, handles=False)[0] for c in ctxs]
tbl = [c.peer_ptrs + [c.peer_flags_ptr] for c in ctxs]
for c in ctxs: c.peer_set(tbl)
ps = [torch.zeros(psi, device="cuda") for _ in range(world)]
ms = [torch.zeros(psi, device="cuda") for _ in range(world)]
vs = [torch.zeros(psi, device="cuda") for _ in range(world)]
res = [torch.zeros(psi, device="cuda") for _ in range(world)]
for t in range(1, 6):
    sl = t % 2
    for q, c in enumerate(ctxs):
        g = gradient(sizes, q, t, dist="D5", alpha=0.5, model="resnet50", device="cuda")
        c.compress(g, res[q], slots[q][sl]); torch.cuda.synchronize(); print("c", t, q, flush=True)
    sc = ld.derive_step_scalars(t, 0.1)
    for q, c in enumerate(ctxs):
        c.exchange_peer_update(sl, sc, ps[q], ms[q], vs[q]); torch.cuda.synchronize(); print("u", t, q, flush=True)
for c in ctxs: c.sync()
print("ok")
