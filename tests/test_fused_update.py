"""NEXT-1: exchange + optimizer step without a dense gradient (lowdiff_exchange_update).

GPU tests: for Adam and SGD, several iterations of compress -> exchange_update equal, bit for bit,
compress -> exchange (dense G) -> the oracle's Adam/SGD step on the host (Alg. 1 lines 5-8,
PAPER.md:231-237; R-8, R-11, R-12)."""
import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from inputs import gradient, table

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _np(t):
    return t.cpu().numpy().astype(np.float32, copy=False)


@pytest.mark.parametrize("optim,model", [(ld.ADAM, "resnet50"), (ld.SGD, "mlp"), (ld.ADAM, "mlp")])
def test_exchange_update_equals_dense_path(ref, optim, model):
    sizes = table(model)
    psi = sum(sizes)
    ctx = ld.Context(sizes, density_ppm=10000, optim=optim)
    gen = torch.Generator(device=DEV).manual_seed(4)
    p = torch.randn(psi, generator=gen, device=DEV) * 0.05
    m = torch.zeros(psi, device=DEV)
    v = torch.zeros(psi, device=DEV)
    rp, rm, rv = _np(p).copy(), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
    r = torch.zeros(psi, device=DEV)
    send = torch.empty(2 * ctx.K, dtype=torch.int32, device=DEV)
    dense = torch.empty(psi, device=DEV)
    consts = ref.adam_consts()
    for t in range(1, 5):
        g = gradient(sizes, 0, t, dist="D4", model=model, device=DEV)
        ctx.compress(g, r, send)
        ctx.exchange(send, None, dense)
        sc = ld.derive_step_scalars(t, 1e-3)
        ctx.exchange_update(send, None, sc, p, m, v)
        torch.cuda.synchronize()
        G = _np(dense)
        if optim == ld.ADAM:
            ref.adam_step(G, consts, np.array([sc.lr, sc.bc1_inv, sc.bc2_inv], np.float32), rp, rm, rv)
        else:
            ref.sgd_step(G, np.float32(sc.lr), rp)
        assert np.array_equal(_np(p).view(np.uint32), rp.view(np.uint32)), f"iteration {t}"
        if optim == ld.ADAM:
            assert np.array_equal(_np(m).view(np.uint32), rm.view(np.uint32))
            assert np.array_equal(_np(v).view(np.uint32), rv.view(np.uint32))
    ctx.close()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_peer_exchange_equals_gathered_merge(world):
    """Peer-memory exchange (NEXT-1) with `world` ranks simulated on one device (each rank a
    context; peers' slots passed as plain device pointers instead of IPC mappings): over several
    iterations with alternating slots (the write-after-read wait path included), every rank's
    merged G equals lowdiff_merge of the concatenated blocks bit for bit."""
    sizes = table("resnet50")
    psi = sum(sizes)
    ctxs = [ld.Context(sizes, density_ppm=10000, world=world, rank=q) for q in range(world)]
    K = ctxs[0].K
    slots, flags = [], []
    for c in ctxs:
        sl, h = c.peer_alloc(2, handles=False)
        assert h is None and len(sl) == 2 and sl[0].numel() == 2 * K
        slots.append(sl)
        flags.append(c.peer_flags_ptr)
    tbl = [c.peer_ptrs + [c.peer_flags_ptr] for c in ctxs]
    for c in ctxs:
        with pytest.raises(ld.LowDiffError):
            c.exchange_peer(0, torch.empty(psi, device=DEV))   # before peer_set
        c.peer_set(tbl)
        with pytest.raises(ld.LowDiffError):
            c.exchange_peer(0, torch.empty(psi, device=DEV))   # nothing compressed yet
    res = [torch.zeros(psi, device=DEV) for _ in range(world)]
    dense = [torch.empty(psi, device=DEV) for _ in range(world)]
    want = torch.empty(psi, device=DEV)
    for t in range(5):
        sl = t % 2
        for q, c in enumerate(ctxs):
            g = gradient(sizes, q, t, dist="D5", alpha=0.5, model="resnet50", device=DEV)
            c.compress(g, res[q], slots[q][sl])
        for q, c in enumerate(ctxs):
            c.exchange_peer(sl, dense[q])
        gathered = torch.cat([slots[q][sl] for q in range(world)])
        ctxs[0].merge(world, gathered, want)
        torch.cuda.synchronize()
        for q in range(world):
            assert torch.equal(dense[q].view(torch.int32), want.view(torch.int32)), (t, q)
    for c in ctxs:
        c.sync()
    for c in ctxs:
        c.close()
