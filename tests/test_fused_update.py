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
# multi-rank peer tests: several tiles, chunks and small layers, but an oracle compress in ~0.1 s
PEER_SIZES = [300000, 5000, 1048576, 70001, 4096, 600000, 7]


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
def test_peer_exchange_equals_gathered_merge(ref, world):
    """Peer-memory exchange (NEXT-1) with `world` ranks simulated on one device (each rank a
    context; peers' slots passed as plain device pointers instead of IPC mappings): over several
    iterations with alternating slots (the write-after-read wait path included), every rank's
    merged G equals the oracle's exchange (R-8) of the oracle's own compressed blocks bit for bit
    (and lowdiff_merge of the concatenated slots)."""
    sizes = PEER_SIZES
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
    R = [np.zeros(psi, np.float32) for _ in range(world)]
    for t in range(5):
        sl = t % 2
        blocks = []
        for q, c in enumerate(ctxs):
            g = gradient(sizes, q, t, dist="D5", alpha=0.5, device=DEV)
            c.compress(g, res[q], slots[q][sl])
            b, R[q] = ref.compress(sizes, 10000, _np(g), R[q], ef=True)
            blocks.append(b)
        for q, c in enumerate(ctxs):
            c.exchange_peer(sl, dense[q])
        gathered = torch.cat([slots[q][sl] for q in range(world)])
        ctxs[0].merge(world, gathered, want)
        torch.cuda.synchronize()
        G = ref.exchange(np.concatenate(blocks), world, K, psi)
        for q in range(world):
            assert np.array_equal(_np(dense[q]).view(np.uint32), G.view(np.uint32)), (t, q)
            assert torch.equal(dense[q].view(torch.int32), want.view(torch.int32)), (t, q)
    for c in ctxs:
        c.sync()
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("world,optim", [(1, ld.ADAM), (2, ld.ADAM), (3, ld.SGD), (4, ld.ADAM), (8, ld.ADAM),
                                         (8, ld.SGD)])
def test_peer_update_equals_oracle(ref, world, optim):
    """NEXT-1 fully fused (lowdiff_exchange_peer_update): every simulated rank reads all ranks'
    entries of each tile from their slots, merges them in shared memory and applies the step to its
    own p, m, v -- no gathered buffer, no dense G.  Every rank's p, m, v equal, bit for bit, the
    oracle's exchange (R-8) of its own compressed blocks followed by its Adam (R-11) / SGD (R-12)
    step, over several iterations with alternating slots and stored per-step scalars."""
    sizes = PEER_SIZES
    psi = sum(sizes)
    ctxs = [ld.Context(sizes, density_ppm=10000, world=world, rank=q, optim=optim) for q in range(world)]
    K = ctxs[0].K
    slots = []
    for c in ctxs:
        sl, _ = c.peer_alloc(2, handles=False)
        slots.append(sl)
    tbl = [c.peer_ptrs + [c.peer_flags_ptr] for c in ctxs]
    for c in ctxs:
        c.peer_set(tbl)
    gen = torch.Generator(device=DEV).manual_seed(9)
    p0 = torch.randn(psi, generator=gen, device=DEV) * 0.05
    ps = [p0.clone() for _ in range(world)]
    ms = [torch.zeros(psi, device=DEV) for _ in range(world)]
    vs = [torch.zeros(psi, device=DEV) for _ in range(world)]
    P, M, V = _np(p0).copy(), np.zeros(psi, np.float32), np.zeros(psi, np.float32)
    res = [torch.zeros(psi, device=DEV) for _ in range(world)]
    R = [np.zeros(psi, np.float32) for _ in range(world)]
    for t in range(1, 6):
        sl = t % 2
        blocks = []
        for q, c in enumerate(ctxs):
            g = gradient(sizes, q, t, dist="D5", alpha=0.5, device=DEV)
            c.compress(g, res[q], slots[q][sl])
            b, R[q] = ref.compress(sizes, 10000, _np(g), R[q], ef=True)
            blocks.append(b)
        sc = ld.derive_step_scalars(t, 1e-3 if optim == ld.ADAM else 0.1)
        for q, c in enumerate(ctxs):
            c.exchange_peer_update(sl, sc, ps[q], ms[q], vs[q])
        torch.cuda.synchronize()
        G = ref.exchange(np.concatenate(blocks), world, K, psi)
        scal = np.array([sc.lr, sc.bc1_inv, sc.bc2_inv], np.float32)
        if optim == ld.ADAM:
            ref.adam_step(G, ref.adam_consts(), scal, P, M, V)
        else:
            ref.sgd_step(G, scal[0], P)
        for q in range(world):
            assert np.array_equal(_np(ps[q]).view(np.uint32), P.view(np.uint32)), (t, q)
            if optim == ld.ADAM:
                assert np.array_equal(_np(ms[q]).view(np.uint32), M.view(np.uint32)), (t, q)
                assert np.array_equal(_np(vs[q]).view(np.uint32), V.view(np.uint32)), (t, q)
    for c in ctxs:
        c.sync()
    for c in ctxs:
        c.close()
