"""NEXT-2: sharded recovery (the exact per-element replay of DESIGN.md R-16 split by parameter range
over ranks; Alg. 1 recovery).

GPU tests: lowdiff_replay_range over any element range equals the same slice of the full fused
replay bit for bit (tile-aligned, unaligned, one element, ranges inside one tile, whole Psi), and
lowdiff_recover_sharded on simulated ranks (one process, no communicator, gather = 0) reproduces
the oracle's live state on every rank's shard, touching nothing outside it."""
import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from test_gpu_parity import oracle_live

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _diffs(sizes, world, T, ppm=10000, seed=1):
    """T steps of `world` ranks' send blocks from the GPU compressor (each rank its own residual)."""
    psi = sum(sizes)
    ctx = ld.Context(sizes, density_ppm=ppm)
    gen = torch.Generator(device=DEV).manual_seed(seed)
    res = [torch.zeros(psi, device=DEV) for _ in range(world)]
    out = torch.empty(T, world, 2 * ctx.K, dtype=torch.int32, device=DEV)
    for t in range(T):
        for r in range(world):
            g = torch.randn(psi, generator=gen, device=DEV) * 1e-2
            ctx.compress(g, res[r], out[t, r])
    torch.cuda.synchronize()
    ctx.close()
    return out


@pytest.mark.parametrize("optim,world", [(ld.ADAM, 3), (ld.ADAM, 1), (ld.SGD, 4)])
def test_replay_range_equals_full_replay(optim, world):
    sizes = [70001, 1600, 50000, 7, 9000]
    psi = sum(sizes)
    T = 9
    diffs = _diffs(sizes, world, T)
    scal = [ld.derive_step_scalars(t, 1e-2) for t in range(1, T + 1)]
    ctx = ld.Context(sizes, density_ppm=10000)
    gen = torch.Generator(device=DEV).manual_seed(3)
    p0 = torch.randn(psi, generator=gen, device=DEV)
    m0 = torch.randn(psi, generator=gen, device=DEV) * 1e-3
    v0 = torch.rand(psi, generator=gen, device=DEV) * 1e-4
    P, M, V = p0.clone(), m0.clone(), v0.clone()
    ctx.replay(optim, world, T, diffs, scal, P, M, V)
    torch.cuda.synchronize()
    ranges = [(0, psi), (0, 2048), (2048, 4096), (1, 2), (2047, 2049), (100, 1900), (12345, 99999),
              (psi - 1, psi), (psi // 3, 2 * psi // 3), (70001, 71601)]
    for a, b in ranges:
        p, m, v = p0[a:b].clone(), m0[a:b].clone(), v0[a:b].clone()
        ctx.replay_range(optim, world, T, diffs, scal, a, b, p, m if optim == ld.ADAM else None,
                         v if optim == ld.ADAM else None)
        torch.cuda.synchronize()
        assert np.array_equal(_u32(p), _u32(P[a:b])), (a, b)
        if optim == ld.ADAM:
            assert np.array_equal(_u32(m), _u32(M[a:b])) and np.array_equal(_u32(v), _u32(V[a:b])), (a, b)
    ctx.replay_range(optim, world, T, diffs, scal, 5, 5, p0[5:5])   # empty range: no-op
    with pytest.raises(ld.LowDiffError):
        ctx.replay_range(optim, world, T, diffs, scal, 10, psi + 1, p0, m0, v0)
    ctx.close()


@pytest.mark.parametrize("world,b", [(3, 2), (4, 3)])
def test_recover_sharded_simulated_ranks(ref, tmp_path, world, b):
    """The oracle writes a `world`-rank checkpoint; each simulated rank recovers only its shard into
    a NaN-filled full-size buffer; the union of the shards is the oracle's live state at every
    target, and each rank leaves the other shards untouched."""
    sizes, ppm, T = [30001, 1600, 50000, 7], 10000, 7
    psi = sum(sizes)
    gen = torch.Generator(device="cpu").manual_seed(0)
    p0 = torch.randn(psi, generator=gen).numpy()
    rng = np.random.default_rng(5)
    grads = [[(rng.standard_normal(psi) * 1e-2).astype(np.float32) for _ in range(world)] for _ in range(T)]
    states = oracle_live(ref, sizes, ppm, world, grads, ld.ADAM, str(tmp_path), b, (0, 3), 1e-2, p0)
    ranks = [ld.Context(sizes, density_ppm=ppm, ckpt_dir=str(tmp_path), world=world, rank=r) for r in range(world)]
    for target in (-1, 2, 5):
        want_t = T if target == -1 else target
        P, M, V = states[want_t]
        q, mq, vq = (torch.full((psi,), float("nan"), device=DEV) for _ in range(3))
        for r, c in enumerate(ranks):
            lo, hi = psi * r // world, psi * (r + 1) // world
            alone = torch.full((psi,), float("nan"), device=DEV)
            ma, va = alone.clone(), alone.clone()
            assert c.recover_sharded(alone, ma, va, target=target, gather=False) == want_t
            assert torch.isnan(alone[:lo]).all() and torch.isnan(alone[hi:]).all()
            assert np.array_equal(_u32(alone[lo:hi]), P[lo:hi].view(np.uint32))
            assert c.recover_sharded(q, mq, vq, target=target, gather=False) == want_t
        assert np.array_equal(_u32(q), P.view(np.uint32))
        assert np.array_equal(_u32(mq), M.view(np.uint32))
        assert np.array_equal(_u32(vq), V.view(np.uint32))
    with pytest.raises(ld.LowDiffError):
        ranks[0].recover_sharded(q, mq, vq, gather=True)       # gather needs a communicator
    for c in ranks:
        c.close()


def test_full_ckpt_staged_write_after_read(ref, tmp_path):
    """D2D-staged full checkpoint: the update enqueued right after lowdiff_full_ckpt
    on the producer stream overwrites p, m, v, yet the shard files hold the state at the call
    (the producer waits for the stage), byte-identical to the oracle's serialisation."""
    sizes = [1 << 22, 4096, 3 << 20]
    psi = sum(sizes)
    world = 2
    gen = torch.Generator(device=DEV).manual_seed(8)
    p = torch.randn(psi, generator=gen, device=DEV)
    m = torch.randn(psi, generator=gen, device=DEV)
    v = torch.rand(psi, generator=gen, device=DEV)
    want = [x.cpu().numpy().copy() for x in (p, m, v)]
    ctxs = [ld.Context(sizes, density_ppm=10000, ckpt_dir=str(tmp_path), world=world, rank=r) for r in range(world)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for c in ctxs:
            c.full_ckpt(5, p, m, v, stream=s)
        for x in (p, m, v):          # the next "update", on the producer stream
            x.mul_(-3.0).add_(1.0)
    torch.cuda.synchronize()
    for c in ctxs:
        c.sync()
    consts = ref.adam_consts()
    for r in range(world):
        got = open(tmp_path / ref.full_name(r, 5), "rb").read()
        exp = ref.full_serialize(r, world, 5, ref.ADAM, ref.FLAG_EF | ref.FLAG_MEAN, consts, *want)
        assert got == exp
    for c in ctxs:
        c.close()
