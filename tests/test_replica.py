"""NEXT-3: LowDiff+ CPU replica (§5.2; Alg. 2 l.11-13).

CPU tests: the product's host optimizer (lowdiff_host_adam_step / lowdiff_host_sgd_step) against
the oracle's Adam/SGD steps bit for bit, on ordinary, special (zeros, subnormals, huge, negative
zero) and many-thread inputs.  The oracle's steps are pinned in test_oracle_exchange_optim.py.

GPU tests: the context-level replica (snapshot -> worker -> host optimizer) against the device
replay of the same differentials, bit for bit; the persisted replica equals the oracle's .ldf of
the same state byte for byte and lowdiff_recover accepts it as a full checkpoint; restore copies
it back; sharded replicas of a 2-rank job persist shards that recover to the full state."""
import os

import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from paper_2509_04084_b200 import lowdiff as B


def _consts_np(c):
    return np.array([c.beta1, c.one_minus_beta1, c.beta2, c.one_minus_beta2, c.eps], np.float32)


def _scal_np(s):
    return np.array([s.lr, s.bc1_inv, s.bc2_inv], np.float32)


def _special(n, rng):
    vals = np.array([0.0, -0.0, 1e-45, -1e-45, 1e-38, 3e38, -3e38, 1.0, -1.0, 1e-8, 65504.0], np.float32)
    x = (rng.standard_normal(n) * 10.0 ** rng.integers(-30, 10, n)).astype(np.float32)
    pick = rng.random(n) < 0.2
    x[pick] = rng.choice(vals, int(pick.sum()))
    return x


@pytest.mark.parametrize("threads", [1, 3, 8])
@pytest.mark.parametrize("n", [1, 17, 4099, 300001])
def test_host_adam_bitwise_vs_oracle(ref, n, threads):
    rng = np.random.default_rng(n * 7 + threads)
    consts = B.derive_adam_consts(0.9, 0.999, 1e-8)
    p0 = _special(n, rng)
    m0 = _special(n, rng)
    v0 = np.abs(_special(n, rng))
    for t in (1, 2, 37):
        scal = B.derive_step_scalars(t, 1e-3)
        G = _special(n, rng)
        p, m, v = p0.copy(), m0.copy(), v0.copy()
        B.host_adam_step(G, consts, scal, p, m, v, threads=threads)
        rp, rm, rv = p0.copy(), m0.copy(), v0.copy()
        ref.adam_step(G, _consts_np(consts), _scal_np(scal), rp, rm, rv)
        for got, want in ((p, rp), (m, rm), (v, rv)):
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), \
                f"t={t}: {int(np.sum(got.view(np.uint32) != want.view(np.uint32)))} words differ"


def test_host_adam_many_steps_and_sgd(ref):
    """50 Adam steps chained (state feeds back, so one mis-rounded op anywhere compounds) and SGD."""
    n = 65537
    rng = np.random.default_rng(11)
    consts = B.derive_adam_consts(0.9, 0.999, 1e-8)
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    for t in range(1, 51):
        G = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        G[rng.random(n) < 0.9] = 0.0        # sparse-like merged gradients
        scal = B.derive_step_scalars(t, 1e-2)
        B.host_adam_step(G, consts, scal, p, m, v, threads=4)
        ref.adam_step(G, _consts_np(consts), _scal_np(scal), rp, rm, rv)
    assert np.array_equal(p.view(np.uint32), rp.view(np.uint32))
    assert np.array_equal(m.view(np.uint32), rm.view(np.uint32))
    assert np.array_equal(v.view(np.uint32), rv.view(np.uint32))
    q = rng.standard_normal(n).astype(np.float32)
    rq = q.copy()
    G = rng.standard_normal(n).astype(np.float32)
    B.host_sgd_step(G, 0.05, q, threads=3)
    ref.sgd_step(G, np.float32(0.05), rq)
    assert np.array_equal(q.view(np.uint32), rq.view(np.uint32))


def test_host_step_argument_errors():
    with pytest.raises(ld.LowDiffError):
        B._check("host_adam_step", B.lib().lowdiff_host_adam_step(5, None, None, None, None, None, None, 1))
    with pytest.raises(ld.LowDiffError):
        B._check("host_sgd_step", B.lib().lowdiff_host_sgd_step(-1, None, 0.1, None, 1))
    assert B.lib().lowdiff_host_sgd_step(0, None, 0.1, None, 1) == 0


# ------------------------------------------------------------------------------------------ GPU
DEV = "cuda"


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _run_job(ctx, sizes, T, lr, seed, p, m, v, snap_dev=None, on_step=None):
    """T LowDiff+ iterations on one rank: compress -> merge (world 1) -> dense G_t -> snapshot ->
    device replay of the same differential.  Returns the differential blocks."""
    psi = sum(sizes)
    gen = torch.Generator(device=DEV).manual_seed(seed)
    r = torch.zeros(psi, device=DEV)
    send = torch.empty(2 * ctx.K, dtype=torch.int32, device=DEV)
    G = torch.empty(psi, device=DEV)
    for t in range(1, T + 1):
        g = torch.randn(psi, generator=gen, device=DEV) * 1e-2
        ctx.compress(g, r, send)
        ctx.merge(1, send, G)
        ctx.snapshot_layer(t, 0, len(sizes), G)
        ctx.wait_persist()      # G is rewritten next iteration: order that after the D2H copy
        scal = B.derive_step_scalars(t, lr)
        ctx.replay(ld.ADAM, 1, 1, send, [scal], p, m, v)
        if on_step:
            on_step(t, scal)
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("threads", [1, 6])
def test_replica_equals_device_replay(ref, tmp_path, threads):
    """The replica advanced from snapshots equals the GPU state after T steps, bit for bit; its
    persisted shard equals the oracle's .ldf of that state byte for byte; recover() and
    replica_restore() both reproduce it.  A large model with 1 thread makes the worker lag, so the
    snapshot back-pressure (t + 2 waits for t) is exercised."""
    sizes = [1 << 20, 3000, 2 << 20, 77, 1 << 20] if threads == 1 else [30000, 1600, 50000, 7]
    T, lr = 12, 1e-2
    psi = sum(sizes)
    ctx = ld.Context(sizes, density_ppm=10000, ckpt_dir=str(tmp_path), write_files=True)
    gen = torch.Generator(device=DEV).manual_seed(5)
    p = torch.randn(psi, generator=gen, device=DEV)
    m = torch.zeros(psi, device=DEV)
    v = torch.zeros(psi, device=DEV)
    ctx.replica_init(0, p, m, v, threads=threads)

    def step(t, scal):
        ctx.replica_step(t, scal)
        if t == 7:
            ctx.replica_persist()

    _run_job(ctx, sizes, T, lr, 9, p, m, v, on_step=step)
    it, rp, rm, rv, sb, se = ctx.replica_wait()
    assert (it, sb, se) == (T, 0, psi)
    assert np.array_equal(rp.numpy().view(np.uint32), _u32(p))
    assert np.array_equal(rm.numpy().view(np.uint32), _u32(m))
    assert np.array_equal(rv.numpy().view(np.uint32), _u32(v))
    if threads == 1:
        assert ctx.stats()["replica_busy_ns"] > 0
    ctx.replica_persist()
    ctx.replica_wait()
    ctx.sync()
    consts = _consts_np(B.derive_adam_consts())
    want = ref.full_serialize(0, 1, T, ref.ADAM, ref.FLAG_EF | ref.FLAG_MEAN, consts, rp.numpy(), rm.numpy(), rv.numpy())
    got = open(os.path.join(tmp_path, ref.full_name(0, T)), "rb").read()
    assert got == want
    assert os.path.exists(os.path.join(tmp_path, ref.full_name(0, 7)))
    # the replica file serves as the full checkpoint of a recovery (no differentials after T)
    q, mq, vq = (torch.empty(psi, device=DEV) for _ in range(3))
    assert ctx.recover(q, mq, vq) == T
    assert torch.equal(q, p) and torch.equal(mq, m) and torch.equal(vq, v)
    # software failure: device state lost, restore from the in-memory replica
    for a in (q, mq, vq):
        a.fill_(float("nan"))
    assert ctx.replica_restore(q, mq, vq) == T
    assert torch.equal(q, p) and torch.equal(mq, m) and torch.equal(vq, v)
    ctx.close()


@pytest.mark.gpu
def test_replica_state_errors(tmp_path):
    sizes = [4096, 100]
    ctx = ld.Context(sizes, density_ppm=10000)
    psi = sum(sizes)
    p, m, v = (torch.zeros(psi, device=DEV) for _ in range(3))
    with pytest.raises(ld.LowDiffError):
        ctx.replica_step(1, B.derive_step_scalars(1, 1e-3))     # no replica
    ctx.replica_init(3, p, m, v, threads=2)
    with pytest.raises(ld.LowDiffError):
        ctx.replica_step(5, B.derive_step_scalars(5, 1e-3))     # not the next iteration
    with pytest.raises(ld.LowDiffError):
        ctx.replica_step(4, B.derive_step_scalars(4, 1e-3))     # iteration 4 never snapshotted
    g = torch.ones(psi, device=DEV)
    ctx.snapshot_layer(4, 0, 1, g[:4096])
    with pytest.raises(ld.LowDiffError):
        ctx.replica_step(4, B.derive_step_scalars(4, 1e-3))     # layer 1 missing
    ctx.snapshot_layer(4, 1, 1, g[4096:])
    ctx.replica_step(4, B.derive_step_scalars(4, 1e-3))
    it = ctx.replica_wait()[0]
    assert it == 4
    with pytest.raises(ld.LowDiffError):
        ctx.replica_persist()                                   # no ckpt_dir
    ctx.close()


@pytest.mark.gpu
def test_sharded_replicas_recover_full_state(ref, tmp_path):
    """world = 2 (no communicator: both ranks simulated in one process).  Each rank's replica holds
    its shard floor(r Psi / 2) .. floor((r+1) Psi / 2), advanced from the same synced gradients;
    the two persisted shards recover to the full device state."""
    sizes = [30001, 1600, 50000, 7]
    psi = sum(sizes)
    T, lr = 5, 1e-2
    dev = ld.Context(sizes, density_ppm=10000)
    gen = torch.Generator(device=DEV).manual_seed(2)
    p = torch.randn(psi, generator=gen, device=DEV)
    m = torch.zeros(psi, device=DEV)
    v = torch.zeros(psi, device=DEV)
    ranks = [ld.Context(sizes, density_ppm=10000, world=2, rank=r, ckpt_dir=str(tmp_path)) for r in range(2)]
    for c in ranks:
        c.replica_init(0, p, m, v, threads=2)
    r = torch.zeros(psi, device=DEV)
    send = torch.empty(2 * dev.K, dtype=torch.int32, device=DEV)
    G = torch.empty(psi, device=DEV)
    g2 = torch.Generator(device=DEV).manual_seed(4)
    for t in range(1, T + 1):
        g = torch.randn(psi, generator=g2, device=DEV) * 1e-2
        dev.compress(g, r, send)
        dev.merge(1, send, G)
        scal = B.derive_step_scalars(t, lr)
        for c in ranks:
            c.snapshot_layer(t, 0, len(sizes), G)
            c.wait_persist()
            c.replica_step(t, scal)
        dev.replay(ld.ADAM, 1, 1, send, [scal], p, m, v)
    torch.cuda.synchronize()
    for rk, c in enumerate(ranks):
        it, rp, rm, rv, sb, se = c.replica_wait()
        assert (it, sb, se) == (T, psi * rk // 2, psi * (rk + 1) // 2)
        assert np.array_equal(rp.numpy().view(np.uint32), _u32(p[sb:se]))
        assert np.array_equal(rv.numpy().view(np.uint32), _u32(v[sb:se]))
        c.replica_persist()
        c.replica_wait()
        c.sync()
        with pytest.raises(ld.LowDiffError):
            c.replica_restore(p, m, v)      # world > 1 needs a communicator
    q, mq, vq = (torch.empty(psi, device=DEV) for _ in range(3))
    assert ranks[0].recover(q, mq, vq) == T
    assert torch.equal(q, p) and torch.equal(mq, m) and torch.equal(vq, v)
    for c in ranks + [dev]:
        c.close()
