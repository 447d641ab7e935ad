"""GPU parity of the union-compacted differentials (R-29) through the C ABI:
lowdiff_union_compact against the oracle's union_compact bit for bit, the .ldu files written by
lowdiff_union_persist byte-identical to the oracle's serializer, and lowdiff_recover_union (all
shards, and per-rank sharded) equal to the oracle's live training states."""
import os

import numpy as np
import pytest
import torch

import paper_2509_04084_b200 as ld
from inputs import gradient

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _blocks(rng, world, psi, K, overlap):
    shared = rng.choice(psi, size=K, replace=False)
    out = []
    for _ in range(world):
        own = rng.choice(psi, size=K, replace=False)
        idx = np.unique(np.where(rng.random(K) < overlap, shared, own))
        while idx.size < K:
            idx = np.unique(np.concatenate([idx, rng.choice(psi, size=K - idx.size, replace=False)]))
        idx = np.sort(idx[:K]).astype(np.uint32)
        val = rng.standard_normal(K).astype(np.float32)
        val[rng.random(K) < 0.05] = -0.0
        out.append(np.concatenate([idx, val.view(np.uint32)]))
    return np.concatenate(out)


def gpu_union(ctx, world, gathered_np, lo, hi):
    g = torch.from_numpy(gathered_np.view(np.int32)).to(DEV)
    cap = max(1, min(world * ctx.K, hi - lo))
    out = torch.full((2 * cap,), -1, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    ctx.union_compact(world, g, lo, hi, out, cap, cnt)
    torch.cuda.synchronize()
    n = int(cnt.item())
    o = out.cpu().numpy().view(np.uint32)
    return o[:n].copy(), o[cap:cap + n].copy()


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("overlap", [0.0, 0.9])
@pytest.mark.parametrize("mean", [True, False])
def test_union_compact_parity(ref, world, overlap, mean):
    sizes = [100000, 77777, 5, 40000]        # 217782 elements: 27 tiles and a ragged tail
    psi = sum(sizes)
    ctx = ld.Context(sizes, density_ppm=30000, mean=mean)
    K = ctx.K
    rng = np.random.default_rng(world * 11 + int(overlap * 10) + int(mean))
    gathered = _blocks(rng, world, psi, K, overlap)
    ranges = [(0, psi)] + [(psi * r // world, psi * (r + 1) // world) for r in range(world)] + [(8191, 8193), (5, 5)]
    for lo, hi in ranges:
        gi, gv = gpu_union(ctx, world, gathered, lo, hi)
        wi, wv = ref.union_compact(gathered, world, K, psi, lo, hi, mean=mean)
        assert np.array_equal(gi, wi), (lo, hi, gi.size, wi.size)
        assert np.array_equal(gv, wv), (lo, hi)
    ctx.close()


def test_union_compact_of_real_compressions(ref):
    """ResNet-50 table, 4 simulated ranks with rank-correlated gradients (D5, alpha = 0.9): the GPU
    compresses, the union of the 4 send blocks compacts to well under 4 K entries."""
    from inputs import table
    sizes, ppm, world = table("resnet50"), 10000, 4
    psi = sum(sizes)
    ctx = ld.Context(sizes, density_ppm=ppm)
    K = ctx.K
    sends = []
    for r in range(world):
        g = gradient(sizes, r, 0, dist="D5", alpha=0.9, model="resnet50", device=DEV)
        s = torch.empty(2 * K, dtype=torch.int32, device=DEV)
        ctx.compress(g, torch.zeros(psi, device=DEV), s)
        sends.append(s)
    torch.cuda.synchronize()
    gathered = torch.cat(sends).cpu().numpy().view(np.uint32)
    for r in range(world):
        lo, hi = psi * r // world, psi * (r + 1) // world
        gi, gv = gpu_union(ctx, world, gathered, lo, hi)
        wi, wv = ref.union_compact(gathered, world, K, psi, lo, hi)
        assert np.array_equal(gi, wi) and np.array_equal(gv, wv)
    gi, _ = gpu_union(ctx, world, gathered, 0, psi)
    assert gi.size < 0.8 * world * K
    ctx.close()


def test_union_compact_rejects_small_cap():
    sizes = [5000, 3000]
    ctx = ld.Context(sizes, density_ppm=10000)
    g = torch.zeros(2 * 2 * ctx.K, dtype=torch.int32, device=DEV)
    out = torch.empty(2 * ctx.K, dtype=torch.int32, device=DEV)
    cnt = torch.zeros(1, dtype=torch.int64, device=DEV)
    with pytest.raises(ld.LowDiffError):
        ctx.union_compact(2, g, 0, 8000, out, ctx.K, cnt)   # worst case is 2 K
    ctx.close()


def _oracle_live(ref, sizes, ppm, world, T, lr, seed):
    """The oracle's training loop: per-iteration gathered blocks, scalars and states (Adam)."""
    rng = np.random.default_rng(seed)
    psi = sum(sizes)
    K = sum(ref.k_table(sizes, ppm))
    consts = ref.adam_consts()
    p = rng.standard_normal(psi).astype(np.float32)
    m = np.zeros(psi, np.float32)
    v = np.zeros(psi, np.float32)
    res = [np.zeros(psi, np.float32) for _ in range(world)]
    states = {0: (p.copy(), m.copy(), v.copy())}
    gath, scals = {}, {}
    for t in range(1, T + 1):
        sends = []
        for r in range(world):
            g = (rng.standard_normal(psi) * 1e-2).astype(np.float32)
            s, res[r] = ref.compress(sizes, ppm, g, res[r], ef=True)
            sends.append(s)
        gath[t] = np.concatenate(sends)
        scals[t] = ref.step_scalars(t, lr)
        ref.adam_step(ref.exchange(gath[t], world, K, psi), consts, scals[t], p, m, v)
        states[t] = (p.copy(), m.copy(), v.copy())
    return states, gath, scals


@pytest.mark.parametrize("world,b", [(1, 2), (2, 3), (3, 4), (8, 2)])
def test_union_persist_files_and_recover(ref, tmp_path, world, b):
    sizes, ppm, T, lr = [30000, 1600, 50000, 7], 10000, 7, 1e-2
    psi = sum(sizes)
    states, gath, scals = _oracle_live(ref, sizes, ppm, world, T, lr, seed=world)
    d = str(tmp_path)
    flags = ref.FLAG_EF | ref.FLAG_MEAN
    consts = ref.adam_consts()
    for r in range(world):   # Full@0 by the oracle (the GPU path's .ldf bytes are tested elsewhere)
        with open(os.path.join(d, ref.full_name(r, 0)), "wb") as f:
            f.write(ref.full_serialize(r, world, 0, ref.ADAM, flags, consts, *states[0]))
    ctxs = [ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=r, batch_size=b, optim=ld.ADAM)
            for r in range(world)]
    for t in range(1, T + 1):
        gd = torch.from_numpy(gath[t].view(np.int32)).to(DEV)
        sc = ld.derive_step_scalars(t, lr)
        assert np.array_equal(np.array([sc.lr, sc.bc1_inv, sc.bc2_inv], np.float32), scals[t])
        for r in range(world):
            ctxs[r].union_persist(t, sc, gd)
    K = ctxs[0].K
    for r in range(world):
        ctxs[r].sync()
        st = ctxs[r].stats()
        assert st["union_files_written"] == (T + b - 1) // b
        lo, hi = psi * r // world, psi * (r + 1) // world
        # byte-identical to the oracle's serialisation of the same batches
        for first in range(1, T + 1, b):
            its = list(range(first, min(T, first + b - 1) + 1))
            unions = [ref.union_compact(gath[t], world, K, psi, lo, hi) for t in its]
            want = ref.union_serialize(r, world, first, sizes, ppm, ref.ADAM, flags, consts,
                                       np.stack([scals[t] for t in its]), unions)
            got = open(os.path.join(d, ref.union_name(r, first)), "rb").read()
            assert got == want, (r, first)
    for c in ctxs:
        c.close()
    # recovery: all shards on one GPU, and each rank's shard alone
    rc = ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=0, optim=ld.ADAM)
    for target in (-1, T, 3, 1, 0):
        q, mq, vq = (torch.full((psi,), 5.0, device=DEV) for _ in range(3))
        got_t = rc.recover_union(q, mq, vq, target=target)
        want_t = T if target == -1 else target
        assert got_t == want_t
        P, M, V = states[want_t]
        assert np.array_equal(q.cpu().numpy(), P) and np.array_equal(mq.cpu().numpy(), M)
        assert np.array_equal(vq.cpu().numpy(), V)
        po, mo, vo, to = ref.recover_union(d, world, sizes, ppm, target)
        assert to == want_t and np.array_equal(po, P)
    rc.close()
    for r in range(world):
        sc_ctx = ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=r, optim=ld.ADAM)
        q, mq, vq = (torch.full((psi,), 5.0, device=DEV) for _ in range(3))
        assert sc_ctx.recover_union(q, mq, vq, sharded=True) == T
        lo, hi = psi * r // world, psi * (r + 1) // world
        P, M, V = states[T]
        qn = q.cpu().numpy()
        assert np.array_equal(qn[lo:hi], P[lo:hi]) and np.array_equal(vq.cpu().numpy()[lo:hi], V[lo:hi])
        assert np.all(qn[:lo] == 5.0) and np.all(qn[hi:] == 5.0)      # nothing outside the shard
        sc_ctx.close()


def test_union_recover_gap(ref, tmp_path):
    sizes, ppm, T, lr, world = [30000, 1600, 50000, 7], 10000, 6, 1e-2, 2
    psi = sum(sizes)
    states, gath, scals = _oracle_live(ref, sizes, ppm, world, T, lr, seed=9)
    d = str(tmp_path)
    flags = ref.FLAG_EF | ref.FLAG_MEAN
    for r in range(world):
        with open(os.path.join(d, ref.full_name(r, 0)), "wb") as f:
            f.write(ref.full_serialize(r, world, 0, ref.ADAM, flags, ref.adam_consts(), *states[0]))
    ctxs = [ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=r, batch_size=2, optim=ld.ADAM)
            for r in range(world)]
    for t in range(1, T + 1):
        gd = torch.from_numpy(gath[t].view(np.int32)).to(DEV)
        for r in range(world):
            ctxs[r].union_persist(t, ld.derive_step_scalars(t, lr), gd)
    with pytest.raises(ld.LowDiffError) as e:   # FIFO: iterations must be consecutive
        ctxs[0].union_persist(T + 2, ld.derive_step_scalars(T + 2, lr), gd)
    assert e.value.code == ld.lowdiff.E_STATE
    for c in ctxs:
        c.close()
    os.remove(os.path.join(d, ref.union_name(1, 3)))
    rc = ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=0, optim=ld.ADAM)
    q, mq, vq = (torch.empty(psi, device=DEV) for _ in range(3))
    assert rc.recover_union(q, mq, vq) == 2
    assert np.array_equal(q.cpu().numpy(), states[2][0])
    with pytest.raises(ld.LowDiffError) as e:
        rc.recover_union(q, mq, vq, target=5)
    assert e.value.code == ld.lowdiff.E_GAP
    rc.close()


@pytest.mark.parametrize("world,b", [(1, 3), (2, 4), (4, 2)])
def test_accumulated_batch_mode_files_and_recover(ref, tmp_path, world, b):
    """Accumulated batch mode (R-30): the writer's tensor addition of each batch's dictionaries gives
    .ldu files byte-identical to the oracle's accumulate + accum_serialize; recovery (all shards and
    sharded) equals the oracle's recover_union over the same files -- and, for b > 1, differs from
    the live state (the mode is inexact by construction).  A mode switch mid-run writes the batch in
    flight in the old mode; the mixed chain recovers like the oracle."""
    sizes, ppm, T, lr = [30000, 1600, 50000, 7], 10000, 9, 1e-2
    psi = sum(sizes)
    states, gath, scals = _oracle_live(ref, sizes, ppm, world, T, lr, seed=20 + world)
    d = str(tmp_path)
    flags = ref.FLAG_EF | ref.FLAG_MEAN
    consts = ref.adam_consts()
    for r in range(world):
        with open(os.path.join(d, ref.full_name(r, 0)), "wb") as f:
            f.write(ref.full_serialize(r, world, 0, ref.ADAM, flags, consts, *states[0]))
    ctxs = [ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=r, batch_size=b, optim=ld.ADAM)
            for r in range(world)]
    switch_at = T - 1          # iterations T-1, T go in record mode (the accumulated batch in flight is cut)
    for c in ctxs:
        c.set_batch_mode(ld.BATCH_ACCUMULATED)
    for t in range(1, T + 1):
        gd = torch.from_numpy(gath[t].view(np.int32)).to(DEV)
        if t == switch_at:
            for c in ctxs:
                c.set_batch_mode(ld.BATCH_RECORD)
        for r in range(world):
            ctxs[r].union_persist(t, ld.derive_step_scalars(t, lr), gd)
    K = ctxs[0].K
    batches = [list(range(f, min(switch_at - 1, f + b - 1) + 1)) for f in range(1, switch_at, b)]
    for r in range(world):
        ctxs[r].sync()
        lo, hi = psi * r // world, psi * (r + 1) // world
        for its in batches:
            acc = ref.accumulate([ref.union_compact(gath[t], world, K, psi, lo, hi) for t in its])
            want = ref.accum_serialize(r, world, its[0], len(its), sizes, ppm, ref.ADAM, flags, consts,
                                       scals[its[-1]], acc)
            got = open(os.path.join(d, ref.union_name(r, its[0])), "rb").read()
            assert got == want, (r, its)
        rec = [ref.union_compact(gath[t], world, K, psi, lo, hi) for t in (switch_at, T)]
        want = ref.union_serialize(r, world, switch_at, sizes, ppm, ref.ADAM, flags, consts,
                                   np.stack([scals[switch_at], scals[T]]), rec)
        assert open(os.path.join(d, ref.union_name(r, switch_at)), "rb").read() == want
    for c in ctxs:
        c.close()
    ends = [its[-1] for its in batches] + [switch_at, T]
    rc = ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=0, optim=ld.ADAM)
    for target in [-1, 0] + ends:
        q, mq, vq = (torch.full((psi,), 5.0, device=DEV) for _ in range(3))
        got_t = rc.recover_union(q, mq, vq, target=target)
        po, mo, vo, to = ref.recover_union(d, world, sizes, ppm, target)
        assert got_t == to == (T if target == -1 else target)
        assert np.array_equal(q.cpu().numpy(), po) and np.array_equal(mq.cpu().numpy(), mo)
        assert np.array_equal(vq.cpu().numpy(), vo)
        if b > 1 and to >= b:
            assert not np.array_equal(po, states[to][0])      # inexact (R-30)
    inner = [t for t in range(1, switch_at) if t not in ends]
    for target in inner[:2]:
        with pytest.raises(ld.LowDiffError) as e:
            rc.recover_union(q, mq, vq, target=target)
        assert e.value.code == ld.lowdiff.E_GAP
    rc.close()
    po, _, vo, _ = ref.recover_union(d, world, sizes, ppm, -1)
    for r in range(world):
        sc_ctx = ld.Context(sizes, density_ppm=ppm, ckpt_dir=d, world=world, rank=r, optim=ld.ADAM)
        q, mq, vq = (torch.full((psi,), 5.0, device=DEV) for _ in range(3))
        assert sc_ctx.recover_union(q, mq, vq, sharded=True) == T
        lo, hi = psi * r // world, psi * (r + 1) // world
        qn = q.cpu().numpy()
        assert np.array_equal(qn[lo:hi], po[lo:hi]) and np.array_equal(vq.cpu().numpy()[lo:hi], vo[lo:hi])
        assert np.all(qn[:lo] == 5.0) and np.all(qn[hi:] == 5.0)
        sc_ctx.close()
