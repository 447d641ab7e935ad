"""Pins of the oracle's union-compacted differentials C^U_t (R-29): the
synchronised compressed gradient G~_t of Alg. 1 line 5-6 kept as an index ->
value dictionary, sharded by parameter range, persisted as .ldu, and replayed.

Pinned against things other than the union code itself: the SPEC worked example of Sync, closed
forms for disjoint and identical supports, Python sets on the index lists, the (separately pinned)
dense exchange, and recovery from the (separately pinned) gathered .ldb chain."""
import os
import struct

import numpy as np
import pytest


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
        out.append(np.concatenate([idx, val.view(np.uint32)]))
    return np.concatenate(out)


def test_sync_worked_example_in_union_form(ref):
    """{0: 2.0} and {3: 4.0} over Psi = 4 -> {0: 1.0, 3: 2.0}; one worker ->
    identity."""
    g = np.array([0, np.float32(2.0).view(np.uint32), 3, np.float32(4.0).view(np.uint32)], np.uint32)
    idx, val = ref.union_compact(g, 2, 1, 4)
    assert idx.tolist() == [0, 3] and val.view(np.float32).tolist() == [1.0, 2.0]
    g1 = np.array([1, 2, np.float32(5.0).view(np.uint32), np.float32(-3.0).view(np.uint32)], np.uint32)
    idx, val = ref.union_compact(g1, 1, 2, 4)
    assert idx.tolist() == [1, 2] and val.view(np.float32).tolist() == [5.0, -3.0]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_disjoint_supports_closed_form(ref, world):
    """Disjoint supports: |U| = N K and every value is v / N (N a power of two: exact scaling)."""
    rng = np.random.default_rng(world)
    psi, K = 4096, 37
    perm = rng.permutation(psi)[: world * K]
    blocks = []
    for r in range(world):
        idx = np.sort(perm[r * K:(r + 1) * K]).astype(np.uint32)
        val = rng.standard_normal(K).astype(np.float32)
        blocks.append((idx, val))
    g = np.concatenate([np.concatenate([i, v.view(np.uint32)]) for i, v in blocks])
    idx, val = ref.union_compact(g, world, K, psi)
    assert idx.size == world * K
    want = {int(i): np.float32(v) * np.float32(1.0 / world) for bi, bv in blocks for i, v in zip(bi, bv)}
    assert idx.tolist() == sorted(want)
    assert np.array_equal(val.view(np.float32), np.array([want[int(i)] for i in idx], np.float32))


def test_identical_supports_closed_form(ref):
    """Two ranks with the same support: |U| = K, value = fl(fl(+0 + a) + b) / 2."""
    rng = np.random.default_rng(5)
    psi, K = 1000, 50
    idx0 = np.sort(rng.choice(psi, K, replace=False)).astype(np.uint32)
    a, b = (rng.standard_normal(K).astype(np.float32) for _ in range(2))
    g = np.concatenate([idx0, a.view(np.uint32), idx0, b.view(np.uint32)])
    idx, val = ref.union_compact(g, 2, K, psi)
    assert np.array_equal(idx, idx0)
    assert np.array_equal(val.view(np.float32), ((np.float32(0) + a) + b) / np.float32(2))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("overlap", [0.0, 0.5, 0.9])
def test_union_is_the_set_union_and_densifies_to_the_exchange(ref, world, overlap):
    rng = np.random.default_rng(100 * world + int(10 * overlap))
    psi, K = 20000, 300
    g = _blocks(rng, world, psi, K, overlap)
    idx, val = ref.union_compact(g, world, K, psi)
    members = set()
    for r in range(world):
        members |= set(g[r * 2 * K:r * 2 * K + K].tolist())
    assert idx.tolist() == sorted(members)                        # Python set union, ascending
    assert idx.size <= world * K
    dense = np.zeros(psi, np.float32)
    dense[idx] = val.view(np.float32)
    G = ref.exchange(g, world, K, psi)
    assert np.array_equal(dense.view(np.uint32), G.view(np.uint32))   # lossless: scatter == Comp^-1
    # sharding: the ranks' shards [floor(r Psi/N), floor((r+1) Psi/N)) concatenate to the whole
    parts = [ref.union_compact(g, world, K, psi, psi * r // world, psi * (r + 1) // world) for r in range(world)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), idx)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), val)
    if overlap == 0.9 and world >= 4:
        assert idx.size < 0.6 * world * K                         # overlapping supports compact


def test_union_capacity_overflow_reports_dim(ref):
    g = np.array([0, 1, 0, 0, 2, 3, 0, 0], np.uint32)             # 2 ranks, K = 2
    lib = ref.lib()
    import ctypes as C
    idx = np.zeros(4, np.uint32)
    val = np.zeros(4, np.uint32)
    cnt = np.zeros(1, np.uint64)
    rc = lib.lowdiff_ref_union_compact(2, 2, 4, g.ctypes.data_as(C.c_void_p), 1, 0, 4,
                                       idx.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p), 3,
                                       cnt.ctypes.data_as(C.c_void_p))
    assert rc == ref.E_DIM and int(cnt[0]) == 4


def test_ldu_layout_parses_by_hand(ref):
    sizes, ppm = [1000, 10, 3000, 7], 10000
    K = sum(ref.k_table(sizes, ppm))
    rng = np.random.default_rng(3)
    unions = [(np.sort(rng.choice(2000, n, replace=False)).astype(np.uint32),
               rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)) for n in (5, 0, 17)]
    scal = np.array([[1e-3, 10.0, 1000.5], [1e-3, 5.26, 500.25], [2e-3, 3.69, 333.6]], np.float32)
    consts = ref.adam_consts()
    data = ref.union_serialize(1, 2, 11, sizes, ppm, ref.ADAM, 3, consts, scal, unions)
    L, psi = len(sizes), sum(sizes)
    assert len(data) == 112 + 16 * L + sum(32 + 8 * len(u[0]) for u in unions) + 4
    head = struct.unpack_from("<4sHHIIQIIQQIIQQQ", data, 0)
    assert head == (b"LDU1", 1, 3, 1, 2, 11, 3, L, psi, K, ppm, 1, psi // 2, psi, 0)
    assert np.array_equal(np.frombuffer(data, np.float32, 5, 80), consts)
    o = 112 + 16 * L
    for it, (ui, uv) in enumerate(unions):
        t, = struct.unpack_from("<Q", data, o)
        cnt, z = struct.unpack_from("<IQ", data, o + 20)
        assert (t, cnt, z) == (11 + it, len(ui), 0)
        assert np.array_equal(np.frombuffer(data, np.float32, 3, o + 8), scal[it])
        assert np.array_equal(np.frombuffer(data, np.uint32, cnt, o + 32), ui)
        assert np.array_equal(np.frombuffer(data, np.uint32, cnt, o + 32 + 4 * cnt), uv)
        o += 32 + 8 * cnt
    assert o + 4 == len(data) and struct.unpack_from("<I", data, o)[0] == ref.crc32c(data[:o])


def live_union(ref, tmp, sizes, ppm, world, T, b, optim, full_at=(0,), lr=1e-2, seed=0):
    """The oracle's training loop writing BOTH forms: every rank's own gathered block (.ldb) and its
    shard of the union-compacted differential (.ldu), batches of b; Full@t for t in full_at."""
    rng = np.random.default_rng(seed)
    psi = sum(sizes)
    K = sum(ref.k_table(sizes, ppm))
    consts = ref.adam_consts()
    flags = ref.FLAG_EF | ref.FLAG_MEAN
    p = rng.standard_normal(psi).astype(np.float32)
    m = np.zeros(psi, np.float32)
    v = np.zeros(psi, np.float32)
    res = [np.zeros(psi, np.float32) for _ in range(world)]
    pend = [[] for _ in range(world)]
    states = {0: (p.copy(), m.copy(), v.copy())}

    def flush(r):
        if not pend[r]:
            return
        first = pend[r][0][0]
        sc = np.stack([x[1] for x in pend[r]])
        with open(os.path.join(tmp, ref.batch_name(r, first)), "wb") as f:
            f.write(ref.batch_serialize(r, world, first, sizes, ppm, optim, flags, consts, sc,
                                       np.stack([x[2] for x in pend[r]])))
        with open(os.path.join(tmp, ref.union_name(r, first)), "wb") as f:
            f.write(ref.union_serialize(r, world, first, sizes, ppm, optim, flags, consts, sc,
                                       [x[3] for x in pend[r]]))
        pend[r] = []

    def full(t):
        for r in range(world):
            with open(os.path.join(tmp, ref.full_name(r, t)), "wb") as f:
                f.write(ref.full_serialize(r, world, t, optim, flags, consts, p, m, v))

    if 0 in full_at:
        full(0)
    sizes_u = 0
    for t in range(1, T + 1):
        sends = []
        for r in range(world):
            g = (rng.standard_normal(psi) * 1e-2).astype(np.float32)
            s, res[r] = ref.compress(sizes, ppm, g, res[r], ef=True)
            sends.append(s)
        gathered = np.concatenate(sends)
        G = ref.exchange(gathered, world, K, psi)
        scal = ref.step_scalars(t, lr)
        if optim == ref.ADAM:
            ref.adam_step(G, consts, scal, p, m, v)
        else:
            ref.sgd_step(G, scal[0], p)
        for r in range(world):
            u = ref.union_compact(gathered, world, K, psi, psi * r // world, psi * (r + 1) // world)
            sizes_u += u[0].size
            pend[r].append((t, scal, sends[r], u))
            if len(pend[r]) == b:
                flush(r)
        if t in full_at:
            full(t)
        states[t] = (p.copy(), m.copy(), v.copy())
    for r in range(world):
        flush(r)
    return states, sizes_u


@pytest.mark.parametrize("optim", [0, 1])
@pytest.mark.parametrize("world,b", [(1, 1), (2, 4), (3, 3), (4, 2)])
def test_recover_union_equals_gathered_recovery_and_live(ref, tmp_path, optim, world, b):
    sizes, ppm, T = [1000, 10, 3000, 7], 20000, 9
    states, n_u = live_union(ref, tmp_path, sizes, ppm, world, T, b, optim, full_at=(0, 5))
    K = sum(ref.k_table(sizes, ppm))
    assert n_u <= T * world * K
    for target in (-1, 9, 7, 5, 4, 1, 0):
        pu, mu, vu, got = ref.recover_union(tmp_path, world, sizes, ppm, target)
        pg, mg, vg, got_g = ref.recover(tmp_path, world, sizes, ppm, target)
        want_t = T if target == -1 else target
        assert got == got_g == want_t
        P, M, V = states[want_t]
        assert np.array_equal(pu.view(np.uint32), pg.view(np.uint32)) and np.array_equal(pu, P)
        if optim == ref.ADAM:
            assert np.array_equal(mu, M) and np.array_equal(vu, V)


def test_recover_union_gap_and_corruption(ref, tmp_path):
    sizes, ppm, world = [1000, 10, 3000, 7], 20000, 2
    live_union(ref, tmp_path, sizes, ppm, world, 8, 2, ref.ADAM)
    assert ref.recover_union(tmp_path, world, sizes, ppm, -1)[3] == 8
    os.remove(os.path.join(tmp_path, ref.union_name(1, 5)))
    assert ref.recover_union(tmp_path, world, sizes, ppm, -1)[3] == 4
    with pytest.raises(ref.OracleError) as e:
        ref.recover_union(tmp_path, world, sizes, ppm, 6)
    assert e.value.code == ref.E_GAP
    path = os.path.join(tmp_path, ref.union_name(0, 3))
    data = bytearray(open(path, "rb").read())
    data[150] ^= 0x04
    open(path, "wb").write(bytes(data))
    with pytest.raises(ref.OracleError) as e:
        ref.recover_union(tmp_path, world, sizes, ppm, 4)
    assert e.value.code == ref.E_CORRUPT
