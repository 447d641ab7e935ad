"""Pins of the oracle's checkpoint files (PAPER.md:276-282 batched writing; Save(M_t) PAPER.md:245)
and of its recovery (Alg. 1 recovery process; Eq. 2)."""
import os
import struct

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_crc32c_check_value(ref):
    with open(os.path.join(GOLD, "crc32c_check.txt")) as f:
        rows = [ln for ln in f if ln.strip() and not ln.startswith("#")]
    for ln in rows:
        data, want = (c.strip() for c in ln.split("|"))
        assert ref.crc32c(data.encode()) == int(want, 16)
    assert ref.crc32c(b"") == 0


def _sizes():
    return [1000, 10, 3000, 7]


def test_batch_layout_parses_by_hand(ref):
    sizes, ppm = _sizes(), 10000
    K = sum(ref.k_table(sizes, ppm))
    rng = np.random.default_rng(1)
    blocks = rng.integers(0, 2**32, size=(3, 2 * K), dtype=np.uint64).astype(np.uint32)
    scal = np.array([[1e-3, 10.0, 1000.5], [1e-3, 5.26, 500.25], [2e-3, 3.69, 333.6]], np.float32)
    consts = ref.adam_consts()
    data = ref.batch_serialize(2, 4, 41, sizes, ppm, ref.ADAM, ref.FLAG_EF | ref.FLAG_MEAN, consts, scal, blocks)
    L = len(sizes)
    assert len(data) == 96 + 16 * L + 3 * (32 + 8 * K) + 4 == ref.batch_bytes(L, K, 3)
    magic, ver, flags, rank, world, first, n_it, nl, psi, kk, p, opt, rsv = struct.unpack_from("<4sHHIIQIIQQIIQ", data, 0)
    assert (magic, ver, flags, rank, world, first, n_it, nl, psi, kk, p, opt, rsv) == \
        (b"LDB1", 1, 3, 2, 4, 41, 3, L, sum(sizes), K, ppm, 1, 0)
    assert np.array_equal(np.frombuffer(data, np.float32, 5, 64), consts)
    for l in range(L):
        n, k, z = struct.unpack_from("<QII", data, 96 + 16 * l)
        assert (n, k, z) == (sizes[l], ref.k_of(sizes[l], ppm), 0)
    o = 96 + 16 * L
    for it in range(3):
        t, = struct.unpack_from("<Q", data, o)
        assert t == 41 + it
        assert np.array_equal(np.frombuffer(data, np.float32, 3, o + 8), scal[it])
        assert np.array_equal(np.frombuffer(data, np.uint32, 2 * K, o + 32), blocks[it])
        o += 32 + 8 * K
    crc, = struct.unpack_from("<I", data, o)
    assert o + 4 == len(data) and crc == ref.crc32c(data[:o])


def test_full_layout_and_size_law(ref):
    rng = np.random.default_rng(2)
    psi = 1003
    p, m, v = (rng.standard_normal(psi).astype(np.float32) for _ in range(3))
    consts = ref.adam_consts()
    shards = []
    for r in range(3):
        data = ref.full_serialize(r, 3, 7, ref.ADAM, 3, consts, p, m, v)
        sb, se = psi * r // 3, psi * (r + 1) // 3
        S = se - sb
        assert len(data) == 96 + 12 * S + 4       # 3 Psi payload, 12 B/param
        hdr = struct.unpack_from("<4sHHIIQQQQIIQ", data, 0)
        assert hdr == (b"LDF1", 1, 3, r, 3, 7, psi, sb, se, 1, 0, 0)
        body = np.frombuffer(data, np.float32, 3 * S, 96)
        assert np.array_equal(body, np.concatenate([p[sb:se], m[sb:se], v[sb:se]]))
        shards.append((sb, se))
    assert shards[0][0] == 0 and shards[-1][1] == psi
    # SGD full checkpoints carry zero moments (one layout)
    d = ref.full_serialize(0, 1, 0, ref.SGD, 1, consts, p)
    assert not np.frombuffer(d, np.float32, 2 * psi, 96 + 4 * psi).any()


def test_finding2_size_law(ref):
    """Finding 2: at the same density a compressed gradient over Psi is one third of a
    compressed differential over the full 3 Psi state."""
    for psi in (10**6, 3 * 10**6, 25_557_032 // 8 * 8):
        for ppm in (1000, 10000):
            if (psi * ppm) % 10**6 == 0:
                assert 3 * 8 * ref.k_of(psi, ppm) == 8 * ref.k_of(3 * psi, ppm)


# ------------------------------------------------------------------ live loop vs recovery
def live_run(ref, tmp, sizes, ppm, world, T, b, optim, full_at=(0,), lr=1e-2, seed=0, write=True):
    """The oracle's training loop (Alg. 1 training + checkpointing processes): per rank compress,
    exchange, update; every rank persists its own block; batches of b; Full@t for t in full_at."""
    rng = np.random.default_rng(seed)
    psi = sum(sizes)
    K = sum(ref.k_table(sizes, ppm))
    consts = ref.adam_consts()
    p = rng.standard_normal(psi).astype(np.float32)
    m = np.zeros(psi, np.float32)
    v = np.zeros(psi, np.float32)
    res = [np.zeros(psi, np.float32) for _ in range(world)]
    pending = [[] for _ in range(world)]
    states = {0: (p.copy(), m.copy(), v.copy())}
    flags = ref.FLAG_EF | ref.FLAG_MEAN

    def flush(r):
        if pending[r] and write:
            first = pending[r][0][0]
            data = ref.batch_serialize(r, world, first, sizes, ppm, optim, flags, consts,
                                       np.stack([s for _, s, _ in pending[r]]),
                                       np.stack([blk for _, _, blk in pending[r]]))
            with open(os.path.join(tmp, ref.batch_name(r, first)), "wb") as f:
                f.write(data)
        pending[r] = []

    def full(t):
        if write:
            for r in range(world):
                with open(os.path.join(tmp, ref.full_name(r, t)), "wb") as f:
                    f.write(ref.full_serialize(r, world, t, optim, flags, consts, p, m, v))

    if 0 in full_at:
        full(0)
    for t in range(1, T + 1):
        sends = []
        for r in range(world):
            g = (rng.standard_normal(psi) * 1e-2).astype(np.float32)
            s, res[r] = ref.compress(sizes, ppm, g, res[r], ef=True)
            sends.append(s)
        G = ref.exchange(np.concatenate(sends), world, K, psi)
        scal = ref.step_scalars(t, lr)
        if optim == ref.ADAM:
            ref.adam_step(G, consts, scal, p, m, v)
        else:
            ref.sgd_step(G, scal[0], p)
        for r in range(world):
            pending[r].append((t, scal, sends[r]))
            if len(pending[r]) == b:
                flush(r)
        if t in full_at:
            full(t)
        states[t] = (p.copy(), m.copy(), v.copy())
    for r in range(world):
        flush(r)   # final partial batch
    return states


@pytest.mark.parametrize("optim", [0, 1])
@pytest.mark.parametrize("world,b", [(1, 1), (2, 4), (3, 3)])
def test_recover_equals_live(ref, tmp_path, optim, world, b):
    sizes, ppm, T = _sizes(), 20000, 9
    states = live_run(ref, tmp_path, sizes, ppm, world, T, b, optim, full_at=(0, 5))
    for target in (-1, 9, 7, 5, 4, 1, 0):
        p, m, v, got = ref.recover(tmp_path, world, sizes, ppm, target)
        want_t = T if target == -1 else target
        assert got == want_t
        P, M, V = states[want_t]
        assert np.array_equal(p, P)
        if optim == ref.ADAM:
            assert np.array_equal(m, M) and np.array_equal(v, V)


def test_recover_gap_and_corruption(ref, tmp_path):
    sizes, ppm, world = _sizes(), 20000, 2
    live_run(ref, tmp_path, sizes, ppm, world, 8, 2, ref.ADAM)
    # files: fulls @0; diffs first = 1,3,5,7 per rank
    assert ref.recover(tmp_path, world, sizes, ppm, -1)[3] == 8
    os.remove(os.path.join(tmp_path, ref.batch_name(1, 5)))
    assert ref.recover(tmp_path, world, sizes, ppm, -1)[3] == 4     # latest complete chain
    with pytest.raises(ref.OracleError) as e:
        ref.recover(tmp_path, world, sizes, ppm, 6)
    assert e.value.code == ref.E_GAP
    # flip one byte of a used batch file -> CRC mismatch
    path = os.path.join(tmp_path, ref.batch_name(0, 3))
    data = bytearray(open(path, "rb").read())
    data[200] ^= 0x10
    open(path, "wb").write(bytes(data))
    with pytest.raises(ref.OracleError) as e:
        ref.recover(tmp_path, world, sizes, ppm, 4)
    assert e.value.code == ref.E_CORRUPT
    # a truncated full checkpoint -> corrupt; a missing one -> gap
    path = os.path.join(tmp_path, ref.full_name(1, 0))
    open(path, "wb").write(open(path, "rb").read()[:-9])
    with pytest.raises(ref.OracleError) as e:
        ref.recover(tmp_path, world, sizes, ppm, 2)
    assert e.value.code == ref.E_CORRUPT
    os.remove(path)
    with pytest.raises(ref.OracleError) as e:
        ref.recover(tmp_path, world, sizes, ppm, 2)
    assert e.value.code == ref.E_GAP
