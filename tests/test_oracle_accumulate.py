"""Pins of the oracle's Accumulated batch mode (R-30): the b union-compacted differentials
of a batch added into one dictionary ("gradient accumulation"; "the addition of
compressed gradients"; "tensor addition or dictionary accumulation") and
replayed as ONE optimizer step per batch.

Pinned against things other than the accumulate code itself: Python sets and dicts, a dense numpy
float32 running sum, the b = 1 identity, the exact (fp64) sum for SGD at a constant learning rate
(where accumulation is exact in real arithmetic), and the separately pinned Adam step.  For Adam with
b > 1 the mode is inexact by construction; the tests pin where it diverges."""
import os
import struct

import numpy as np
import pytest

U24 = 2.0 ** -24


def _dicts(rng, psi, n_iters, nnz, overlap):
    shared = rng.choice(psi, size=nnz, replace=False)
    out = []
    for _ in range(n_iters):
        own = rng.choice(psi, size=nnz, replace=False)
        idx = np.unique(np.where(rng.random(nnz) < overlap, shared, own)).astype(np.uint32)
        val = rng.standard_normal(idx.size).astype(np.float32)
        out.append((idx, val.view(np.uint32)))
    return out


def test_accumulate_single_dictionary_is_identity(ref):
    rng = np.random.default_rng(1)
    (idx, val), = _dicts(rng, 5000, 1, 300, 0.0)
    a_idx, a_val = ref.accumulate([(idx, val)])
    assert np.array_equal(a_idx, idx) and np.array_equal(a_val, val)
    e_idx, e_val = ref.accumulate([(np.zeros(0, np.uint32), np.zeros(0, np.uint32))])
    assert e_idx.size == 0 and e_val.size == 0


def test_accumulate_hand_example(ref):
    """{1: 1.5, 4: 2} + {0: 3, 4: -2} + {4: 0.25, 9: 1} -> {0: 3, 1: 1.5, 4: (2 + -2) + 0.25, 9: 1}."""
    f = lambda *x: np.array(x, np.float32).view(np.uint32)
    u = [(np.array([1, 4], np.uint32), f(1.5, 2.0)), (np.array([0, 4], np.uint32), f(3.0, -2.0)),
         (np.array([4, 9], np.uint32), f(0.25, 1.0))]
    idx, val = ref.accumulate(u)
    assert idx.tolist() == [0, 1, 4, 9]
    assert val.view(np.float32).tolist() == [3.0, 1.5, 0.25, 1.0]


@pytest.mark.parametrize("overlap", [0.0, 0.5, 0.95])
@pytest.mark.parametrize("n_iters", [2, 3, 8])
def test_accumulate_is_the_dense_running_sum_over_the_set_union(ref, overlap, n_iters):
    """Support = the set union of the supports; densified values = the dense float32 sum in
    iteration order from +0 (an absent index adds +0, which leaves a non-(-0) sum unchanged)."""
    rng = np.random.default_rng(7 + n_iters)
    psi = 20000
    us = _dicts(rng, psi, n_iters, 700, overlap)
    idx, val = ref.accumulate(us)
    want_support = sorted(set().union(*[set(i.tolist()) for i, _ in us]))
    assert idx.tolist() == want_support
    dense = np.zeros(psi, np.float32)
    for i, v in us:
        d = np.zeros(psi, np.float32)
        d[i] = v.view(np.float32)
        dense = (dense + d).astype(np.float32)
    got = np.zeros(psi, np.float32)
    got[idx] = val.view(np.float32)
    assert np.array_equal(got.view(np.uint32), dense.view(np.uint32))


def test_accumulate_order_is_iteration_order(ref):
    """Float addition is not associative: (1 + 2^-24) + 2^-24 != 1 + (2^-24 + 2^-24); the oracle
    adds in iteration order from +0."""
    f = lambda x: np.array([x], np.float32).view(np.uint32)
    one = np.array([3], np.uint32)
    u = [(one, f(1.0)), (one, f(U24)), (one, f(U24))]
    assert ref.accumulate(u)[1].view(np.float32)[0] == np.float32(1.0)            # ties-to-even twice
    assert ref.accumulate(u[1:] + u[:1])[1].view(np.float32)[0] == np.float32(1.0 + 2 * U24)


def _live_accumulated(ref, tmp, sizes, ppm, world, T, b, optim, lr, seed, const_lr, full_at=(0,)):
    """The oracle's training loop; every rank writes its shard's union dictionaries of each batch
    ACCUMULATED into one .ldu (partial last batch flushed).  Returns the live states and the dense
    merged gradients G_t."""
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
    Gs = {}

    def flush(r):
        if not pend[r]:
            return
        first, n = pend[r][0][0], len(pend[r])
        acc = ref.accumulate([x[2] for x in pend[r]])
        with open(os.path.join(tmp, ref.union_name(r, first)), "wb") as fh:
            fh.write(ref.accum_serialize(r, world, first, n, sizes, ppm, optim, flags, consts, pend[r][-1][1], acc))
        pend[r] = []

    for r in range(world):
        if 0 in full_at:
            with open(os.path.join(tmp, ref.full_name(r, 0)), "wb") as fh:
                fh.write(ref.full_serialize(r, world, 0, optim, flags, consts, p, m, v))
    for t in range(1, T + 1):
        sends = []
        for r in range(world):
            g = (rng.standard_normal(psi) * 1e-2).astype(np.float32)
            s, res[r] = ref.compress(sizes, ppm, g, res[r], ef=True)
            sends.append(s)
        gathered = np.concatenate(sends)
        G = ref.exchange(gathered, world, K, psi)
        Gs[t] = G
        scal = ref.step_scalars(t, lr if const_lr else lr * (1 + 0.1 * t))
        if optim == ref.ADAM:
            ref.adam_step(G, consts, scal, p, m, v)
        else:
            ref.sgd_step(G, scal[0], p)
        for r in range(world):
            u = ref.union_compact(gathered, world, K, psi, psi * r // world, psi * (r + 1) // world)
            pend[r].append((t, scal, u))
            if len(pend[r]) == b:
                flush(r)
        states[t] = (p.copy(), m.copy(), v.copy())
    for r in range(world):
        flush(r)
    return states, Gs


SIZES, PPM = [1000, 10, 3000, 7], 20000


@pytest.mark.parametrize("optim", [0, 1])
@pytest.mark.parametrize("world", [1, 3])
def test_accumulated_b1_recovers_the_live_state_exactly(ref, tmp_path, optim, world):
    states, _ = _live_accumulated(ref, tmp_path, SIZES, PPM, world, 5, 1, optim, 1e-2, 3, False)
    for target in (-1, 5, 3, 1):
        p, m, v, got = ref.recover_union(tmp_path, world, SIZES, PPM, target)
        want = 5 if target == -1 else target
        assert got == want
        P, M, V = states[want]
        assert np.array_equal(p, P)
        if optim == ref.ADAM:
            assert np.array_equal(m, M) and np.array_equal(v, V)


@pytest.mark.parametrize("world,b", [(1, 4), (2, 3), (4, 2)])
def test_accumulated_sgd_constant_lr_equals_the_exact_sum_within_rounding(ref, tmp_path, world, b):
    """SGD at a constant lr: b steps p - lr G_1 - ... - lr G_b equal p - lr (G_1 + ... + G_b) in real
    arithmetic, so the accumulated recovery lies within the rounding of b additions, one product and
    one subtraction of the fp64 value -- and so does the live fp32 state."""
    T, lr = 9, 0.05
    states, Gs = _live_accumulated(ref, tmp_path, SIZES, PPM, world, T, b, ref.SGD, lr, 5, True)
    lr32 = float(ref.step_scalars(1, lr)[0])
    p0 = states[0][0].astype(np.float64)
    for target in [t for t in range(b, T + 1, b)] + [-1]:
        p, _, _, got = ref.recover_union(tmp_path, world, SIZES, PPM, target, with_moments=False)
        want = T if target == -1 else target
        assert got == want
        Gsum = sum(Gs[t].astype(np.float64) for t in range(1, want + 1))
        Gabs = sum(np.abs(Gs[t].astype(np.float64)) for t in range(1, want + 1))
        exact = p0 - lr32 * Gsum
        bound = 2 * (want + 2) * U24 * (np.abs(p0) + lr32 * Gabs) + 1e-45
        assert np.all(np.abs(p.astype(np.float64) - exact) <= bound)
        assert np.all(np.abs(states[want][0].astype(np.float64) - exact) <= bound)


def test_accumulated_adam_is_one_step_on_the_summed_gradient_and_diverges(ref, tmp_path):
    """Adam, b = 4: the recovered state after a batch is ONE Adam step of the previous batch end's
    state with G = sum of the batch's G_t and the last iteration's scalars -- not the live state."""
    T, b, lr = 8, 4, 1e-2
    states, Gs = _live_accumulated(ref, tmp_path, SIZES, PPM, 1, T, b, ref.ADAM, lr, 9, False)
    consts = ref.adam_consts()
    P, M, V = (x.copy() for x in states[0])
    for end in (4, 8):
        G = np.zeros_like(P)
        for t in range(end - b + 1, end + 1):
            G = (G + Gs[t]).astype(np.float32)
        ref.adam_step(G, consts, ref.step_scalars(end, lr * (1 + 0.1 * end)), P, M, V)
        p, m, v, got = ref.recover_union(tmp_path, 1, SIZES, PPM, end)
        assert got == end
        assert np.array_equal(p, P) and np.array_equal(m, M) and np.array_equal(v, V)
        live = states[end][0]
        assert not np.array_equal(p, live)                         # inexact for b > 1 (R-30)
        touched = G != 0
        # the moments saw one update instead of b: m is the single step's (1-b1) G, not the b-step EMA
        assert np.max(np.abs(p - live)[touched]) > 0


def test_accumulated_targets_batch_boundaries_and_partial_batch(ref, tmp_path):
    T, b = 10, 4   # batches 1-4, 5-8, partial 9-10
    _live_accumulated(ref, tmp_path, SIZES, PPM, 2, T, b, ref.ADAM, 1e-2, 11, False)
    assert ref.recover_union(tmp_path, 2, SIZES, PPM, -1)[3] == 10
    for target in (0, 4, 8, 10):
        assert ref.recover_union(tmp_path, 2, SIZES, PPM, target)[3] == target
    for target in (1, 3, 6, 9):
        with pytest.raises(ref.OracleError) as e:
            ref.recover_union(tmp_path, 2, SIZES, PPM, target)
        assert e.value.code == ref.E_GAP
    os.remove(os.path.join(tmp_path, ref.union_name(1, 5)))
    assert ref.recover_union(tmp_path, 2, SIZES, PPM, -1)[3] == 4


def test_accumulated_ldu_layout_parses_by_hand(ref):
    sizes, ppm = [100, 30], 100000
    acc = (np.array([2, 50, 101], np.uint32), np.array([1.0, -2.0, 0.5], np.float32).view(np.uint32))
    sc = np.array([0.01, 2.0, 3.0], np.float32)
    data = ref.accum_serialize(1, 2, 17, 4, sizes, ppm, 1, 3, ref.adam_consts(), sc, acc)
    assert data[:4] == b"LDU1"
    ver, flags, rank, world, first, n_iters, n_layers = struct.unpack_from("<HHIIQII", data, 4)
    assert (ver, flags, rank, world, first, n_iters, n_layers) == (1, 3 | 4, 1, 2, 17, 4, 2)
    o = 112 + 16 * 2
    it, lr, b1, b2, cnt = struct.unpack_from("<QfffI", data, o)
    assert it == 20 and cnt == 3 and np.float32(lr) == sc[0] and (b1, b2) == (2.0, 3.0)
    assert list(struct.unpack_from("<3I", data, o + 32)) == [2, 50, 101]
    assert list(struct.unpack_from("<3f", data, o + 44)) == [1.0, -2.0, 0.5]
    assert len(data) == o + 32 + 24 + 4 == ref.union_bytes(2, [3])
    assert struct.unpack_from("<I", data, len(data) - 4)[0] == ref.crc32c(data[:-4])
