"""Pins of the oracle's exchange/merge (Alg. 1 lines 5, 7) and optimizers
(Eq. 1) against things other than the oracle itself."""
import math
import os

import numpy as np
import pytest
import torch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_sync_worked_examples(ref):
    with open(os.path.join(GOLD, "sync_examples.txt")) as f:
        rows = [ln for ln in f if ln.strip() and not ln.startswith("#")]
    for ln in rows:
        world, psi, blocks, want = (c.strip() for c in ln.split("|"))
        world, psi = int(world), int(psi)
        gathered = []
        for blk in blocks.split(";"):
            pairs = [p.split(":") for p in blk.split(",")]
            gathered += [int(i) for i, _ in pairs]
            gathered += np.array([float(v) for _, v in pairs], np.float32).view(np.uint32).tolist()
        K = len(gathered) // (2 * world)
        out = ref.exchange(np.array(gathered, np.uint32), world, K, psi)
        assert out.tolist() == [float(t) for t in want.split()]


def _random_blocks(rng, world, psi, K, overlap):
    """world sorted, unique-per-rank index lists of length K with controllable overlap."""
    shared = rng.choice(psi, size=K, replace=False)
    blocks = []
    for r in range(world):
        own = rng.choice(psi, size=K, replace=False)
        take = rng.random(K) < overlap
        idx = np.where(take, shared, own)
        idx = np.unique(idx)
        while idx.size < K:
            idx = np.unique(np.concatenate([idx, rng.choice(psi, size=K - idx.size, replace=False)]))
        idx = np.sort(idx[:K]).astype(np.uint32)
        val = rng.standard_normal(K).astype(np.float32)
        blocks.append(np.concatenate([idx, val.view(np.uint32)]))
    return blocks


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("overlap", [0.0, 0.9])
def test_densify_then_average(ref, world, overlap):
    """equals densify-each-rank, sum in rank order from +0, then mean."""
    rng = np.random.default_rng(world * 10 + int(overlap * 10))
    psi, K = 5000, 400
    blocks = _random_blocks(rng, world, psi, K, overlap)
    out = ref.exchange(np.concatenate(blocks), world, K, psi, mean=True)
    dense_sum = np.zeros(psi, np.float32)          # +0.0f start (R-8)
    for b in blocks:
        d = np.zeros(psi, np.float32)
        d[b[:K]] = b[K:].view(np.float32)
        dense_sum = dense_sum + d                  # untouched positions add +0: exact
    want = dense_sum / np.float32(world)
    assert np.array_equal(out, want)
    # fp64 bound: the fp32 rank-order sum is within world * ulp of the exact mean
    exact = np.zeros(psi)
    mag = np.zeros(psi)
    for b in blocks:
        vals = b[K:].view(np.float32).astype(np.float64)
        np.add.at(exact, b[:K].astype(np.int64), vals)
        np.add.at(mag, b[:K].astype(np.int64), np.abs(vals))
    exact /= world
    mag /= world
    # recursive summation bound: |fl(sum) - sum| <= (N-1) u sum|v|, plus one rounding of the divide
    assert np.all(np.abs(out - exact) <= world * 2.0 ** -24 * mag + 2.0 ** -24 * np.abs(exact))
    if world in (1, 2, 4, 8):
        # power-of-two N: the mean is the sum scaled by 2^-log2 N, exactly
        s = ref.exchange(np.concatenate(blocks), world, K, psi, mean=False)
        assert np.array_equal(out, s * np.float32(1.0 / world))


def test_merge_never_negative_zero(ref):
    K, psi = 2, 4
    b0 = np.array([0, 1] + np.array([-0.0, -0.0], np.float32).view(np.uint32).tolist(), np.uint32)
    b1 = np.array([1, 2] + np.array([0.0, -0.0], np.float32).view(np.uint32).tolist(), np.uint32)
    out = ref.exchange(np.concatenate([b0, b1]), 2, K, psi)
    assert not np.any(np.signbit(out))


# ------------------------------------------------------------------ optimizer scalars / Adam / SGD
def test_scalar_derivation(ref):
    c = ref.adam_consts(0.9, 0.999, 1e-8)
    assert c[0] == np.float32(0.9) and c[2] == np.float32(0.999)
    assert c[1] == np.float32(0.1)          # fl32(1 - 0.9) in double, not 1f - 0.9f = 0.100000024
    assert c[3] == np.float32(0.001)        # not 1f - 0.999f = 0.0009999871
    assert c[4] == np.float32(1e-8)
    for t in (1, 2, 3, 10, 100, 1000, 54321):
        s = ref.step_scalars(t, 1e-3)
        assert s[0] == np.float32(1e-3)
        assert s[1] == np.float32(1.0 / (1.0 - math.pow(0.9, t)))
        assert s[2] == np.float32(1.0 / (1.0 - math.pow(0.999, t)))
    assert ref.step_scalars(1, 1e-3)[1] == np.float32(10.0)


def test_adam_zero_gradient_zero_moments(ref):
    """fresh state, zero gradient -> params unchanged."""
    p = np.linspace(-1, 1, 101).astype(np.float32)
    p0 = p.copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    ref.adam_step(np.zeros_like(p), ref.adam_consts(), ref.step_scalars(1, 0.1), p, m, v)
    assert np.array_equal(p, p0) and not m.any() and not v.any()


def test_adam_first_step_is_signed_lr(ref):
    """from zero state, delta p = -lr * g / (|g| + eps*sqrt(...)) ~= -lr*sign(g)."""
    g = np.array([1.0, -1.0, 3e-3, -250.0, 1e-2], np.float32)
    p = np.zeros_like(g)
    m = np.zeros_like(g)
    v = np.zeros_like(g)
    ref.adam_step(g, ref.adam_consts(), ref.step_scalars(1, 0.1), p, m, v)
    assert np.all(np.abs(p + 0.1 * np.sign(g)) < 1e-6)


def test_adam_matches_fp64_recurrence(ref):
    """Kingma-Ba in float64 (textbook form): the fp32 oracle stays within a few ulps * steps."""
    rng = np.random.default_rng(11)
    n, T, lr, b1, b2, eps = 2000, 50, 1e-3, 0.9, 0.999, 1e-8
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    P, M, V = p.astype(np.float64), np.zeros(n), np.zeros(n)
    for t in range(1, T + 1):
        g = (rng.standard_normal(n) * (rng.random(n) < 0.3)).astype(np.float32)
        ref.adam_step(g, ref.adam_consts(b1, b2, eps), ref.step_scalars(t, lr, b1, b2), p, m, v)
        G = g.astype(np.float64)
        M = b1 * M + (1 - b1) * G
        V = b2 * V + (1 - b2) * G * G
        P = P - lr * (M / (1 - b1 ** t)) / (np.sqrt(V / (1 - b2 ** t)) + eps)
    err = np.max(np.abs(p - P) / np.maximum(np.abs(P), 1.0))
    assert err < 1e-5
    # a plausible bug (e.g. swapped bias corrections) would be far outside this bound
    assert np.max(np.abs(m - M)) < 1e-5


def test_adam_cross_check_torch(ref):
    """torch.optim.Adam(foreach=False) on the same dense G_t: a different formula (lerp/addcdiv),
    so only norm-wise agreement ~1e-6 is expected (SURVEY §8(c) replay pin (iii))."""
    rng = np.random.default_rng(12)
    n, T, lr = 4096, 100, 1e-3
    p = rng.standard_normal(n).astype(np.float32)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    tp = torch.nn.Parameter(torch.from_numpy(p.copy()))
    opt = torch.optim.Adam([tp], lr=lr, betas=(0.9, 0.999), eps=1e-8, foreach=False)
    for t in range(1, T + 1):
        g = (rng.standard_normal(n) * 1e-3 * (rng.random(n) < 0.08)).astype(np.float32)
        ref.adam_step(g, ref.adam_consts(), ref.step_scalars(t, lr), p, m, v)
        tp.grad = torch.from_numpy(g.copy())
        opt.step()
    q = tp.detach().numpy()
    assert np.max(np.abs(p - q)) / np.max(np.abs(q)) < 1e-5


def test_sgd_step(ref):
    p = np.array([1.0, -0.0, 2.0, 0.0], np.float32)
    G = np.array([0.5, 0.0, 0.0, -4.0], np.float32)
    ref.sgd_step(G, 0.25, p)
    assert p.tolist() == [0.875, -0.0, 2.0, 1.0]
    assert np.signbit(p[1])  # p - lr*(+0) keeps -0 (R-12)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_density_one_sgd_equals_dense_dp(ref, world):
    """Closed special case (north_star): ppm = 1e6 + SGD is plain dense data-parallel SGD."""
    rng = np.random.default_rng(world)
    sizes = [300, 17, 1000]
    psi = sum(sizes)
    p = rng.standard_normal(psi).astype(np.float32)
    q = p.copy()
    res = [np.zeros(psi, np.float32) for _ in range(world)]
    lr = np.float32(0.1)
    for t in range(5):
        grads = [rng.standard_normal(psi).astype(np.float32) for _ in range(world)]
        sends = []
        for r in range(world):
            s, res[r] = ref.compress(sizes, 1000000, grads[r], res[r], ef=True)
            sends.append(s)
        G = ref.exchange(np.concatenate(sends), world, psi, psi)
        ref.sgd_step(G, lr, p)
        dense = np.zeros(psi, np.float32)
        for g in grads:
            dense = dense + g
        q = q - lr * (dense / np.float32(world))
        assert all(not r_.any() for r_ in res)
    assert np.array_equal(p, q)
