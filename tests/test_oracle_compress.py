"""Pins of the oracle's compress (Alg. 1 line 4) against things other than itself.

- brute force of the rank definition on tiny inputs (O(n^2), pure numpy)
- the worked examples of SPEC.md:132-134 (tests/golden/spec_compress_examples.txt)
- invariants: exactly k_l per layer; ascending in-layer indices; send + residual' == acc;
  every selected key >= every unselected key; inf-norm error == (k+1)-th largest |acc|
- special cases: ppm = 1e6 is the identity with residual' == 0; ef = 0 leaves r alone
- the k rule (R-3) against the K totals of SURVEY Appendix A
"""
import os

import numpy as np
import pytest

from inputs import adversarial_layers, table

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def brute_select(acc: np.ndarray, k: int) -> np.ndarray:
    """sel(j) <=> #{i : key_i > key_j or (key_i == key_j and i < j)} < k  (R-4)."""
    key = acc.view(np.uint32) & np.uint32(0x7FFFFFFF)
    n = acc.size
    sel = []
    for j in range(n):
        beats = int(np.sum(key > key[j])) + int(np.sum(key[:j] == key[j]))
        if beats < k:
            sel.append(j)
    return np.array(sel, dtype=np.int64)


def split(send, K):
    return send[:K], send[K:].view(np.float32)


def test_k_rule_matches_appendix_a(ref):
    # K at 0.1% / 0.25% / 0.5% / 1%
    expect = {
        "mlp": (103, 255, 509, 1017),
        "resnet50": (25595, 63881, 127745, 255513),
        "bert_large": (335063, 837646, 1675560, 3351266),
        "gpt2_xl": (1557379, 3894028, 7788056, 15576112),
    }
    for name, ks in expect.items():
        sizes = table(name)
        got = tuple(sum(ref.k_table(sizes, ppm)) for ppm in (1000, 2500, 5000, 10000))
        assert got == ks, name
    assert ref.k_table(table("mlp"), 10000) == [1003, 1, 12, 1]
    assert ref.k_of(5, 1) == 1 and ref.k_of(7, 1000000) == 7


def test_spec_worked_examples(ref):
    with open(os.path.join(GOLD, "spec_compress_examples.txt")) as f:
        rows = [ln for ln in f if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 3
    for ln in rows:
        ppm, dense, idx, val = (c.strip() for c in ln.split("|"))
        x = np.array([float(t) for t in dense.split()], np.float32)
        for ef in (False, True):
            send, r = ref.compress([x.size], int(ppm), x, np.zeros_like(x), ef=ef)
            K = send.size // 2
            i, v = split(send, K)
            assert i.tolist() == [int(t) for t in idx.split()]
            assert v.tolist() == [float(t) for t in val.split()]


@pytest.mark.parametrize("dist", ["normal", "bf16", "small_int", "zeros_mixed"])
@pytest.mark.parametrize("ppm", [1000, 10000, 123456, 500000])
def test_brute_force_rank_definition(ref, dist, ppm):
    rng = np.random.default_rng(abs(hash((dist, ppm))) % (2**32))
    sizes = [1, 7, 300, 1024, 2048]
    psi = sum(sizes)
    if dist == "normal":
        g = rng.standard_normal(psi).astype(np.float32)
    elif dist == "bf16":
        g = (rng.standard_normal(psi).astype(np.float32).view(np.uint32) & 0xFFF00000).view(np.float32)
    elif dist == "small_int":
        g = rng.integers(-3, 4, psi).astype(np.float32)
    else:
        g = rng.standard_normal(psi).astype(np.float32) * (rng.random(psi) < 0.05)
    r = (rng.standard_normal(psi) * 0.5).astype(np.float32)
    send, r2 = ref.compress(sizes, ppm, g, r, ef=True)
    K = sum(ref.k_table(sizes, ppm))
    idx, val = split(send, K)
    acc = (r + g).astype(np.float32)          # one fp32 add per element
    off = koff = 0
    for n in sizes:
        k = ref.k_of(n, ppm)
        want = brute_select(acc[off:off + n], k) + off
        assert idx[koff:koff + k].tolist() == want.tolist()
        off += n
        koff += k


def test_invariants(ref):
    rng = np.random.default_rng(7)
    sizes = [5000, 12345, 3, 40000]
    psi = sum(sizes)
    for ppm in (1000, 10000, 100000):
        g = rng.standard_normal(psi).astype(np.float32) * 1e-3
        r = rng.standard_normal(psi).astype(np.float32) * 1e-3
        send, r2 = ref.compress(sizes, ppm, g, r, ef=True)
        K = sum(ref.k_table(sizes, ppm))
        idx, val = split(send, K)
        acc = r + g
        # decompress(send) + residual' == acc, as floats
        dense = np.zeros(psi, np.float32)
        dense[idx] = val
        assert np.array_equal(dense + r2, acc)
        assert np.all(r2[idx] == 0) and np.all(np.signbit(r2[idx]) == 0)
        off = koff = 0
        for n in sizes:
            k = ref.k_of(n, ppm)
            li = idx[koff:koff + k]
            assert np.all((li >= off) & (li < off + n))
            assert np.all(np.diff(li.astype(np.int64)) > 0)
            a = np.abs(acc[off:off + n])
            mask = np.zeros(n, bool)
            mask[li - off] = True
            if k < n:
                assert a[~mask].max() <= a[mask].min()
                # inf-norm error of the sparsified layer == (k+1)-th largest magnitude
                err = np.abs(r2[off:off + n]).max()
                assert err == np.sort(a)[::-1][k]
            off += n
            koff += k


def test_density_one_is_identity(ref):
    rng = np.random.default_rng(3)
    sizes = [10, 1000, 77]
    g = rng.standard_normal(sum(sizes)).astype(np.float32)
    send, r2 = ref.compress(sizes, 1000000, g, np.zeros_like(g), ef=True)
    K = sum(sizes)
    idx, val = split(send, K)
    assert idx.tolist() == list(range(K))
    assert np.array_equal(val, g)
    assert np.all(r2 == 0)


def test_ef_off_matches_spec_and_leaves_residual(ref):
    rng = np.random.default_rng(5)
    sizes = [3000, 100]
    g = rng.standard_normal(sum(sizes)).astype(np.float32)
    s0, r0 = ref.compress(sizes, 10000, g, None, ef=False)
    assert r0 is None
    s1, r1 = ref.compress(sizes, 10000, g, np.zeros_like(g), ef=True)
    # no -0.0 in g, so acc = +0 + g == g bit for bit and the two modes agree
    assert np.array_equal(s0, s1)
    # with ef = 1 the unselected mass stays in the residual: residual' == g off the selection
    K = s1.size // 2
    off = np.ones(g.size, bool)
    off[s1[:K]] = False
    assert np.array_equal(r1[off], g[off]) and np.all(r1[~off] == 0)


def test_adversarial_layers(ref):
    for name, x in adversarial_layers():
        x = x.numpy().astype(np.float32)
        for ppm in (10000, 250000):
            send, _ = ref.compress([x.size], ppm, x, np.zeros_like(x), ef=True)
            k = ref.k_of(x.size, ppm)
            acc = (np.zeros_like(x) + x).astype(np.float32)
            want = brute_select(acc, k) if x.size <= 4100 else None
            if want is not None:
                assert send[:k].tolist() == want.tolist(), name
            if name == "all_zero":
                assert send[:k].tolist() == list(range(k))


def test_non_finite_is_numeric_error(ref):
    for bad in (np.nan, np.inf, -np.inf):
        g = np.ones(100, np.float32)
        g[17] = bad
        with pytest.raises(ref.OracleError) as e:
            ref.compress([100], 10000, g, np.zeros_like(g), ef=True)
        assert e.value.code == ref.E_NUMERIC
    # overflow in the EF add itself: residual + grad = inf
    g = np.full(10, 3e38, np.float32)
    with pytest.raises(ref.OracleError):
        ref.compress([10], 100000, g, g.copy(), ef=True)
