"""NEXT-4: checkpointing configuration (§4.3, Eq. 3-5; module PAPER.md:454-455).

Pins: the oracle's Eq. 3 is written term by term from the itemised model; its
Eq. 5 optimum is checked against a brute-force grid minimisation of Eq. 3 and against the
first-order conditions (Eq. 4) by finite differences; the qualitative shape of Table 1 (the
optimal batch size grows with the full-checkpoint interval) is checked on the model.  The product
(C ABI) must agree with the oracle."""
import math
import os

import numpy as np
import pytest

import paper_2509_04084_b200 as ld
from paper_2509_04084_b200 import lowdiff as B

GOLD = os.path.join(os.path.dirname(__file__), "golden")

# a GPT-2-S-like setting in iteration units: 1.4 GB full checkpoint, 2 GB/s SSD at 0.3 s/iteration,
# 8 GPUs, MTBF 2 h at 0.3 s/iteration, 1e5 iterations, R_F = 5 iterations, R_D = 0.2 iterations
CASES = [
    dict(N=8, M=24000, W=0.6e9, S=1.4e9, T=1e5, R_F=5.0, R_D=0.2),
    dict(N=64, M=1800, W=2e9, S=8.7e9, T=5e4, R_F=20.0, R_D=1.0),
    dict(N=1, M=1e6, W=5e8, S=3e8, T=1e6, R_F=1.0, R_D=0.05),
]


def ref_args(p):
    return (p["N"], p["M"], p["W"], p["S"], p["T"], p["R_F"], p["R_D"])


@pytest.mark.parametrize("p", CASES)
def test_oracle_closed_form_is_grid_minimum(ref, p):
    f_star, b_star = ref.optimal_config(p["M"], p["W"], p["S"], p["R_D"])
    fs = f_star * np.exp(np.linspace(-1.5, 1.5, 301))
    bs = b_star * np.exp(np.linspace(-1.5, 1.5, 301))
    grid = np.array([[ref.wasted_time(*ref_args(p), f, b) for b in bs] for f in fs])
    i, j = np.unravel_index(np.argmin(grid), grid.shape)
    assert abs(math.log(fs[i] / f_star)) <= 0.011 and abs(math.log(bs[j] / b_star)) <= 0.011
    # Eq. 4: both partial derivatives vanish at the optimum (central differences)
    h = 1e-6
    tw = lambda f, b: ref.wasted_time(*ref_args(p), f, b)
    df = (tw(f_star * (1 + h), b_star) - tw(f_star * (1 - h), b_star)) / (2 * h * f_star)
    db = (tw(f_star, b_star * (1 + h)) - tw(f_star, b_star * (1 - h))) / (2 * h * b_star)
    scale = tw(f_star, b_star)
    assert abs(df * f_star) < 1e-5 * scale and abs(db * b_star) < 1e-5 * scale


def test_table1_shape(ref):
    """Table 1: the best BS per row is non-decreasing in FCF.  The model gives
    b_opt(f) = sqrt(R_D / f) for a fixed f, which grows with the interval 1/f."""
    rows = [ln for ln in open(os.path.join(GOLD, "table1_fcf_bs.txt")) if ln.strip() and not ln.startswith("#")]
    paper_best = []
    for ln in rows:
        fcf, vals = ln.split("|")
        paper_best.append((int(fcf), 1 + int(np.argmin([float(x) for x in vals.split()]))))
    assert [b for _, b in paper_best] == sorted(b for _, b in paper_best) == [2, 2, 3, 3]
    p = dict(N=8, M=24000, W=0.6e9, S=1.4e9, T=1e5, R_F=5.0, R_D=0.1)
    model_best = []
    for fcf, _ in paper_best:
        vals = [ref.wasted_time(*ref_args(p), 1.0 / fcf, b) for b in range(1, 7)]
        model_best.append(1 + int(np.argmin(vals)))
    assert model_best == sorted(model_best) and model_best[0] < model_best[-1]


@pytest.mark.parametrize("p", CASES)
def test_product_matches_oracle(ref, p):
    f, b = ld.lowdiff.optimal_config(p)
    rf, rb = ref.optimal_config(p["M"], p["W"], p["S"], p["R_D"])
    assert f == rf and b == rb
    for ff in (f, 2 * f, 0.5 * f):
        for bb in (1.0, b, 3.0):
            assert math.isclose(B.wasted_time(p, ff, bb), ref.wasted_time(*ref_args(p), ff, bb), rel_tol=1e-12)


@pytest.mark.parametrize("p", CASES)
def test_stepwise_adaptation_converges_and_never_worsens(ref, p):
    f_star, b_star = ref.optimal_config(p["M"], p["W"], p["S"], p["R_D"])
    fcf, batch = 1, 1
    prev = ref.wasted_time(*ref_args(p), 1.0 / fcf, batch)
    for _ in range(200):
        fcf, batch = B.config_step(p, fcf, batch)
        cur = ref.wasted_time(*ref_args(p), 1.0 / fcf, batch)
        assert cur <= prev * (1 + 1e-12)
        prev = cur
    assert abs(fcf - round(1.0 / f_star)) <= max(1, 0.1 * round(1.0 / f_star))
    assert abs(batch - round(b_star)) <= 1
    with pytest.raises(ld.LowDiffError):
        B.config_step(dict(p, M=0.0), 10, 2)


# ---------------------------------------------------------------- failure-injection simulator
SIM = dict(N=8, M=2000.0, W=0.6e9, S=1.4e9, T=2e5, R_F=5.0, R_D=0.2)


def test_sim_trace_is_poisson_and_deterministic(ref):
    """The trace has N T / M failures in expectation (Poisson: within 4 sigma), is a pure function
    of the seed, and the kind draw follows sw_fraction."""
    a = ref.simulate(*ref_args(SIM), 1 / 200.0, 4.0, 0.0, 0.0, seed=11)
    assert a == ref.simulate(*ref_args(SIM), 1 / 200.0, 4.0, 0.0, 0.0, seed=11)
    assert a != ref.simulate(*ref_args(SIM), 1 / 200.0, 4.0, 0.0, 0.0, seed=12)
    lam = SIM["N"] * SIM["T"] / SIM["M"]
    assert abs(a[0] - lam) < 4 * math.sqrt(lam)
    assert a[1] == a[0]                                     # sw_fraction 0: all hardware
    s1 = ref.simulate(*ref_args(SIM), 1 / 200.0, 4.0, 1.0, 3.0, seed=11)
    assert s1[0] == a[0] and s1[1] == 0                     # same arrival draws, all software
    assert s1[2] == 0.0 and s1[3] == 3.0 * s1[0]            # software: R_S each, no lost work
    h = ref.simulate(*ref_args(SIM), 1 / 200.0, 4.0, 0.5, 3.0, seed=11)
    assert abs(h[1] - 0.5 * h[0]) < 4 * math.sqrt(0.25 * h[0])


def test_sim_ledger_and_no_failure_limit(ref):
    n, hw, lost, rec, steady, wasted = ref.simulate(*ref_args(SIM), 1 / 250.0, 5.0, 0.2, 1.0, seed=3)
    assert wasted == lost + rec + steady
    assert steady == SIM["N"] * (SIM["S"] / SIM["W"]) * math.floor(SIM["T"] / 250.0)
    assert 0 <= lost <= 5.0 * hw
    quiet = dict(SIM, M=1e30)
    assert ref.simulate(*ref_args(quiet), 1 / 250.0, 5.0, seed=3)[:4] == (0, 0, 0.0, 0.0)


@pytest.mark.parametrize("fcf,b", [(200, 4), (300, 10), (60, 1)])
def test_sim_mean_matches_eq3(ref, fcf, b):
    """Over 300 seeds the mean simulated wasted time equals Eq. 3's prediction within 3 standard
    errors (1/f a multiple of b, where Eq. 3's b/2 and (1/(fb) - 1)/2 are exact expectations).
    This pins the recovery terms of the oracle's Eq. 3 by simulation of Alg. 1's recovery."""
    f = 1.0 / fcf
    xs = np.array([ref.simulate(*ref_args(SIM), f, float(b), seed=s)[5] for s in range(300)])
    pred = ref.wasted_time(*ref_args(SIM), f, float(b))
    se = xs.std(ddof=1) / math.sqrt(xs.size)
    assert abs(xs.mean() - pred) < 3 * se + 1e-9 * pred, (xs.mean(), pred, se)


def test_sim_product_matches_oracle(ref):
    for seed in (0, 1, 99):
        for swf in (0.0, 0.3):
            want = ref.simulate(*ref_args(SIM), 1 / 180.0, 3.0, swf, 2.5, seed=seed)
            got = B.simulate_failures(SIM, 1 / 180.0, 3.0, swf, 2.5, seed)
            assert (got["failures"], got["hw_failures"]) == want[:2]
            for k, w in zip(("lost_work", "recovery", "steady", "wasted"), want[2:]):
                assert math.isclose(got[k], w, rel_tol=1e-12, abs_tol=1e-12), (k, got[k], w)
            assert got["effective_ratio"] == SIM["T"] / (SIM["T"] + got["wasted"])
    with pytest.raises(ld.LowDiffError):
        B.simulate_failures(SIM, 0.0, 3.0)


# ---------------------------------------------------------------- domain f b <= 1
# a cluster where Eq. 5's stationary point leaves the model's domain: f* b* = cbrt(R_D^2 W / (2 S M)) > 1
FAST = dict(N=8, M=100.0, W=1e10, S=1e9, T=1e5, R_F=2.0, R_D=10.0)


def test_wasted_time_rejects_batch_beyond_full_interval():
    with pytest.raises(ld.LowDiffError):
        B.wasted_time(CASES[0], 0.5, 3.0)                  # f b = 1.5: the merge term would be negative
    with pytest.raises(ld.LowDiffError):
        B.simulate_failures(SIM, 0.5, 3.0)
    assert B.wasted_time(CASES[0], 0.5, 2.0) > 0            # f b = 1 is inside


def test_feasible_optimum_is_grid_minimum_on_the_domain(ref):
    f, b, clamped, fu, bu = B.optimal_config_feasible(FAST)
    rf, rb = ref.optimal_config(FAST["M"], FAST["W"], FAST["S"], FAST["R_D"])
    assert (fu, bu) == (rf, rb) and fu * bu > 1 and clamped
    assert math.isclose(f * b, 1.0, rel_tol=1e-12)
    best = min(ref.wasted_time(*ref_args(FAST), ff, bb)
               for ff in f * np.exp(np.linspace(-2, 2, 201)) for bb in b * np.exp(np.linspace(-2, 2, 201))
               if ff * bb <= 1.0)
    assert ref.wasted_time(*ref_args(FAST), f, b) <= best * (1 + 1e-9)
    for p in CASES:                                        # inside the domain: the Eq. 5 point itself
        f2, b2, cl2, fu2, bu2 = B.optimal_config_feasible(p)
        assert not cl2 and (f2, b2) == (fu2, bu2) == ref.optimal_config(p["M"], p["W"], p["S"], p["R_D"])


def test_stepwise_adaptation_stays_in_domain():
    fcf, batch = 1, 1
    for _ in range(100):
        fcf, batch = B.config_step(FAST, fcf, batch)
        assert 1 <= batch <= fcf
    with pytest.raises(ld.LowDiffError):
        B.config_step(FAST, 2, 3)
