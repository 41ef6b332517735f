"""Pins of the oracle for the paper's PRINTED GPU rule (election + argmin selection,
PAPER.md:304-380, 498-560; NEXT-1): SPEC's hand-worked election/selection examples, the
exact quadrature law (closed forms for 2 reactions), Monte-Carlo vs that law, the
paper's own Table 1 MSE and the zero-rejection claim."""
import numpy as np
import pytest

import oracle
import synth


def test_election_spec_examples():
    # D=(2,1,0), T=2, v=(0.9,0.3,0.5) -> u=(1.8,0.6,1.0); ratings (0.9,0.6,sentinel)
    f = np.float32
    R = [oracle.election(2.0, float(f(0.9)), 2.0), oracle.election(1.0, float(f(0.3)), 2.0),
         oracle.election(0.0, 0.5, 2.0)]
    assert R[0] == pytest.approx(0.9, abs=1e-7) and R[1] == pytest.approx(0.6, abs=1e-7) and R[2] == 1.0
    # single reaction at the maximum: always eligible, rating v
    assert oracle.election(5.0, float(f(0.7)), 5.0) == pytest.approx(0.7, abs=1e-7)
    assert oracle.election(5.0, 1.0 - 2**-24, 5.0) < 1.0


def test_selection_spec_examples():
    # SPEC.md:217-219
    assert oracle.selection([0.9, 0.6, 1.0]) == 1
    assert oracle.selection([0.5, 0.5]) == 0
    assert oracle.selection([1.0, 1.0, 1.0]) == -1


def test_law_closed_forms():
    # two reactions D=(a,b), a>=b, T=a: P(1) = int_0^1 (b/a) dr * ... = b/(2a) (exact)
    for a, b in [(2, 1), (3, 1), (5, 4)]:
        P = oracle.argmin_law([a, b])
        assert P[1] == pytest.approx(b / (2 * a), rel=1e-12)
        assert P.sum() == pytest.approx(1.0, rel=1e-12)
    # SPEC.md:325 (2,1), T=2 -> (0.75, 0.25)
    np.testing.assert_allclose(oracle.argmin_law([2, 1]), [0.75, 0.25], rtol=1e-12)
    # rejection at w: prod (1 - D_i/T); w = 1 -> 0 (the argmax is always eligible)
    _, rej = oracle.argmin_law([1, 2, 3, 4], w=1.0, reject=True)
    assert rej == 0.0
    P, rej = oracle.argmin_law([1, 2, 3, 4], w=2.0, reject=True)
    assert rej == pytest.approx((1 - 1 / 8) * (1 - 2 / 8) * (1 - 3 / 8) * (1 - 4 / 8), rel=1e-12)
    assert P.sum() + rej == pytest.approx(1.0, rel=1e-12)


def test_monte_carlo_matches_quadrature_law():
    for alpha in ([1, 2, 3, 4], [0.5, 0.0, 3.0, 1.0, 2.5]):
        a = np.asarray(alpha, np.float32)
        r = oracle.argmin_select(a, 40_000, seed=17, nthreads=8)
        assert (r["idx"] >= 0).all()                   # w = 1: zero rejection
        h = np.bincount(r["idx"], minlength=a.size)
        P = oracle.argmin_law(a)
        assert (h[P == 0] == 0).all()
        assert oracle.chi2_pvalue(h[P > 0], P[P > 0])[1] > 0.001
        # and it is NOT the propensity law (the bias SURVEY §0.2 identifies)
        if a.size == 4:
            assert oracle.chi2_pvalue(h, a / a.sum())[1] < 1e-6


def test_rejection_rate_w2():
    a = np.asarray([1, 2, 3, 4], np.float32)
    K = 40_000
    r = oracle.argmin_select(a, K, seed=5, w=2.0, nthreads=8)
    _, rej = oracle.argmin_law(a, w=2.0, reject=True)
    n = (r["idx"] < 0).sum()
    assert abs(n - K * rej) < 5 * np.sqrt(K * rej * (1 - rej))


def test_table1_mse_m64_closed_form_in_paper_range():
    # PAPER.md:586-590 (Table 1, M=64 Gaussian, 10^7 selections, worst of 10 runs):
    # 1.565e-07 ... 1.645e-07.  Expected MSE = bias^2 term + sampling noise at n = 10^7.
    M, n = 64, 10**7
    d = synth.discrete_gaussian(M)
    P = oracle.argmin_law(d)
    p = d.astype(np.float64) / d.sum()
    expected = float(np.mean((P - p) ** 2) + (P * (1 - P)).sum() / (M * n))
    assert 1.565e-7 <= expected <= 1.645e-7


def test_table1_mse_monte_carlo_m64():
    M, n = 64, 2_000_000
    d = synth.discrete_gaussian(M)
    r = oracle.argmin_select(d, n, seed=99, nthreads=8)
    h = np.bincount(r["idx"], minlength=M)
    P = oracle.argmin_law(d)
    p = d.astype(np.float64) / d.sum()
    expected = float(np.mean((P - p) ** 2) + (P * (1 - P)).sum() / (M * n))
    mse = oracle.mse_normalized(d, h)
    assert 0.8 * expected < mse < 1.25 * expected


def test_scale_invariance_and_partition():
    a = np.asarray([0.3, 1.7, 0.0, 2.2, 0.9], np.float32)
    base = oracle.argmin_select(a, 500, seed=2)
    r = oracle.argmin_select(a * np.float32(2.0**9), 500, seed=2)
    np.testing.assert_array_equal(r["idx"], base["idx"])
    parts = [oracle.argmin_select(a, 250, seed=2, s0=s) for s in (0, 250)]
    np.testing.assert_array_equal(np.concatenate([p["idx"] for p in parts]), base["idx"])
    mat = oracle.argmin_select(np.tile(a, (500, 1)), 500, seed=2)
    np.testing.assert_array_equal(mat["idx"], base["idx"])
