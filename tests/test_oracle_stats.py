"""Statistical pins of the oracle against the exact law the method must sample:
P(idx = j) = alpha_j / alpha_0 and trials ~ Geometric(p),
p = alpha_0 / (M alpha_max) (north_star invariant).  Fixed seeds; the multi-seed test
checks that chi-square p-values are uniform, so a 1% false-fail rate cannot hide a bias."""
import math

import numpy as np
import pytest
from scipy import stats as sst

import oracle
import synth

SMALL = {
    "1234": [1, 2, 3, 4],
    "21": [2, 1],
    "051": [0, 5, 1],
    "333": [3, 3, 3],
}


@pytest.mark.parametrize("name", list(SMALL))
def test_chi_square_exact_law(name):
    a = np.asarray(SMALL[name], np.float32)
    r = oracle.ar_select(a, 10_000, seed=20140327)
    h, _ = oracle.histogram(r["idx"], r["trials"], a.size)
    assert h[a.size] == 0                                   # no rejection
    probs = oracle.exact_law(a)
    assert (h[:a.size][probs == 0] == 0).all()              # zero-alpha never selected
    _, pval, _ = oracle.chi2_pvalue(h[:a.size][probs > 0], probs[probs > 0])
    assert pval > 0.01


def test_chi_square_pvalues_uniform_over_seeds():
    a = np.asarray([1, 2, 3, 4], np.float32)
    probs = oracle.exact_law(a)
    pv = []
    for seed in range(32):
        r = oracle.ar_select(a, 10_000, seed=1000 + seed)
        h, _ = oracle.histogram(r["idx"], r["trials"], 4)
        pv.append(oracle.chi2_pvalue(h[:4], probs)[1])
    assert sst.kstest(pv, "uniform").pvalue > 0.001


def test_biased_law_is_detected():
    # power check: the paper's argmin rule law for {1,2,3,4} (SURVEY §0.2,
    # (0.0807, 0.1745, 0.2891, 0.4557)) must FAIL the same test at K = 10^4
    a = np.asarray([1, 2, 3, 4], np.float32)
    r = oracle.ar_select(a, 10_000, seed=20140327)
    h, _ = oracle.histogram(r["idx"], r["trials"], 4)
    assert oracle.chi2_pvalue(h[:4], [0.0807, 0.1745, 0.2891, 0.4557])[1] < 1e-6


@pytest.mark.parametrize("name", ["1234", "21", "051"])
def test_trials_geometric(name):
    a = np.asarray(SMALL[name], np.float32)
    p = oracle.acceptance_rate(a)
    K = 20_000
    r = oracle.ar_select(a, K, seed=77)
    t = r["trials"].astype(np.float64)
    sd = math.sqrt((1 - p) / K) / p
    assert abs(t.mean() - 1 / p) < 4 * sd
    # full pmf: P(T = n) = (1-p)^(n-1) p, tail pooled
    nmax = 12
    counts = np.array([(t == n).sum() for n in range(1, nmax)] + [(t >= nmax).sum()], np.float64)
    pmf = np.array([(1 - p) ** (n - 1) * p for n in range(1, nmax)] + [(1 - p) ** (nmax - 1)])
    assert oracle.chi2_pvalue(counts, pmf)[1] > 0.001


def test_acceptance_rate_yeast_like():
    a = synth.yeast_like()
    p = oracle.acceptance_rate(a)
    K = 4000
    r = oracle.ar_select(a, K, seed=5)
    phat = K / r["trials"].sum()
    sd_mean = math.sqrt((1 - p) / K) / p
    assert abs(r["trials"].mean() - 1 / p) < 4 * sd_mean
    assert 0.5 * p < phat < 2 * p


def test_tau_exponential():
    # a0 * tau ~ Exp(1)
    a = np.asarray([1, 2, 3, 4], np.float32)
    r = oracle.ar_select(a, 20_000, seed=123)
    assert sst.kstest(r["tau_ref"] * 10.0, "expon").pvalue > 0.001


def test_it_and_ar_agree_in_law():
    a = synth.discrete_gaussian(64)
    K = 100_000
    ar = oracle.ar_select(a, K, seed=31, nthreads=4)
    it = oracle.it_select(a, K, seed=31, nthreads=4)
    h_ar = np.bincount(ar["idx"], minlength=64)
    h_it = np.bincount(it, minlength=64)
    table = np.vstack([h_ar, h_it])
    table = table[:, table.sum(0) >= 10]
    assert sst.chi2_contingency(table)[1] > 0.001
    # IT alone against the exact law
    probs = oracle.exact_law(a)
    assert oracle.chi2_pvalue(h_it, probs)[1] > 0.001


def test_mse_noise_floor_gaussian():
    # An exact sampler's MSE has expectation sum p(1-p)/(M n).
    # The paper's Table 1 (1.57e-7 at M=64, 10^7 draws) is the argmin rule's bias; the
    # classic rule must sit at the noise floor instead.
    M, n = 64, 400_000
    a = synth.discrete_gaussian(M)
    probs = oracle.exact_law(a)
    r = oracle.ar_select(a, n, seed=4, nthreads=8)
    h, _ = oracle.histogram(r["idx"], r["trials"], M)
    mse = oracle.mse_normalized(a, h[:M])
    floor = float((probs * (1 - probs)).sum() / (M * n))
    assert 0.5 * floor < mse < 1.8 * floor


def test_mse_definition_examples():
    # SPEC.md:463-466
    assert oracle.mse_normalized([3, 1], [1, 1]) == pytest.approx(0.0625)
    assert oracle.mse_normalized([1, 2, 3], [2, 4, 6]) == 0.0
