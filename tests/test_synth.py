"""The seeded input generators (synth/): recipes follow DESIGN.md "Input recipe"."""
import math

import numpy as np

import synth


def test_discrete_gaussian_recipe():
    # x_j = -5 + j*10/(M-1), D_j = phi(x_j) * 1e5
    d = synth.discrete_gaussian(64)
    assert d.dtype == np.float32 and d.shape == (64,)
    assert d[0] == np.float32(math.exp(-12.5) / math.sqrt(2 * math.pi) * 1e5)
    np.testing.assert_allclose(d, d[::-1], rtol=1e-6)          # symmetric about x = 0
    assert d.argmax() in (31, 32)


def test_shared_families_shapes_and_ranges():
    for kind in ("uniform", "exponential", "pareto", "yeast", "gaussian"):
        a = synth.distribution(kind, 1029)
        assert a.dtype == np.float32 and a.shape == (1029,)
        assert np.all(a >= 0) and np.all(np.isfinite(a))
    u = synth.uniform(10_000)
    assert u.min() > 0 and u.max() <= 1
    assert synth.pareto(10_000).min() >= 1.0
    np.testing.assert_array_equal(synth.uniform(100, 5), synth.uniform(100, 5))   # seeded


def test_yeast_rates_recipe():
    r = synth.yeast_rates()
    assert r.size == synth.YEAST_M
    assert (r >= 0.1 * (1 - 1e-6)).all() and (r <= 1000 * (1 + 1e-6)).all()
    assert (r > 10.0).sum() >= 1


def test_rows_counter_based():
    rates = synth.yeast_rates()
    a = synth.rows(rates, 7, 0, 40)
    b = synth.rows(rates, 7, 25, 15)              # any row regenerates on its own
    np.testing.assert_array_equal(a[25:40], b)
    frac = (a > 0).mean()
    assert 0.45 < frac < 0.55                      # Bernoulli(1/2) enable mask
    nz = a > 0
    np.testing.assert_array_equal(a[nz], np.broadcast_to(rates, a.shape)[nz])
    padded = synth.rows(rates, 7, 0, 4, ld=1032)
    np.testing.assert_array_equal(padded[:, :1029], a[:4])
    assert (padded[:, 1029:] == 0).all()


def test_yeast_like_is_matrix_row_zero():
    np.testing.assert_array_equal(synth.yeast_like(), synth.rows(synth.yeast_rates(), synth.GEN_SEED, 0, 1)[0])
