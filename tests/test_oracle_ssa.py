"""Pins of the SSA oracle (NEXT-2): mass-action propensities by hand,
the immigration-death closed form X(t) ~ Poisson(k/g (1 - e^-g t)) (SPEC.md:418-419,
584), conservation in the dimerisation model, and step/epoch composition."""
import math

import numpy as np
import pytest
from scipy import stats as sst

import oracle
import synth


def test_propensity_mass_action_by_hand():
    X = [7, 3, 1, 0]
    assert oracle.propensity(X, -1, -1, 2.5) == 2.5                  # 0 -> ...
    assert oracle.propensity(X, 0, -1, 2.0) == 14.0                  # c X
    assert oracle.propensity(X, 0, 1, 0.5) == 10.5                   # c X_a X_b
    assert oracle.propensity(X, 0, 0, 1.0) == 21.0                   # c X(X-1)/2
    assert oracle.propensity(X, 2, 2, 1.0) == 0.0                    # X < 2: no dimerisation
    assert math.copysign(1.0, oracle.propensity(X, 3, 3, 1.0)) == 1.0  # +0, never -0
    assert oracle.propensity(X, 3, -1, 9.0) == 0.0


def test_immigration_death_poisson():
    k, g, T = 10.0, 1.0, 2.0
    K = 20_000
    r = oracle.ssa_run(synth.immigration_death(k, g), np.zeros((K, 1), np.int32), np.zeros(K), 10**6,
                       seed=3, t_end=T, nthreads=8)
    x = r["X"][:, 0]
    lam = k / g * (1 - math.exp(-g * T))
    assert abs(x.mean() - lam) < 4 * math.sqrt(lam / K)
    assert (r["t"] <= T).all()
    # full pmf against Poisson(lam)
    kmax = 20
    counts = np.array([(x == i).sum() for i in range(kmax)] + [(x >= kmax).sum()], np.float64)
    pmf = np.append(sst.poisson.pmf(np.arange(kmax), lam), sst.poisson.sf(kmax - 1, lam))
    assert oracle.chi2_pvalue(counts, pmf)[1] > 0.001


def test_dimerisation_conserves_and_halts():
    net = synth.dimerisation()
    X0 = np.tile(np.array([[50, 7]], np.int32), (500, 1))
    r = oracle.ssa_run(net, X0, np.zeros(500), 300, seed=1)
    assert (r["X"][:, 0] + 2 * r["X"][:, 1] == 64).all()
    assert (r["X"] >= 0).all()
    # a state with nothing to fire halts immediately
    r = oracle.ssa_run(net, np.array([[1, 0]], np.int32), np.zeros(1), 10, seed=1)
    assert r["steps"][0] == 0 and r["t"][0] == 0.0


def test_steps_compose_over_epochs():
    net = synth.yeast_like_network()
    X0 = synth.initial_state(641, 64)
    whole = oracle.ssa_run(net, X0, np.zeros(64), 40, seed=9, epoch0=5)
    a = oracle.ssa_run(net, X0, np.zeros(64), 15, seed=9, epoch0=5)
    b = oracle.ssa_run(net, a["X"], a["t"], 25, seed=9, epoch0=20)
    np.testing.assert_array_equal(b["X"], whole["X"])
    np.testing.assert_array_equal(b["t"], whole["t"])


def test_one_step_is_one_selection():
    net = synth.yeast_like_network()
    X0 = synth.initial_state(641, 32)
    r = oracle.ssa_run(net, X0, np.zeros(32), 1, seed=4, epoch0=2)
    for k in range(32):
        row = np.array([oracle.propensity(X0[k], *net["reac"][j], net["rate"][j]) for j in range(net["rate"].size)],
                       np.float32)
        sel = oracle.ar_select(row, 1, seed=4, epoch=2, s0=k)
        j = sel["idx"][0]
        expect = X0[k].copy()
        for sp, v in zip(net["didx"][j], net["dval"][j]):
            if sp >= 0:
                expect[sp] += v
        np.testing.assert_array_equal(r["X"][k], expect)
        assert r["t"][k] == float(sel["tau"][0])
