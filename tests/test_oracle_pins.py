"""Pins of the CPU oracle against things other than itself: published known-answer
vectors, closed forms, hand-worked cases, independently derived golden values and exact
brute force.  (DESIGN.md "Oracle pins".)"""
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], tuple(v[6:10])))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answers(ctr, key, out):
    # Random123 KAT vectors (tests/golden/philox_kat.txt)
    assert oracle.philox4x32_10(ctr, key) == out


def test_index_mapping_closed_form():
    # j = floor(x*M/2^32): bucket boundaries at multiples of 2^32/M (R5)
    assert oracle.index_of(0x55555555, 3) == 0
    assert oracle.index_of(0x55555556, 3) == 1
    assert oracle.index_of(0xAAAAAAAA, 3) == 1
    assert oracle.index_of(0xAAAAAAAB, 3) == 2
    assert oracle.index_of(0xFFFFFFFF, 3) == 2
    assert oracle.index_of(0x80000000, 4) == 2
    assert oracle.index_of(0xC0000000, 4) == 3
    assert oracle.index_of(0x00000000, 1029) == 0
    assert oracle.index_of(0xFFFFFFFF, 1029) == 1028
    # every bucket of M=7 is hit by exactly floor or ceil(2^32/7) inputs: check edges
    M = 7
    for j in range(M):
        lo = -(-(j << 32) // M)         # ceil(j*2^32/M)
        assert oracle.index_of(lo, M) == j
        if lo > 0:
            assert oracle.index_of(lo - 1, M) == j - 1


def test_unit_mappings():
    # u = (x>>8) 2^-24 in [0,1); u1 = (2(x>>9)+1) 2^-24 in (0,1) (R3, R10)
    assert oracle.unit(0) == 0.0
    assert oracle.unit(0xFFFFFFFF) == 1.0 - 2.0**-24
    assert oracle.unit(0x80000000) == 0.5
    assert oracle.unit(0x000000FF) == 0.0          # low 8 bits ignored
    assert oracle.unit(0x00000100) == 2.0**-24
    assert oracle.unit_open(0) == 2.0**-24
    assert oracle.unit_open(0xFFFFFFFF) == 1.0 - 2.0**-24
    assert oracle.unit_open(0x80000000) == 0.5 + 2.0**-24


def test_acceptance_strict_and_handworked():
    # alpha = (1,2,3,4), T = 4 (SURVEY §8c pins, worked by hand)
    u = oracle.unit(0xBFFFFF00)                    # 0.74999994
    assert oracle.index_of(0x80000000, 4) == 2
    assert oracle.accept(u, 4.0, 3.0)              # 2.9999998 < 3 -> accept
    assert not oracle.accept(oracle.unit(0xC0000000), 4.0, 3.0)   # 3 < 3 is false (strict)
    assert oracle.accept(0.0, 4.0, 1.0)            # u = 0 accepts any alpha_j > 0
    assert not oracle.accept(0.0, 5.0, 0.0)        # alpha_j = 0 never accepted


def test_acceptance_is_binary32_round_to_nearest():
    # fl32(u*T) differs from the exact product: exact/double arithmetic would accept
    u = oracle.unit(0xD5555500)                    # 0xD55555 * 2^-24
    assert u * 3.0 < 2.5                           # exact (double) product accepts
    assert not oracle.accept(u, 3.0, 2.5)          # binary32 RN product rounds up to 2.5 -> reject
    f = np.float32
    u2 = oracle.unit(0x55555500)
    assert float(u2) * float(f(0.3)) < float(f(0.1))
    assert not oracle.accept(u2, float(f(0.3)), float(f(0.1)))


def _golden_rows():
    out = []
    with open(os.path.join(GOLDEN, "ar_seed14040027.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            name, alpha, epoch, s0, idx, trials, tau = [p.strip() for p in line.split("|")]
            out.append((name, [float(x) for x in alpha.split(",")], int(epoch), int(s0),
                        [int(x) for x in idx.split(",")], [int(x) for x in trials.split(",")],
                        [float(x) for x in tau.split(",")] if tau else None))
    return out


@pytest.mark.parametrize("name,alpha,epoch,s0,idx,trials,tau", _golden_rows())
def test_end_to_end_golden(name, alpha, epoch, s0, idx, trials, tau):
    r = oracle.ar_select(alpha, len(idx), seed=14040027, epoch=epoch, s0=s0)
    assert r["idx"].tolist() == idx
    assert r["trials"].tolist() == trials
    if tau is not None:
        np.testing.assert_allclose(r["tau"], tau, rtol=2e-6)


def test_stats_and_validity():
    amax, a0, st = oracle.stats([1, 2, 3, 4])
    assert (amax, a0, st) == (4.0, 10.0, oracle.OK)
    assert oracle.stats([0, 0, 0])[0:2] == (0.0, 0.0)
    for bad in ([1, -1], [1, float("nan")], [1, float("inf")], [1, -0.0]):
        assert oracle.stats(bad)[2] == oracle.EPROPENSITY
    # alpha_0 sums exactly for integers (binary64 accumulation)
    a = np.arange(1, 1001, dtype=np.float32)
    assert oracle.stats(a)[1] == 500500.0


def test_tau_range_and_exact_scaling():
    # SPEC.md:398-400's sampleTau examples (a0=2, u1=e^-2 -> 1; a0=4, u1=1/2 -> ln2/4) cannot
    # be reproduced through the stream: u1 = (2 (x >> 9) + 1) 2^-24 is an odd multiple of
    # 2^-24 (R10), never e^-2 or 1/2.  What the closed form fixes and this test
    # checks: a0 * tau_ref = -ln(u1) lies in [-ln(1 - 2^-24), -ln(2^-24)] = (0, 16.64], and
    # tau scales exactly as 1/a0.  tau's law (a0 tau ~ Exp(1)) is pinned by the KS test in
    # test_oracle_stats.py and its values by the golden file (tests/golden/ar_seed14040027.txt).
    r = oracle.ar_select([1, 1], 4096, seed=7)
    x = r["tau_ref"] * 2.0
    assert np.all(x > 0) and np.all(x <= -math.log(2.0**-24) + 1e-12)
    # a0 scaling: doubling every propensity halves tau exactly (binary32 division by 2a0)
    r2 = oracle.ar_select([2, 2], 4096, seed=7)
    np.testing.assert_array_equal(r2["tau"], r["tau"] / np.float32(2))
    np.testing.assert_array_equal(r2["idx"], r["idx"])


def test_degenerate_all_zero():
    r = oracle.ar_select([0, 0, 0], 16, seed=1)
    assert (r["idx"] == -1).all() and (r["trials"] == 0).all() and np.isinf(r["tau"]).all()


def test_invalid_vector_flagged():
    r = oracle.ar_select([1, -2, 3], 8, seed=1)
    assert r["status"] == oracle.EPROPENSITY
    assert (r["idx"] == -1).all() and np.isnan(r["tau"]).all()


def test_max_trials_one_and_odd():
    # max_trials = 1: only trial 0 exists; rejected selections report trials = 1, idx = -1
    r = oracle.ar_select([1, 2, 3, 4], 2000, seed=3, max_trials=1)
    assert set(r["trials"].tolist()) == {1}
    full = oracle.ar_select([1, 2, 3, 4], 2000, seed=3)
    acc = full["trials"] == 1
    np.testing.assert_array_equal(r["idx"][acc], full["idx"][acc])
    assert (r["idx"][~acc] == -1).all()
    # odd cap 3 agrees with the uncapped run wherever the uncapped run needed <= 3 trials
    r3 = oracle.ar_select([1, 2, 3, 4], 2000, seed=3, max_trials=3)
    ok = full["trials"] <= 3
    np.testing.assert_array_equal(r3["idx"][ok], full["idx"][ok])
    assert (r3["trials"][~ok] == 3).all() and (r3["idx"][~ok] == -1).all()


def test_single_nonzero_and_all_equal():
    a = np.zeros(50, np.float32)
    a[17] = 3.0
    r = oracle.ar_select(a, 4000, seed=11)
    assert (r["idx"] == 17).all()
    # trials ~ Geometric(1/M): mean M within 5 sigma
    sd = math.sqrt((1 - 1 / 50) * 50**2 / 4000)
    assert abs(r["trials"].mean() - 50) < 5 * sd
    r = oracle.ar_select(np.full(9, 0.7, np.float32), 1000, seed=11)
    assert (r["trials"] == 1).all()                 # u < 1 -> fl32(u*T) < T always


def test_it_spec_examples_and_partition():
    # SPEC.md:280-282
    assert oracle.it_one([1, 1, 2], 0.6) == 2
    assert oracle.it_one([1, 1, 2], 0.0) == 0
    assert oracle.it_one([0, 5], 0.1) == 1
    # partition exactness: on a dense u2 grid the chosen j satisfies
    # C_{j-1} <= u2 a0 < C_j, brute force over every grid point
    alpha = np.array([0.5, 0, 2, 1.25, 0, 0.25], np.float32)
    C = np.cumsum(alpha.astype(np.float64))
    a0 = C[-1]
    for k in range(0, 4096):
        u2 = k / 4096.0
        j = oracle.it_one(alpha, u2)
        lo = C[j - 1] if j > 0 else 0.0
        assert lo <= u2 * a0 < C[j]
        assert alpha[j] > 0


def test_it_prefix_is_the_sequential_binary64_sum():
    """DESIGN.md R24 (the reading the GPU's IT paths are bit-checked against): C_j is the
    SEQUENTIAL binary64 prefix.  Hand-worked: alpha = (1, 2^-54, 2^-54, 1).  In binary64
    1 + 2^-54 rounds back to 1 (2^-54 is below half an ulp of 1, 2^-53), so C = (1, 1, 1, 2)
    and alpha_0 = 2; for u2 = 1/2 the target is exactly 1 and the first C_j > 1 is j = 3.
    Exact (or extended-precision, or compensated) prefix sums would cross at j = 1."""
    a = np.array([1.0, 2.0 ** -54, 2.0 ** -54, 1.0], np.float32)
    assert oracle.it_one(a, 0.5) == 3
    assert oracle.it_one(a, 0.4999999) == 0


def test_shard_partition_independence():
    # outputs depend only on the global selection index: shards concatenate to the whole
    a = np.array([1, 5, 0.5, 2], np.float32)
    whole = oracle.ar_select(a, 300, seed=5, epoch=3)
    parts = [oracle.ar_select(a, 100, seed=5, epoch=3, s0=s) for s in (0, 100, 200)]
    for key in ("idx", "trials", "tau"):
        np.testing.assert_array_equal(np.concatenate([p[key] for p in parts]), whole[key])


def test_matrix_rows_equal_shared_vector():
    a = np.array([0.3, 1.7, 0.0, 2.2, 0.9], np.float32)
    shared = oracle.ar_select(a, 64, seed=9)
    mat = oracle.ar_select(np.tile(a, (64, 1)), 64, seed=9)
    for key in ("idx", "trials", "tau"):
        np.testing.assert_array_equal(mat[key], shared[key])


def test_power_of_two_scale_invariance():
    a = np.array([0.3, 1.7, 0.0, 2.2, 0.9], np.float32)
    base = oracle.ar_select(a, 500, seed=2)
    for k in (-20, -3, 1, 7, 30):
        r = oracle.ar_select(a * np.float32(2.0**k), 500, seed=2)
        np.testing.assert_array_equal(r["idx"], base["idx"])
        np.testing.assert_array_equal(r["trials"], base["trials"])
        np.testing.assert_array_equal(r["tau"], base["tau"] * np.float32(2.0**-k))
