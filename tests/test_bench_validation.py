"""bench.py's validation law for a shared vector (law_and_trials): the exact law of the
DISCRETE draws -- index words n_j = #{x < 2^32 : (x M) >> 32 = j}, acceptance counts
T_j = #{v < 2^24 : fl32(fl32(v 2^-24) alpha_max) < alpha_j} -- checked against brute force
of those definitions and against closed forms (CPU; untimed validation code, not the
product path)."""
import importlib.util
import os

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ceil_div(a, b):
    return -(-a // b)


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_hand_vector_is_exact():
    """{1,2,3,4}: every u alpha_max is exact, so T_j = alpha_j / 4 * 2^24 and n_j = 2^30:
    the law is alpha / 10 and p = 0.625 exactly (SURVEY §8(c) pins)."""
    law, e, v, p = _bench().law_and_trials({"M": 4}, None, torch.tensor([1.0, 2.0, 3.0, 4.0]))
    assert p == 0.625 and e == 1.6
    np.testing.assert_array_equal(law.numpy(), np.array([0.1, 0.2, 0.3, 0.4]))


def test_thresholds_and_index_counts_by_brute_force():
    """T_j by enumerating all 2^24 uniforms; n_j for M = 3 from the index pins
    (0x55555555 -> 0, 0x55555556 -> 1, 0xAAAAAAAA -> 1, 0xAAAAAAAB -> 2)."""
    a = np.array([1.0, 1e-6, 0.3, 0.7000001, 2.5e-3], np.float32)
    amax = np.float32(a.max())
    u = (np.arange(1 << 24, dtype=np.float32) * np.float32(2.0 ** -24)) * amax   # fl32 RN products
    T = np.array([np.count_nonzero(u < x) for x in a], np.float64)
    M = a.size
    # n_j = #{x : floor(x M / 2^32) = j} = ceil((j+1) 2^32 / M) - ceil(j 2^32 / M)
    n = np.array([_ceil_div((j + 1) << 32, M) - _ceil_div(j << 32, M) for j in range(M)], np.float64)
    law, e, v, p = _bench().law_and_trials({"M": M}, None, torch.from_numpy(a))
    np.testing.assert_allclose(law.numpy(), n * T / (n * T).sum(), rtol=1e-15)
    assert abs(p - (n * T).sum() / 2.0 ** 56) <= 1e-15 * p
    assert T[1] == 17            # 1e-6 * 2^24 = 16.78: v = 0..16 accepted
    n3 = [_ceil_div((j + 1) << 32, 3) - _ceil_div(j << 32, 3) for j in range(3)]
    assert n3 == [0x55555556, 0xAAAAAAAB - 0x55555556, (1 << 32) - 0xAAAAAAAB]


def test_quantisation_moves_p_only_for_tiny_ratios():
    """The discrete p exceeds the continuum a0/(M alpha_max) by ~0.5 * 2^-24 per reaction
    relative to alpha_max: negligible on the yeast-like vector, visible on a heavy tail."""
    import synth
    b = _bench()
    for vec, bound in ((synth.yeast_like(), 2e-4), (synth.pareto(100_000), 5e-3)):
        t = torch.from_numpy(vec)
        p = b.law_and_trials({"M": vec.size}, None, t)[3]
        pc = float(t.double().sum() / (vec.size * t.double().max()))
        assert 0.0 <= p / pc - 1.0 < bound
