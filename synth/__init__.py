"""Seeded synthetic propensity generators -- the ONE module both the oracle side and the
CUDA side draw inputs from.  It holds none of the selection method's arithmetic (no
Philox, no acceptance test, no reductions): it only manufactures alpha vectors/matrices
with the shapes and value distributions of the paper's workloads (DESIGN.md "Input
recipe").

Shared vectors are drawn on the host with numpy's PCG64 (bit-stable for a given numpy
version) and cast to binary32 once; the same host buffer is uploaded to the GPU and
handed to the oracle.

Per-realization K x M matrices (config c4, 4 GiB at K=2^20) are defined cell by cell
by an integer-only counter hash, so any row can be regenerated anywhere: row k, column
j is ``rates[j]`` if bit 63 of ``mix64(gen_seed, k*M + j)`` is set, else 0 (a Bernoulli(1/2)
enable mask over yeast-like rate constants -- species on/off as in the paper's boolean
SSA of the iron model).  ``synth/synth_rows.cu`` is the same recipe as a
CUDA kernel (libsynth.so) so the bench can fill 4 GiB in HBM in milliseconds;
tests/test_synth.py checks the two agree bit for bit.
"""
from __future__ import annotations

import math

import numpy as np

GEN_SEED = 14040027          # default generator seed
SELECT_SEED = 20140327       # default selection seed
YEAST_M = 1029               # reactions of the iron-homeostasis model
YEAST_FAST = 40              # "fast" reactions (DESIGN.md input recipe)

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def mix64(gen_seed: int, counter: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser of gen_seed + (counter + 1) * golden (wrapping uint64)."""
    with np.errstate(over="ignore"):
        z = np.uint64(gen_seed & (2**64 - 1)) + (np.asarray(counter, np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def _rng(gen_seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(gen_seed))


# ----------------------------------------------------------------- shared vectors

def hand(values) -> np.ndarray:
    """Hand-set propensities, e.g. {1,2,3,4} of config c1."""
    return np.asarray(values, np.float32)


def discrete_gaussian(M: int) -> np.ndarray:
    """x_j = -5 + j*10/(M-1), D_j = phi(x_j) * 1e5 (M = 64, 256, 1024)."""
    x = -5.0 + np.arange(M, dtype=np.float64) * (10.0 / (M - 1))
    d = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi) * 1e5
    return d.astype(np.float32)


def uniform(M: int, gen_seed: int = GEN_SEED) -> np.ndarray:
    """alpha_j = 1 - m_j 2^-24, m_j uniform on [0, 2^24): uniform on (0, 1], exact in binary32."""
    m = _rng(gen_seed).integers(0, 1 << 24, size=M, dtype=np.int64)
    return (1.0 - m.astype(np.float64) * 2.0**-24).astype(np.float32)


def exponential(M: int, gen_seed: int = GEN_SEED) -> np.ndarray:
    """alpha_j ~ Exp(1)."""
    a = _rng(gen_seed).standard_exponential(M).astype(np.float32)
    return np.maximum(a, np.float32(2.0**-24))


def pareto(M: int, gen_seed: int = GEN_SEED, tail: float = 1.5) -> np.ndarray:
    """Heavy tail: Pareto(x_m = 1, shape `tail`), alpha_j = U^(-1/tail)."""
    u = 1.0 - _rng(gen_seed).random(M)               # (0, 1]
    return (u ** (-1.0 / tail)).astype(np.float32)


def yeast_rates(M: int = YEAST_M, gen_seed: int = GEN_SEED, n_fast: int = YEAST_FAST) -> np.ndarray:
    """Yeast-like rate constants (the iron model's data is unpublished):
    bulk 10^U(-1,1), plus n_fast reactions at 100 * 10^U(-1,1)."""
    rng = _rng(gen_seed)
    r = 10.0 ** rng.uniform(-1.0, 1.0, M)
    fast = rng.choice(M, size=min(n_fast, M), replace=False)
    r[fast] = 100.0 * 10.0 ** rng.uniform(-1.0, 1.0, fast.size)
    return r.astype(np.float32)


def yeast_like(M: int = YEAST_M, gen_seed: int = GEN_SEED) -> np.ndarray:
    """Shared yeast-like vector (config c2): rates times a Bernoulli(1/2) enable mask
    (row 0 of the matrix recipe, so c2 and c4 share their family)."""
    return rows(yeast_rates(M, gen_seed), gen_seed, 0, 1)[0]


def distribution(kind: str, M: int, gen_seed: int = GEN_SEED) -> np.ndarray:
    kinds = {"uniform": uniform, "exponential": exponential, "pareto": pareto}
    if kind == "yeast":
        return yeast_like(M, gen_seed)
    if kind == "gaussian":
        return discrete_gaussian(M)
    return kinds[kind](M, gen_seed)


# ----------------------------------------------------------------- per-realization matrix

def rows(rates: np.ndarray, gen_seed: int, k0: int, n: int, ld: int | None = None) -> np.ndarray:
    """Rows k0 .. k0+n-1 (GLOBAL row indices) of the per-realization matrix, shape (n, ld),
    padding columns (j >= M) zero.  Cell (k, j) = rates[j] if bit 63 of mix64(gen_seed,
    k*M + j) else 0."""
    rates = np.asarray(rates, np.float32)
    M = rates.size
    ld = M if ld is None else ld
    k = np.arange(k0, k0 + n, dtype=np.uint64)[:, None]
    j = np.arange(M, dtype=np.uint64)[None, :]
    bit = (mix64(gen_seed, k * np.uint64(M) + j) >> np.uint64(63)).astype(bool)
    out = np.zeros((n, ld), np.float32)
    out[:, :M] = np.where(bit, rates[None, :], np.float32(0.0))
    return out


# ----------------------------------------------------------------- reaction networks (NEXT-2)
# A network is a dict of int32/float32 arrays: reac (M,2) reactant species (-1 = none),
# rate (M,) mass-action constants, didx/dval (M,D) sparse state-change vector v_j
# (species -1 = unused slot).  Shapes only -- the propensity arithmetic is not here.

def immigration_death(k: float = 10.0, gamma: float = 1.0) -> dict:
    """0 -> X (rate k), X -> 0 (rate gamma X): X(t) ~ Poisson(k/gamma (1 - e^-gamma t)) from
    X(0) = 0 (SPEC.md:418-419 uses the stationary mean 10)."""
    return dict(reac=np.array([[-1, -1], [0, -1]], np.int32), rate=np.array([k, gamma], np.float32),
                didx=np.array([[0], [0]], np.int32), dval=np.array([[1], [-1]], np.int32), N=1)


def dimerisation(kf: float = 0.01, kb: float = 0.5) -> dict:
    """2A -> B (rate kf A(A-1)/2), B -> 2A (rate kb B): A + 2B is conserved."""
    return dict(reac=np.array([[0, 0], [1, -1]], np.int32), rate=np.array([kf, kb], np.float32),
                didx=np.array([[0, 1], [0, 1]], np.int32), dval=np.array([[-2, 1], [2, -1]], np.int32), N=2)


def yeast_like_network(N: int = 641, M: int = YEAST_M, gen_seed: int = GEN_SEED, D: int = 4) -> dict:
    """A random mass-action network with the iron model's size (641 species, 1029 reactions,
    PAPER.md:86-89; the model itself is unpublished): 15 % zeroth-order productions, 50 %
    first-order (degradation or conversion), 35 % second-order (5 % of them dimerisations);
    rates from yeast_rates, second-order ones scaled by 1e-2."""
    rng = _rng(gen_seed + 7)
    rates = yeast_rates(M, gen_seed).astype(np.float64)
    reac = np.full((M, 2), -1, np.int32)
    didx = np.full((M, D), -1, np.int32)
    dval = np.zeros((M, D), np.int32)
    for j in range(M):
        order = rng.choice(3, p=[0.15, 0.50, 0.35])
        if order >= 1:
            reac[j, 0] = rng.integers(N)
        if order == 2:
            reac[j, 1] = reac[j, 0] if rng.random() < 0.05 else rng.integers(N)
            rates[j] *= 1e-2
        delta = {}
        for r in reac[j]:
            if r >= 0:
                delta[int(r)] = delta.get(int(r), 0) - 1
        for _ in range(rng.integers(0, 3) if order > 0 else 1):
            sp = int(rng.integers(N))
            delta[sp] = delta.get(sp, 0) + 1
        items = [(sp, v) for sp, v in delta.items() if v != 0][:D]
        for d, (sp, v) in enumerate(items):
            didx[j, d], dval[j, d] = sp, v
    return dict(reac=reac, rate=rates.astype(np.float32), didx=didx, dval=dval, N=N)


def initial_state(N: int, K: int, gen_seed: int = GEN_SEED, high: int = 10) -> np.ndarray:
    """K x N initial copy numbers, uniform on [0, high)."""
    return _rng(gen_seed + 11).integers(0, high, size=(K, N), dtype=np.int32)
