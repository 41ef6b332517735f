"""CPU oracle for GPU acceptance-rejection next-reaction selection (arXiv 1404.0027).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product
package ``paper_1404_0027_b200`` never imports it, and the two share no code.

The arithmetic lives in ``oracle/oracle.c`` (plain C, binary32 round-to-nearest, no
FMA contraction, see its header for the passage each step follows); this module only
compiles it (gcc) and marshals numpy arrays through ctypes.  The statistical helpers
at the bottom (exact law, chi-square, MSE) are plain numpy/scipy definitions.

Parity pins: every function here is pinned by ``tests/test_oracle_*.py`` against the
Random123 known-answer vectors, closed forms, hand-worked cases, exact probabilities
(chi-square) and invariants -- see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", "-Wall", "-Wextra"]
_lock = threading.Lock()
_lib = None

OK = 0
EPROPENSITY = -5


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc).  Returns the library path."""
    with _lock:
        stale = (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
        if force or stale:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.run(["gcc", *_CFLAGS, "-o", tmp, _SRC, "-lm"], check=True)
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
        lib.oracle_philox4x32_10.restype = None
        lib.oracle_index.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        lib.oracle_index.restype = ctypes.c_uint32
        lib.oracle_unit.argtypes = [ctypes.c_uint32]
        lib.oracle_unit.restype = ctypes.c_float
        lib.oracle_unit_open.argtypes = [ctypes.c_uint32]
        lib.oracle_unit_open.restype = ctypes.c_float
        lib.oracle_accept.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
        lib.oracle_accept.restype = ctypes.c_int
        lib.oracle_stats.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double)]
        lib.oracle_stats.restype = ctypes.c_int
        lib.oracle_it_one.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_float]
        lib.oracle_it_one.restype = ctypes.c_int32
        lib.oracle_ar_batch.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_ar_batch.restype = ctypes.c_int
        lib.oracle_it_batch.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int]
        lib.oracle_it_batch.restype = ctypes.c_int
        lib.oracle_argmin_batch.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_float,
            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int]
        lib.oracle_argmin_batch.restype = ctypes.c_int
        lib.oracle_election.argtypes = [ctypes.c_float, ctypes.c_float, ctypes.c_float]
        lib.oracle_election.restype = ctypes.c_float
        lib.oracle_selection.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.oracle_selection.restype = ctypes.c_int32
        lib.oracle_propensity.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_float]
        lib.oracle_propensity.restype = ctypes.c_float
        lib.oracle_ssa_run.argtypes = [
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
            ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
        lib.oracle_ssa_run.restype = ctypes.c_int
        lib.oracle_histogram.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_histogram.restype = None
        _lib = lib
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------- primitives

def philox4x32_10(ctr, key) -> tuple:
    """Philox4x32-10 block function (Salmon et al. SC'11) -> 4 uint32 words."""
    lib = _load()
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib.oracle_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def index_of(x: int, M: int) -> int:
    """Candidate index j = floor(x*M/2^32) (R5)."""
    return int(_load().oracle_index(x & 0xFFFFFFFF, M))


def unit(x: int) -> float:
    """u = (x>>8) * 2^-24 in [0,1) (R3)."""
    return float(_load().oracle_unit(x & 0xFFFFFFFF))


def unit_open(x: int) -> float:
    """u1 = (2(x>>9)+1) * 2^-24 in (0,1) (R10)."""
    return float(_load().oracle_unit_open(x & 0xFFFFFFFF))


def accept(u: float, amax: float, alpha_j: float) -> bool:
    """PAPER.md:296 acceptance test fl32(u*T) < alpha_j."""
    return bool(_load().oracle_accept(u, amax, alpha_j))


def stats(alpha) -> tuple[float, float, int]:
    """(alpha_max, alpha_0, status) -- PAPER.md:259-260, 361-365."""
    a = _f32(alpha)
    amax = ctypes.c_float()
    a0 = ctypes.c_double()
    st = _load().oracle_stats(_ptr(a), a.size, ctypes.byref(amax), ctypes.byref(a0))
    return float(amax.value), float(a0.value), int(st)


def it_one(alpha, u2: float) -> int:
    """Inverse transform, linear search."""
    a = _f32(alpha)
    _, a0, _ = stats(a)
    return int(_load().oracle_it_one(_ptr(a), a.size, a0, u2))


# ----------------------------------------------------------------- batches

def ar_select(alpha, K: int, seed: int, epoch: int = 0, s0: int = 0,
              max_trials: int = 1 << 20, M: int | None = None, nthreads: int = 1) -> dict:
    """K classic-AR selections on the canonical Philox stream.

    ``alpha`` is a 1-D shared vector (M,) or a 2-D per-realization matrix (K, ld);
    ``M`` defaults to the last dimension.  Returns numpy arrays idx (int32, -1 =
    rejected/degenerate), tau (float32), trials (uint32), tau_ref (float64), and the
    per-selection amax (float32) / a0 (float64) plus the call's status code.
    """
    a = _f32(alpha)
    if a.ndim == 1:
        rows, ld = 1, a.shape[0]
    else:
        rows, ld = a.shape[0], a.shape[1]
        if rows != K:
            raise ValueError("matrix rows must equal K")
    M = ld if M is None else M
    idx = np.empty(K, np.int32)
    tau = np.empty(K, np.float32)
    trials = np.empty(K, np.uint32)
    amax = np.empty(K, np.float32)
    a0 = np.empty(K, np.float64)
    tau_ref = np.empty(K, np.float64)
    st = _load().oracle_ar_batch(_ptr(a), M, rows, ld, K, seed & (2**64 - 1), s0, epoch,
                                 max_trials, _ptr(idx), _ptr(tau), _ptr(trials),
                                 _ptr(amax), _ptr(a0), _ptr(tau_ref), nthreads)
    return dict(idx=idx, tau=tau, trials=trials, amax=amax, a0=a0, tau_ref=tau_ref, status=int(st))


def it_select(alpha, K: int, seed: int, epoch: int = 0, s0: int = 0,
              M: int | None = None, nthreads: int = 1) -> np.ndarray:
    """K inverse-transform selections on uniform stream tag 2."""
    a = _f32(alpha)
    if a.ndim == 1:
        rows, ld = 1, a.shape[0]
    else:
        rows, ld = a.shape[0], a.shape[1]
    M = ld if M is None else M
    idx = np.empty(K, np.int32)
    _load().oracle_it_batch(_ptr(a), M, rows, ld, K, seed & (2**64 - 1), s0, epoch, _ptr(idx), nthreads)
    return idx


def election(alpha_j: float, v: float, T: float) -> float:
    """Election step: R = fl32(v T)/alpha_j if fl32(v T) < alpha_j else 1."""
    return float(_load().oracle_election(alpha_j, v, T))


def selection(ratings) -> int:
    """Selection step: argmin, ties to the lowest index, -1 if min >= 1."""
    r = _f32(ratings)
    return int(_load().oracle_selection(_ptr(r), r.size))


def argmin_select(alpha, K: int, seed: int, w: float = 1.0, epoch: int = 0, s0: int = 0,
                  M: int | None = None, nthreads: int = 1) -> dict:
    """The paper's printed GPU/AR rule (election + argmin selection, PAPER.md:304-380,
    498-560) on Philox stream tag 3, threshold T = fl32(w * alpha_max).  Returns idx (int32,
    -1 = rejected/degenerate), tau, tau_ref and the status."""
    a = _f32(alpha)
    if a.ndim == 1:
        rows, ld = 1, a.shape[0]
    else:
        rows, ld = a.shape[0], a.shape[1]
        if rows != K:
            raise ValueError("matrix rows must equal K")
    M = ld if M is None else M
    idx = np.empty(K, np.int32)
    tau = np.empty(K, np.float32)
    tau_ref = np.empty(K, np.float64)
    st = _load().oracle_argmin_batch(_ptr(a), M, rows, ld, K, float(w), seed & (2**64 - 1), s0, epoch,
                                     _ptr(idx), _ptr(tau), _ptr(tau_ref), nthreads)
    return dict(idx=idx, tau=tau, tau_ref=tau_ref, status=int(st))


def argmin_law(alpha, w: float = 1.0, reject: bool = False):
    """Exact law of the argmin rule with continuous uniforms:
    P(j) = int_0^1 (D_j/T) prod_{i != j} (1 - r D_i/T) dr,  T = w max D.
    The integrand is a polynomial of degree M-1 in r, so Gauss-Legendre with ceil(M/2)+1
    nodes is exact.  With reject=True also returns P(rejected) = prod_i (1 - D_i/T)."""
    d = np.asarray(alpha, np.float64) / (w * float(np.max(alpha)))
    M = d.size
    x, wts = np.polynomial.legendre.leggauss(M // 2 + 2)
    r = 0.5 * (x + 1.0)
    wts = 0.5 * wts
    one_minus = 1.0 - np.outer(r, d)                      # (nodes, M)
    with np.errstate(divide="ignore"):
        logs = np.log(np.abs(one_minus))
    zero = one_minus == 0.0
    # prod over i != j: exp(sum log - log_j), handling exact zeros (d_i = 1 at r = 1 only)
    total = logs.sum(axis=1, keepdims=True)
    prod_except = np.exp(total - logs)
    nz = zero.sum(axis=1, keepdims=True)
    prod_except = np.where(nz == 0, prod_except, 0.0)
    P = (d[None, :] * prod_except * wts[:, None]).sum(axis=0)
    if reject:
        return P, float(np.prod(1.0 - d))
    return P


def propensity(X, r0: int, r1: int, c: float) -> float:
    """Mass-action propensity (R20)."""
    x = np.ascontiguousarray(X, np.int32)
    return float(_load().oracle_propensity(_ptr(x), r0, r1, c))


def ssa_run(net: dict, X0, t0, n_steps: int, seed: int, t_end: float = float("inf"), epoch0: int = 0,
            s0: int = 0, max_trials: int = 1 << 20, nthreads: int = 1) -> dict:
    """K SSA realizations of the network net = {reac (M,2) int32,
    rate (M,) float32, didx (M,D) int32, dval (M,D) int32}; X0 (K,N) int32, t0 (K,) float64.
    Returns X, t, steps (events fired) and the status."""
    reac = np.ascontiguousarray(net["reac"], np.int32)
    rate = _f32(net["rate"])
    didx = np.ascontiguousarray(net["didx"], np.int32)
    dval = np.ascontiguousarray(net["dval"], np.int32)
    X = np.array(X0, dtype=np.int32, order="C", copy=True)
    t = np.array(t0, dtype=np.float64, copy=True)
    K, N = X.shape
    M, D = didx.shape
    steps = np.zeros(K, np.uint32)
    st = _load().oracle_ssa_run(N, M, D, _ptr(reac), _ptr(rate), _ptr(didx), _ptr(dval), K, _ptr(X), _ptr(t),
                                _ptr(steps), n_steps, t_end, seed & (2**64 - 1), s0, epoch0, max_trials, nthreads)
    return dict(X=X, t=t, steps=steps, status=int(st))


def histogram(idx, trials, M: int) -> tuple[np.ndarray, int]:
    """hist[M+1] (bin M = rejected/degenerate) and the sum of trials."""
    i = np.ascontiguousarray(idx, np.int32)
    t = np.ascontiguousarray(trials, np.uint32)
    h = np.zeros(M + 1, np.uint64)
    ts = ctypes.c_uint64()
    _load().oracle_histogram(_ptr(i), _ptr(t), i.size, M, _ptr(h), ctypes.byref(ts))
    return h, int(ts.value)


# ----------------------------------------------------------------- exact law & metrics

def exact_law(alpha) -> np.ndarray:
    """P(idx = j) = alpha_j / alpha_0 -- the law the SSA direct method samples
    (PAPER.md:270-275); classic AR conditioned on acceptance has the same law."""
    a = np.asarray(alpha, np.float64)
    return a / a.sum()


def acceptance_rate(alpha) -> float:
    """Per-trial acceptance probability p = alpha_0 / (M * alpha_max) (north_star)."""
    a = np.asarray(alpha, np.float64)
    return float(a.sum() / (a.size * a.max()))


def chi2_pvalue(counts, probs, min_expected: float = 5.0) -> tuple[float, float, int]:
    """Pearson chi-square goodness of fit, bins with expected < min_expected pooled.
    Returns (statistic, p-value, dof)."""
    from scipy.stats import chi2 as _chi2
    counts = np.asarray(counts, np.float64)
    probs = np.asarray(probs, np.float64)
    n = counts.sum()
    exp = probs * n
    keep = exp >= min_expected
    obs_k, exp_k = counts[keep], exp[keep]
    if (~keep).any():
        obs_k = np.append(obs_k, counts[~keep].sum())
        exp_k = np.append(exp_k, exp[~keep].sum())
    mask = exp_k > 0
    obs_k, exp_k = obs_k[mask], exp_k[mask]
    stat = float(((obs_k - exp_k) ** 2 / exp_k).sum())
    dof = max(int(obs_k.size) - 1, 1)
    return stat, float(_chi2.sf(stat, dof)), dof


def mse_normalized(target, counts) -> float:
    """MSE = (1/M) sum_j (D_j - O_j)^2 of the normalised vectors."""
    d = np.asarray(target, np.float64)
    o = np.asarray(counts, np.float64)
    d = d / d.sum()
    o = o / o.sum()
    return float(np.mean((d - o) ** 2))
