"""Helper of tests/test_gpu_parity.py::test_matrix_exact_size_allocation (run as a
subprocess, optionally under compute-sanitizer memcheck): matrices whose last element ends
mid-16-byte-chunk, each in an EXACT-size cudaMalloc allocation ((K-1) ld + M floats), so
any byte the library reads past the caller's buffer is an out-of-bounds access memcheck
reports.  No torch: cudart through ctypes, libgpuar through its C ABI.  Exits non-zero on
a parity mismatch with the oracle."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1404_0027_b200 import _abi  # noqa: E402

rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
rt.cudaMalloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t]
rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
rt.cudaFree.argtypes = [ctypes.c_void_p]
H2D, D2H = 1, 2


def dmalloc(nbytes):
    p = ctypes.c_void_p()
    assert rt.cudaMalloc(ctypes.byref(p), nbytes) == 0
    return p


def run(M, K, ld, mode, seed=11):
    rng = np.random.default_rng(M * 7919 + K)
    full = np.zeros((K, ld), np.float32)
    full[:, :M] = (rng.exponential(size=(K, M)) * (rng.random((K, M)) < 0.6)).astype(np.float32)
    n = (K - 1) * ld + M                       # the caller's exact buffer: no padding after the last row
    flat = np.ascontiguousarray(full.reshape(-1)[:n])
    d_a = dmalloc(4 * n)
    rt.cudaMemcpy(d_a, flat.ctypes.data_as(ctypes.c_void_p), 4 * n, H2D)
    outs = [dmalloc(4 * K) for _ in range(3)]
    lib = _abi.load()
    h = ctypes.c_void_p()
    assert lib.gpuar_create(ctypes.byref(h), M, K, seed) == 0
    if mode == "argmin":
        assert lib.gpuar_set_rule(h, _abi.RULE_ARGMIN, 1.0) == 0
    elif mode in ("it", "it_scan"):
        assert lib.gpuar_set_rule(h, _abi.RULE_IT if mode == "it" else _abi.RULE_IT_SCAN, 1.0) == 0
    assert lib.gpuar_set_propensities(h, d_a, K, ld) == 0
    if mode == "stats":
        amax_d, a0_d = dmalloc(4 * K), dmalloc(8 * K)
        assert lib.gpuar_row_stats(h, amax_d, a0_d) == 0
    else:
        assert lib.gpuar_select(h, K, outs[0], outs[1], outs[2]) == 0
    assert lib.gpuar_sync(h) == 0
    rows = full[:, :M]
    if mode == "stats":
        amax = np.empty(K, np.float32)
        rt.cudaMemcpy(amax.ctypes.data_as(ctypes.c_void_p), amax_d, 4 * K, D2H)
        ok = np.array_equal(amax, rows.max(axis=1))
        rt.cudaFree(amax_d)
        rt.cudaFree(a0_d)
    else:
        idx = np.empty(K, np.int32)
        tr = np.empty(K, np.uint32)
        rt.cudaMemcpy(idx.ctypes.data_as(ctypes.c_void_p), outs[0], 4 * K, D2H)
        rt.cudaMemcpy(tr.ctypes.data_as(ctypes.c_void_p), outs[2], 4 * K, D2H)
        if mode == "argmin":
            ref = oracle.argmin_select(np.ascontiguousarray(rows), K, seed=seed, w=1.0, nthreads=4)
            ok = np.array_equal(idx, ref["idx"])
        elif mode in ("it", "it_scan"):
            ok = np.array_equal(idx, oracle.it_select(np.ascontiguousarray(rows), K, seed=seed, nthreads=4))
        else:
            ref = oracle.ar_select(np.ascontiguousarray(rows), K, seed=seed, nthreads=4)
            ok = np.array_equal(idx, ref["idx"]) and np.array_equal(tr, ref["trials"])
    lib.gpuar_destroy(h)
    for p in outs + [d_a]:
        rt.cudaFree(p)
    return ok


MODES = ("classic", "argmin", "stats", "it", "it_scan")


def main():
    bad = []
    # (M, K, ld): last-element ends at 4, 8 or 12 bytes into a 16-byte chunk; tiny rows whose
    # last 1-3 rows all overhang (M = 1, 2 with ld = M); padded pitch
    cases = [(2, 333, 2), (1, 7, 1), (1, 6, 1), (3, 5, 3), (1029, 257, 1029), (5, 4097, 7), (7, 100, 7),
             (1029, 3, 1030)]
    for M, K, ld in cases:
        for mode in MODES:
            if not run(M, K, ld, mode):
                bad.append((M, K, ld, mode))
    if bad:
        print("MISMATCH", bad)
        sys.exit(1)
    print("ok", len(cases) * len(MODES), "cases")


if __name__ == "__main__":
    main()
