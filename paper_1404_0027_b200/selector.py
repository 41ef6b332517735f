"""Thin Python binding over libgpuar (include/gpuar.h): the same operations under the same
names, with torch tensors for device memory and torch's current CUDA stream.  Argument
marshalling only -- every step of the selection runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _abi
from ._abi import check

PATHS = {0: "none", 1: "smem_thresholds", 2: "smem_bracket16", 3: "smem_group_max", 4: "rows"}


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _check_buf(t: torch.Tensor | None, n: int, dtype: torch.dtype, device: torch.device | None, name: str,
               optional: bool = False) -> None:
    """An output buffer handed to the library as a raw pointer: at least n contiguous
    elements of `dtype` on `device` (None: host memory) -- the library writes n elements."""
    if t is None:
        if optional:
            return
        raise ValueError(f"{name} is required")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if device is None:
        if t.device.type != "cpu":
            raise ValueError(f"{name} must be a host tensor")
    elif t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() < n:
        raise ValueError(f"{name} holds {t.numel()} elements, {n} needed")


# The current stream's raw cudaStream_t for a device index: torch's own fast accessor when
# present (a plain int, ~10x cheaper than building a torch.cuda.Stream), else the public API.
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _current_stream_ptr(device: torch.device) -> int:
    if _raw_stream is not None:
        return int(_raw_stream(device.index))
    return torch.cuda.current_stream(device).cuda_stream


class Selector:
    """GPU-AR selector for M reactions and up to K selections per call (gpuar_create).

    Usage::

        sel = Selector(M, K, seed)
        sel.set_propensities(alpha)          # (M,) shared vector or (K, ld) matrix, cuda fp32
        idx, tau, trials = sel.select()      # gpuar_select, epoch += 1
    """

    def __init__(self, M: int, K: int, seed: int, device: int | torch.device | None = None):
        self._lib = _abi.load()
        if device is None:
            index = torch.cuda.current_device()
        elif isinstance(device, int):
            index = device
        else:
            index = torch.device(device).index or 0
        self.device = torch.device("cuda", index)
        self.M, self.K, self.seed = int(M), int(K), int(seed)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self._lib.gpuar_create(ctypes.byref(h), self.M, self.K, self.seed & (2**64 - 1)), "gpuar_create")
        self._h = h
        self._alpha = None      # keeps the borrowed propensity tensor alive
        self._rows = 0
        self._last_stream = None
        self._out_ok = None     # key of the last output buffers select() validated

    # ----------------------------------------------------------------- lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.gpuar_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _stream(self) -> None:
        s = _current_stream_ptr(self.device)
        if s != self._last_stream:  # gpuar_set_stream orders the new stream after the old one
            check(self._lib.gpuar_set_stream(self._h, ctypes.c_void_p(s)), "gpuar_set_stream")
            self._last_stream = s

    # ----------------------------------------------------------------- state
    @property
    def epoch(self) -> int:
        e = ctypes.c_uint32()
        check(self._lib.gpuar_get_epoch(self._h, ctypes.byref(e)), "gpuar_get_epoch")
        return int(e.value)

    @epoch.setter
    def epoch(self, e: int) -> None:
        check(self._lib.gpuar_set_epoch(self._h, int(e) & 0xFFFFFFFF), "gpuar_set_epoch")

    def set_selection_offset(self, s0: int) -> None:
        check(self._lib.gpuar_set_selection_offset(self._h, int(s0)), "gpuar_set_selection_offset")

    def set_rule(self, rule: str = "classic", w: float = 1.0) -> None:
        """gpuar_set_rule: "classic" (first accept, the hot path), "argmin" (the paper's
        printed election + argmin selection with threshold T = w * alpha_max), "it" (the
        classic inverse transform: prefix sums + search) or "it_scan" (the same selection by
        a linear scan of each row, matrix only)."""
        code = {"classic": _abi.RULE_CLASSIC, "argmin": _abi.RULE_ARGMIN, "it": _abi.RULE_IT,
                "it_scan": _abi.RULE_IT_SCAN}[rule]
        check(self._lib.gpuar_set_rule(self._h, code, float(w)), "gpuar_set_rule")

    def set_max_trials(self, n: int) -> None:
        check(self._lib.gpuar_set_max_trials(self._h, int(n)), "gpuar_set_max_trials")

    @property
    def last_team(self) -> int:
        """gpuar_last_team: lanes per selection of the last shared-vector classic select."""
        g = ctypes.c_int32()
        check(self._lib.gpuar_last_team(self._h, ctypes.byref(g)), "gpuar_last_team")
        return int(g.value)

    @property
    def path(self) -> str:
        p = ctypes.c_int32()
        check(self._lib.gpuar_path(self._h, ctypes.byref(p)), "gpuar_path")
        return PATHS[p.value]

    # ----------------------------------------------------------------- registration
    def set_propensities(self, alpha: torch.Tensor) -> None:
        """gpuar_set_propensities: (M,) shared vector or (rows, ld) row-major matrix."""
        if alpha.device.type != "cuda" or alpha.dtype != torch.float32:
            raise TypeError("alpha must be a float32 CUDA tensor")
        if alpha.dim() == 1:
            if alpha.numel() != self.M or not alpha.is_contiguous():
                raise ValueError("shared vector must be contiguous with M elements")
            rows, ld = 1, self.M
        elif alpha.dim() == 2:
            if alpha.stride(1) != 1:
                raise ValueError("matrix rows must be contiguous")
            rows, ld = alpha.shape[0], alpha.stride(0)
            if alpha.shape[1] != self.M:
                raise ValueError("matrix must have M columns (use a padded view for ld > M)")
        else:
            raise ValueError("alpha must be 1-D or 2-D")
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_set_propensities(self._h, _ptr(alpha), rows, ld), "gpuar_set_propensities")
        self._alpha = alpha
        self._rows = rows

    # ----------------------------------------------------------------- selection
    def select(self, K: int | None = None, out: tuple | None = None, with_tau: bool = True,
               with_trials: bool = True):
        """gpuar_select -> (idx int32, tau float32, trials int32-view of uint32) CUDA tensors."""
        K = (self._rows if self._rows > 1 else self.K) if K is None else int(K)
        if out is None:
            idx = torch.empty(K, dtype=torch.int32, device=self.device)
            tau = torch.empty(K, dtype=torch.float32, device=self.device) if with_tau else None
            trials = torch.empty(K, dtype=torch.int32, device=self.device) if with_trials else None
        else:
            idx, tau, trials = out
        p_idx = idx.data_ptr()
        p_tau = None if tau is None else tau.data_ptr()
        p_tr = None if trials is None else trials.data_ptr()
        if out is not None:
            # the full checks once per (buffers, K); a repeat call with the same buffers (the
            # usual SSA / bench loop) only re-keys on their addresses and sizes (~0.3 us
            # instead of ~2.5 us of Python per call, which a launch-bound c1 call would feel)
            key = (p_idx, idx.numel(), p_tau, -1 if tau is None else tau.numel(), p_tr,
                   -1 if trials is None else trials.numel(), K)
            if key != self._out_ok:
                _check_buf(idx, K, torch.int32, self.device, "idx")
                _check_buf(tau, K, torch.float32, self.device, "tau", optional=True)
                _check_buf(trials, K, torch.int32, self.device, "trials", optional=True)
                self._out_ok = key
        # (no torch device context: the library switches to the handle's device itself;
        # raw integer addresses: ctypes converts them for the void* parameters)
        self._stream()
        st = self._lib.gpuar_select(self._h, K, p_idx, p_tau, p_tr)
        if st:
            check(st, "gpuar_select")
        return idx, tau, trials

    def select_epochs(self, n_epochs: int, K: int | None = None, out: tuple | None = None,
                      with_tau: bool = True, with_trials: bool = True):
        """gpuar_select_epochs -> (idx, tau, trials) of shape (n_epochs, K): n_epochs
        consecutive selects in one call (one launch for a shared vector, classic rule)."""
        K = (self._rows if self._rows > 1 else self.K) if K is None else int(K)
        n = int(n_epochs)
        if out is None:
            idx = torch.empty((n, K), dtype=torch.int32, device=self.device)
            tau = torch.empty((n, K), dtype=torch.float32, device=self.device) if with_tau else None
            trials = torch.empty((n, K), dtype=torch.int32, device=self.device) if with_trials else None
        else:
            idx, tau, trials = out
        _check_buf(idx, n * K, torch.int32, self.device, "idx")
        _check_buf(tau, n * K, torch.float32, self.device, "tau", optional=True)
        _check_buf(trials, n * K, torch.int32, self.device, "trials", optional=True)
        self._stream()
        st = self._lib.gpuar_select_epochs(self._h, K, n, idx.data_ptr(), None if tau is None else tau.data_ptr(),
                                           None if trials is None else trials.data_ptr())
        if st:
            check(st, "gpuar_select_epochs")
        return idx, tau, trials

    def select_host(self, alpha: np.ndarray | torch.Tensor, K: int | None = None, out: tuple | None = None):
        """gpuar_select_host: host (ideally pinned) propensities in, host outputs out."""
        a = alpha if isinstance(alpha, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(alpha, np.float32))
        if a.dtype != torch.float32 or a.device.type != "cpu":
            raise TypeError("alpha must be a float32 host array")
        if a.dim() == 1:
            if a.numel() != self.M or not a.is_contiguous():
                raise ValueError("shared vector must be contiguous with M elements")
            rows, ld = 1, self.M
        elif a.dim() == 2:
            if a.shape[1] != self.M or a.stride(1) != 1:
                raise ValueError("matrix must have M contiguous columns (pitch = stride(0))")
            rows, ld = a.shape[0], a.stride(0)
        else:
            raise ValueError("alpha must be 1-D or 2-D")
        K = (rows if rows > 1 else self.K) if K is None else int(K)
        if out is None:
            pin = a.is_pinned()
            idx = torch.empty(K, dtype=torch.int32, pin_memory=pin)
            tau = torch.empty(K, dtype=torch.float32, pin_memory=pin)
            trials = torch.empty(K, dtype=torch.int32, pin_memory=pin)
        else:
            idx, tau, trials = out
        _check_buf(idx, K, torch.int32, None, "idx")
        _check_buf(tau, K, torch.float32, None, "tau")
        _check_buf(trials, K, torch.int32, None, "trials")
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_select_host(self._h, _ptr(a), rows, ld, K, _ptr(idx), _ptr(tau), _ptr(trials)),
                  "gpuar_select_host")
        self._alpha = None
        self._rows = 0
        return idx, tau, trials

    # ----------------------------------------------------------------- full SSA (NEXT-2)
    def set_network(self, reac: torch.Tensor, rate: torch.Tensor, didx: torch.Tensor, dval: torch.Tensor,
                    N: int) -> None:
        """gpuar_set_network: mass-action network (cuda int32 reac (M,2), float32 rate (M,),
        int32 didx/dval (M,D)); tensors are kept alive by the selector."""
        D = didx.shape[1]
        with torch.cuda.device(self.device):
            check(self._lib.gpuar_set_network(self._h, int(N), int(D), _ptr(reac), _ptr(rate), _ptr(didx), _ptr(dval)),
                  "gpuar_set_network")
        self._net = (reac, rate, didx, dval)
        self._net_N = int(N)

    def ssa_run(self, X: torch.Tensor, t: torch.Tensor, n_steps: int, t_end: float = float("inf"),
                steps: torch.Tensor | None = None) -> torch.Tensor:
        """gpuar_ssa_run: advance K realizations in place (X (K,N) int32, t (K,) float64)."""
        K = X.shape[0]
        N = getattr(self, "_net_N", None)
        if X.dim() != 2 or (N is not None and X.shape[1] != N):
            raise ValueError("X must be (K, N) with the registered network's N species")
        _check_buf(X, X.numel(), torch.int32, self.device, "X")
        _check_buf(t, K, torch.float64, self.device, "t")
        if steps is None:
            steps = torch.zeros(K, dtype=torch.int32, device=self.device)
        _check_buf(steps, K, torch.int32, self.device, "steps")
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_ssa_run(self._h, _ptr(X), _ptr(t), _ptr(steps), K, int(n_steps), float(t_end)),
                  "gpuar_ssa_run")
        return steps

    # ----------------------------------------------------------------- statistics / validation
    def stats(self) -> tuple[float, float, float]:
        amax, a0, p = ctypes.c_float(), ctypes.c_double(), ctypes.c_float()
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_get_stats(self._h, ctypes.byref(amax), ctypes.byref(a0), ctypes.byref(p)),
                  "gpuar_get_stats")
        return float(amax.value), float(a0.value), float(p.value)

    def row_stats(self) -> tuple[torch.Tensor, torch.Tensor]:
        amax = torch.empty(self._rows, dtype=torch.float32, device=self.device)
        a0 = torch.empty(self._rows, dtype=torch.float64, device=self.device)
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_row_stats(self._h, _ptr(amax), _ptr(a0)), "gpuar_row_stats")
        return amax, a0

    def sync(self) -> None:
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_sync(self._h), "gpuar_sync")

    def histogram(self, idx: torch.Tensor, trials: torch.Tensor | None, hist: torch.Tensor | None = None,
                  totals: torch.Tensor | None = None):
        """gpuar_histogram: hist[M+1] (bin M = idx -1) and totals = (sum trials, #rejected), int64."""
        if hist is None:
            hist = torch.zeros(self.M + 1, dtype=torch.int64, device=self.device)
        if totals is None:
            totals = torch.zeros(2, dtype=torch.int64, device=self.device)
        _check_buf(idx, idx.numel(), torch.int32, self.device, "idx")
        _check_buf(trials, idx.numel(), torch.int32, self.device, "trials", optional=True)
        _check_buf(hist, self.M + 1, torch.int64, self.device, "hist")
        _check_buf(totals, 2, torch.int64, self.device, "totals")
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_histogram(self._h, _ptr(idx), _ptr(trials), idx.numel(), _ptr(hist), _ptr(totals)),
                  "gpuar_histogram")
        return hist, totals

    def bench_philox(self, n_threads: int, calls: int, sink: torch.Tensor) -> None:
        with torch.cuda.device(self.device):
            self._stream()
            check(self._lib.gpuar_bench_philox(self._h, int(n_threads), int(calls), _ptr(sink)), "gpuar_bench_philox")
