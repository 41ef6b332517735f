"""GPU side of the matrix recipe in synth/__init__.py (libsynth.so, synth/synth_rows.cu):
fills a CUDA tensor with rows k0 .. k0+n-1 of the per-realization matrix.  Input
generation only."""
from __future__ import annotations

import ctypes
import os

import torch

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB)
        lib.synth_rows.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        lib.synth_rows.restype = ctypes.c_int
        _lib = lib
    return _lib


def fill_rows(out: torch.Tensor, rates: torch.Tensor, gen_seed: int, k0: int) -> torch.Tensor:
    """out: (n, ld) float32 CUDA tensor (row-contiguous); rates: (M,) float32 CUDA tensor."""
    n, M = out.shape[0], rates.numel()
    ld = out.stride(0) if out.dim() == 2 else M
    st = torch.cuda.current_stream(out.device).cuda_stream
    rc = _load().synth_rows(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(rates.data_ptr()), M, ld, k0, n,
                            gen_seed & (2**64 - 1), ctypes.c_void_p(st))
    if rc != 0:
        raise RuntimeError(f"synth_rows failed ({rc})")
    return out
