"""Build libgpuar.so (and the input generator libsynth.so) in-tree for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false: every binary32
multiply/add in the kernels is a separately rounded IEEE operation (the acceptance
test is bit-compared against the CPU oracle, R4).
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIBGPUAR = os.path.join(LIBDIR, "libgpuar.so")
SYNTH_SRC = os.path.join(ROOT, "synth", "synth_rows.cu")
LIBSYNTH = os.path.join(ROOT, "synth", "libsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-shared", "-Xcompiler", "-fPIC"]

SOURCES = ["gpuar_api.cu", "kernels_misc.cu", "kernels_select.cu", "kernels_rows.cu", "kernels_argmin.cu", "kernels_ssa.cu", "kernels_it.cu"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _nvcc(out: str, srcs: list[str], extra: list[str] | None = None) -> None:
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, *(extra or []), "-o", tmp, *srcs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)


def build(force: bool = False, verbose_ptxas: bool = False) -> list[str]:
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "gpuar.h"))
    if force or _stale(LIBGPUAR, deps):
        _nvcc(LIBGPUAR, srcs, ["-Xptxas", "-v"] if verbose_ptxas else None)
    if force or _stale(LIBSYNTH, [SYNTH_SRC]):
        _nvcc(LIBSYNTH, [SYNTH_SRC])
    return [LIBGPUAR, LIBSYNTH]


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv))
