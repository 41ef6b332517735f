"""The C-ABI library builds, loads without a GPU and exports every entry point
include/gpuar.h declares; the product never touches the oracle (and vice versa)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpuar.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gpuar_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1404_0027_b200 import _build
    _build.build()
    from paper_1404_0027_b200 import _abi
    return _abi.load()


def test_every_declared_symbol_exported(lib):
    from paper_1404_0027_b200 import _abi
    names = _declared()
    assert len(names) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.library_path()], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (gpuar_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(_abi.SIGNATURES), "binding must cover exactly the header"
    for n in names:
        assert hasattr(lib, n)


def test_strerror_and_argument_errors_without_gpu(lib):
    assert lib.gpuar_strerror(0) == b"success"
    assert b"invalid propensity" in lib.gpuar_strerror(-5)
    h = ctypes.c_void_p()
    assert lib.gpuar_create(ctypes.byref(h), 0, 10, 1) == -1      # M < 1
    assert lib.gpuar_create(ctypes.byref(h), 4, 0, 1) == -1       # K < 1
    assert lib.gpuar_create(None, 4, 4, 1) == -1
    assert lib.gpuar_select(None, 4, None, None, None) == -1
    assert lib.gpuar_destroy(None) == 0


def test_sm100a_code_in_library(lib):
    from paper_1404_0027_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _abi.library_path()], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass            # 1-D bulk async copy (row staging)
    assert "SYNCS" in sass             # mbarrier


def test_product_and_oracle_share_nothing():
    pkg = os.path.join(ROOT, "paper_1404_0027_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", s, re.M), f
                assert "oracle.c" not in s and "liboracle" not in s, f
    osrc = open(os.path.join(ROOT, "oracle", "oracle.c")).read()
    assert "#include \"" not in osrc                       # only system headers
    opy = open(os.path.join(ROOT, "oracle", "__init__.py")).read()
    assert not re.search(r"^\s*(import|from)\s+(paper_1404_0027_b200|synth)\b", opy, re.M)
