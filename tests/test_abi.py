"""CPU-side checks of the C ABI library (no GPU needed, no compute calls).

* libhpnfft.so loads and exports every function declared in include/hpnfft.h;
* argument validation is host logic that runs before any CUDA call, so its status codes are
  checked here (SURVEY.md §8(b) contract table);
* the product package never imports the oracle.
"""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hpnfft.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2001_01583_b200 import build as pb

    pb.build()
    import paper_2001_01583_b200 as hp

    return hp.load_library()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hpnfft_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert {"hpnfft_plan", "hpnfft_set_points", "hpnfft_adjoint", "hpnfft_destroy"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {lib._name}").read()
    for name in names:
        assert re.search(rf"\bT {name}\b", out), name


def test_version_string(lib):
    import paper_2001_01583_b200 as hp

    assert "sm_100a" in hp.version()


def _plan(lib, N, M=10, m=6, sigma=2.0, window=0, d=None):
    h = ctypes.c_void_p()
    d = len(N) if d is None else d
    arr = (ctypes.c_int64 * max(len(N), 1))(*N)
    rc = lib.hpnfft_plan(ctypes.byref(h), d, arr, M, m, sigma, window, None)
    return rc, h


@pytest.mark.parametrize("N,kw,code", [
    ((15, 16, 16), {}, -1),            # odd bandwidth (N_t in 2N)
    ((0, 16, 16), {}, -1),
    ((16, 16, 16, 16), {}, -2),        # d = 4 (the oracle and the GPU cover d = 1..3)
    ((16, 16, 16), {"m": 16}, -2),     # m outside PAPER.md:266 range 1..15
    ((16, 16, 16), {"m": 0}, -2),
    ((16, 16, 16), {"sigma": 1.0}, -1),
    ((16, 16, 16), {"sigma": 1.5}, -2),  # n_t = 24 is not a power of two
    ((16, 16, 16), {"window": 7}, -1),
    ((16, 16, 16), {"M": -1}, -1),
    ((1024, 16, 16), {}, -2),          # n_t = 2048 beyond the FFT kernels
])
def test_plan_validation_is_host_side(lib, N, kw, code):
    rc, h = _plan(lib, N, **kw)
    assert rc == code
    assert h.value is None
    assert lib.hpnfft_last_error()


def test_null_arguments(lib):
    assert lib.hpnfft_set_points(None, None) == -1
    assert lib.hpnfft_adjoint(None, None, None) == -1
    assert lib.hpnfft_destroy(None) == 0
    assert lib.hpnfft_workspace_bytes(None) == 0


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2001_01583_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), fn
                assert "liboracle" not in txt, fn


def test_dist_plan_validation_is_host_side(lib):
    """hpnfft_plan_dist rejects bad rank/nranks/mode/id before touching CUDA or NCCL."""
    h = ctypes.c_void_p()
    arr = (ctypes.c_int64 * 3)(16, 16, 16)
    uid = b"\0" * 128
    assert lib.hpnfft_plan_dist(ctypes.byref(h), 3, arr, 10, 6, 2.0, 0, None, 0, 0, uid, 0) == -1
    assert lib.hpnfft_plan_dist(ctypes.byref(h), 3, arr, 10, 6, 2.0, 0, None, 2, 2, uid, 0) == -1
    assert lib.hpnfft_plan_dist(ctypes.byref(h), 3, arr, 10, 6, 2.0, 0, None, 2, 0, uid, 9) == -1
    assert lib.hpnfft_plan_dist(ctypes.byref(h), 3, arr, 10, 6, 2.0, 0, None, 2, 0, None, 0) == -1
    assert h.value is None
    assert lib.hpnfft_output_shape(None, None) == -1
    edges = (ctypes.c_int64 * 3)(0, 16, 32)
    assert lib.hpnfft_set_slabs(None, edges) == -1
    assert lib.hpnfft_ewald_reciprocal(None, None, 1.0, 1.0, None) == -1
