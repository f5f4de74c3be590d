"""Device-side generation of the seeded inputs (bit-identical to inputs/__init__.py)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import SEED_UNIFORM, SEED_CENTERS, cluster_centers

_lib = None


def _load():
    global _lib
    if _lib is None:
        from .build import LIB, build

        if not os.path.exists(LIB):
            build()
        lib = ctypes.CDLL(LIB)
        vp, i64, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
        lib.hpnfft_gen_uniform_points.argtypes = [vp, i64, i64, u64, vp]
        lib.hpnfft_gen_uniform_values.argtypes = [vp, i64, i64, u64, vp]
        lib.hpnfft_gen_clustered_points.argtypes = [vp, i64, i64, u64, vp, ctypes.c_int, ctypes.c_double, vp]
        _lib = lib
    return _lib


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def uniform_points(M: int, seed: int = SEED_UNIFORM, start: int = 0, device="cuda"):
    import torch

    x = torch.empty((M, 3), dtype=torch.float64, device=device)
    if M:
        assert _load().hpnfft_gen_uniform_points(ctypes.c_void_p(x.data_ptr()), M, start, seed, _stream()) == 0
    return x


def uniform_values(M: int, seed: int = SEED_UNIFORM, start: int = 0, device="cuda"):
    import torch

    f = torch.empty(M, dtype=torch.complex128, device=device)
    if M:
        assert _load().hpnfft_gen_uniform_values(ctypes.c_void_p(f.data_ptr()), M, start, seed, _stream()) == 0
    return f


def clustered_points(M: int, K: int = 16, s: float = 0.05, seed: int = SEED_UNIFORM,
                     center_seed: int = SEED_CENTERS, start: int = 0, device="cuda"):
    import torch

    c = torch.from_numpy(np.ascontiguousarray(cluster_centers(K, center_seed))).to(device)
    x = torch.empty((M, 3), dtype=torch.float64, device=device)
    if M:
        assert _load().hpnfft_gen_clustered_points(ctypes.c_void_p(x.data_ptr()), M, start, seed,
                                                   ctypes.c_void_p(c.data_ptr()), K, s, _stream()) == 0
    return x
