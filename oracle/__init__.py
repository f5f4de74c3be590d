"""CPU oracle for the HP-NFFT adjoint hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product path
(paper_2001_01583_b200/) never imports, links or executes anything here, and
this package never imports the product path.

Parts:
  O1 ndft_direct        direct NDFT, Eq. (5), Kahan-summed (oracle.c)
  O2 nfft_adjoint       CUNFFT steps in the paper's order: spread -> FFT -> scale
                        (Fig. 1, Alg. 2)
  O1i ndft_inverse_direct  direct inverse NDFT, Eq. (6), Kahan-summed (oracle.c)
  O2i nfft_inverse      inverse CUNFFT in the paper's order: subdivide -> inverse FFT ->
                        interpolate (Fig. 2, Alg. 5)
  O3 windows            window/deconvolution pair (windows.py)
  O4 ewald              Madelung constant via Eqs. 10-12 (ewald.py)
  O5 rel_l2_error       Eq. (9)
Every function here is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import windows  # noqa: F401
from .windows import B_SPLINE, GAUSSIAN, KAISER_BESSEL, SINC_POWER  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, no fast-math, no FMA contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-o", _LIB_PATH, src, "-lm"]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_ndft.argtypes = [ctypes.c_int, i64p, ctypes.c_int64, dp, dp, ctypes.c_int64, i64p, dp,
                                    ctypes.c_int]
        lib.oracle_ndft.restype = ctypes.c_int
        lib.oracle_spread.argtypes = [ctypes.c_int, i64p, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int64,
                                      dp, dp, dp, ctypes.c_int]
        lib.oracle_spread.restype = ctypes.c_int
        lib.oracle_taps.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                    dp, i64p]
        lib.oracle_taps.restype = ctypes.c_int
        lib.oracle_ndft_inverse.argtypes = [ctypes.c_int, i64p, ctypes.c_int64, dp, dp, dp, ctypes.c_int]
        lib.oracle_ndft_inverse.restype = ctypes.c_int
        lib.oracle_interp.argtypes = [ctypes.c_int, i64p, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int64,
                                      dp, dp, dp, ctypes.c_int]
        lib.oracle_interp.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _check_N(N):
    N = tuple(int(v) for v in N)
    for v in N:
        if v < 2 or v % 2:
            raise ValueError("invalid bandwidth: every N_t must be even and >= 2 (PAPER.md:27)")
    return N


def index_set(N) -> np.ndarray:
    """I_N = {k : -N_t/2 <= k_t < N_t/2}, lexicographic. Shape [|I_N|, d]."""
    N = _check_N(N)
    axes = [np.arange(-n // 2, n // 2, dtype=np.int64) for n in N]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in mesh], axis=1)


def ndft_direct(x, f, N, ks=None, nthreads: int = 0) -> np.ndarray:
    """O1: fhat(k) = sum_j f_j exp(-2 pi i k.x_j) (Eq. 5).

    Returns an array of shape N (all k in I_N, index k + N/2) or [len(ks)] for
    sampled frequencies ks (integer array [K, d]).  M = 0 gives zeros.
    """
    N = _check_N(N)
    d = len(N)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
    f = np.ascontiguousarray(np.asarray(f, dtype=np.complex128).reshape(-1))
    if x.shape[0] != f.shape[0]:
        raise ValueError("shape error: x and f disagree on M")
    M = x.shape[0]
    fv = f.view(np.float64).copy() if M else np.zeros(2)
    Na = np.array(N, dtype=np.int64)
    lib = _load()
    if ks is None:
        K = int(np.prod(N))
        out = np.zeros(2 * K, dtype=np.float64)
        rc = lib.oracle_ndft(d, _ip(Na), M, _dp(x) if M else _dp(np.zeros(d)), _dp(fv), K, None, _dp(out), nthreads)
        if rc:
            raise RuntimeError("oracle_ndft failed")
        return out.view(np.complex128).reshape(N)
    ks = np.ascontiguousarray(ks, dtype=np.int64).reshape(-1, d)
    K = ks.shape[0]
    out = np.zeros(2 * max(K, 1), dtype=np.float64)
    rc = lib.oracle_ndft(d, _ip(Na), M, _dp(x) if M else _dp(np.zeros(d)), _dp(fv), K, _ip(ks), _dp(out), nthreads)
    if rc:
        raise RuntimeError("oracle_ndft failed")
    return out.view(np.complex128)[:K]


def grid_size(N, sigma: float):
    """n_t = sigma * N_t, required to be a power of two (Q6)."""
    n = []
    for v in N:
        nt = sigma * v
        if abs(nt - round(nt)) > 1e-9:
            raise ValueError("sigma*N_t must be an integer")
        nt = int(round(nt))
        if nt & (nt - 1):
            raise ValueError("n_t = sigma*N_t must be a power of two")
        n.append(nt)
    return tuple(n)


def taps_1d(n: int, m: int, sigma: float, window: int, x: float):
    """Weights and grid indices of the 2m taps of one coordinate (oracle.c convention)."""
    w = np.zeros(2 * m)
    idx = np.zeros(2 * m, dtype=np.int64)
    _load().oracle_taps(n, m, sigma, window, float(x), _dp(w), _ip(idx))
    return w, idx


def spread(x, f, n, m: int, sigma: float, window: int = KAISER_BESSEL, nthreads: int = 0) -> np.ndarray:
    """O2 step 1 (Spreading): g(l) = sum_j f_j prod_t Phi(n_t x_jt - l_t), l mod n,
    for d = len(n) in 1..3 (threads own grid planes; bit-identical for any thread count)."""
    n = tuple(int(v) for v in n)
    d = len(n)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
    f = np.ascontiguousarray(np.asarray(f, dtype=np.complex128).reshape(-1))
    g = np.zeros(n + (2,), dtype=np.float64)
    M = x.shape[0]
    if M:
        fv = f.view(np.float64).copy()
        na = np.array(n, dtype=np.int64)
        rc = _load().oracle_spread(d, _ip(na), m, sigma, window, M, _dp(x), _dp(fv), _dp(g), int(nthreads))
        if rc:
            raise RuntimeError("oracle_spread failed")
    return g.view(np.complex128).reshape(n)


def spread_naive_gather(x, f, n, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """Spreading written per lattice node l as a gather over all points:
    g(l) = sum_j f_j prod_t Phi(periodic distance), used to pin oracle_spread on tiny grids."""
    n = tuple(int(v) for v in n)
    x = np.asarray(x, dtype=np.float64).reshape(-1, 3)
    f = np.asarray(f, dtype=np.complex128).reshape(-1)
    g = np.zeros(n, dtype=np.complex128)
    for j in range(x.shape[0]):
        w = []
        for t in range(3):
            u = n[t] * x[j, t]
            l = np.arange(n[t])
            # all periodic images l + r n_t; Phi vanishes beyond m so a few images suffice
            tot = np.zeros(n[t])
            for r in range(-3, 4):
                tot += windows.phi(u - (l + r * n[t]), m, sigma, window)
            w.append(tot)
        g += f[j] * w[0][:, None, None] * w[1][None, :, None] * w[2][None, None, :]
    return g


def _workers() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def fft_grid(g: np.ndarray) -> np.ndarray:
    """O2 step 2 (FFT): ghat(k) = sum_l g(l) exp(-2 pi i k.l/n), unnormalised
    (scipy.fft on all host cores)."""
    import scipy.fft

    return scipy.fft.fftn(g, workers=_workers())


def deconvolve_crop(ghat: np.ndarray, N, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """O2 step 3 (Scaling): fhat(k) = ghat(k mod n) / prod_t c_k, k in I_N."""
    N = _check_N(N)
    d = len(N)
    n = ghat.shape
    out = ghat
    for t in range(d):
        k = np.arange(-N[t] // 2, N[t] // 2)
        out = np.take(out, k % n[t], axis=t)
    for t in range(d):
        c = windows.deconv_factors(N[t], n[t], m, sigma, window)
        shape = [1] * d
        shape[t] = N[t]
        out = out / c.reshape(shape)
    return out


def nfft_adjoint(x, f, N, m: int = 6, sigma: float = 2.0, window: int = KAISER_BESSEL) -> np.ndarray:
    """O2: the CPU NFFT of Eq. (5) in Alg. 2's order: spread -> FFT -> scale/crop (d = len(N) in
    1..3)."""
    N = _check_N(N)
    if not 1 <= len(N) <= 3:
        raise ValueError("oracle NFFT: d must be 1, 2 or 3")
    n = grid_size(N, sigma)
    g = spread(x, f, n, m, sigma, window)
    return deconvolve_crop(fft_grid(g), N, m, sigma, window)


def ndft_inverse_direct(x, fhat, N, nthreads: int = 0) -> np.ndarray:
    """O1i: f(x_j) = sum_{k in I_N} fhat(k) exp(+2 pi i k.x_j) (Eq. 6).

    fhat: array of shape N (index k + N/2).  Returns [M] complex.
    """
    N = _check_N(N)
    d = len(N)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
    fh = np.ascontiguousarray(np.asarray(fhat, dtype=np.complex128).reshape(N))
    M = x.shape[0]
    out = np.zeros(2 * max(M, 1), dtype=np.float64)
    if M == 0:
        return np.zeros(0, dtype=np.complex128)
    fv = fh.reshape(-1).view(np.float64).copy()
    rc = _load().oracle_ndft_inverse(d, _ip(np.array(N, dtype=np.int64)), M, _dp(x), _dp(fv), _dp(out), nthreads)
    if rc:
        raise RuntimeError("oracle_ndft_inverse failed")
    return out.view(np.complex128)[:M].copy()


def subdivide(fhat, N, n, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """O2i step 1 (Subdividing): ghat(k mod n) = fhat(k) / prod_t c_k for k in I_N,
    0 for the other k in I_n (the transpose of deconvolve_crop)."""
    N = _check_N(N)
    d = len(N)
    fh = np.asarray(fhat, dtype=np.complex128).reshape(N)
    for t in range(d):
        c = windows.deconv_factors(N[t], n[t], m, sigma, window)
        shape = [1] * d
        shape[t] = N[t]
        fh = fh / c.reshape(shape)
    ghat = np.zeros(tuple(n), dtype=np.complex128)
    idx = np.ix_(*[np.arange(-N[t] // 2, N[t] // 2) % n[t] for t in range(d)])
    ghat[idx] = fh
    return ghat


def ifft_grid(ghat: np.ndarray) -> np.ndarray:
    """O2i step 2 (Inverse FFT): g(l) = sum_k ghat(k) exp(+2 pi i k.l/n),
    unnormalised (numpy's ifftn divides by prod n_t)."""
    import scipy.fft

    return scipy.fft.ifftn(ghat, workers=_workers()) * float(np.prod(ghat.shape))


def interpolate(g: np.ndarray, x, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """O2i step 3 (Interpolating): f_j = sum_l g(l) prod_t Phi(n_t x_jt - l_t)."""
    n = g.shape
    d = len(n)
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
    M = x.shape[0]
    f = np.zeros(2 * max(M, 1), dtype=np.float64)
    if M:
        gv = np.ascontiguousarray(g, dtype=np.complex128).reshape(-1).view(np.float64)
        rc = _load().oracle_interp(d, _ip(np.array(n, dtype=np.int64)), m, sigma, window, M, _dp(x), _dp(gv), _dp(f),
                                   0)
        if rc:
            raise RuntimeError("oracle_interp failed")
    return f.view(np.complex128)[:M].copy()


def nfft_inverse(x, fhat, N, m: int = 6, sigma: float = 2.0, window: int = KAISER_BESSEL) -> np.ndarray:
    """O2i: the CPU inverse CUNFFT of Eq. (6) in Alg. 5's order: subdivide -> inverse FFT ->
    interpolate."""
    N = _check_N(N)
    n = grid_size(N, sigma)
    return interpolate(ifft_grid(subdivide(fhat, N, n, m, sigma, window)), x, m, sigma, window)


def rel_l2_error(a, b) -> float:
    """O5: E = ||a - b||_2 / ||b||_2 over all entries (Eq. 9; reading Q11)."""
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    nb = np.sqrt(np.sum(np.abs(b) ** 2))
    if nb == 0:
        raise ValueError("undefined reference: ||s|| = 0")
    return float(np.sqrt(np.sum(np.abs(a - b) ** 2)) / nb)
