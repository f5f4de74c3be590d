"""Oracle O3: window functions Phi and their Fourier transforms Phi_hat (CPU, fp64).

TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ may be imported by the product
path (paper_2001_01583_b200/); only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs use it.

The paper names the windows (GAUSSIAN ... KAISER_BESSEL, §4) and
states that the scaling step divides by the Fourier weight c_k of the
periodised window (§3 "Scaling"), deferring the formulas to its
Ref. [28].  Reading Q3/Q5 of DESIGN.md: we use the standard NFFT
conventions, with the window measured in grid cells u = n x:

  Kaiser-Bessel (primary):  b = pi (2 - 1/sigma)
      Phi(u)     = sinh(b sqrt(m^2 - u^2)) / (pi sqrt(m^2 - u^2)),   |u| < m
                 = 0                                                 |u| >= m  (strict truncation, Q4)
      Phi_hat(xi) = I0(m sqrt(b^2 - (2 pi xi)^2))                    |2 pi xi| <= b
  Gaussian:                 b = 2 sigma/(2 sigma - 1) * m / pi
      Phi(u)      = (pi b)^(-1/2) exp(-u^2 / b),                     |u| < m
      Phi_hat(xi) = exp(-b pi^2 xi^2)

  B-spline (NEXT #3):        Phi(u) = M_{2m}(u), the centred cardinal B-spline of order 2m
      (support exactly [-m, m]: no truncation), by the Cox-de Boor recursion
      M_1(u) = [-1/2 <= u < 1/2],  M_p(u) = ((p/2 + u) M_{p-1}(u + 1/2) + (p/2 - u) M_{p-1}(u - 1/2)) / (p - 1)
      Phi_hat(xi) = sinc(pi xi)^{2m}
  Sinc power (NEXT #3):      beta = (2 sigma - 1) / (2 m sigma)
      Phi(u)      = sinc(pi beta u)^{2m},                            |u| < m
      Phi_hat(xi) = M_{2m}(xi / beta) / beta
  (sinc(y) = sin(y)/y; both as in the NFFT library's window family, reading Q21.)

Phi_hat(xi) = int Phi_untruncated(v) e^{-2 pi i xi v} dv, so the deconvolution
factor for frequency k on an n-point grid is Phi_hat(k/n) (Q5: the closed form of
the untruncated window; the truncation error is part of the method's error).
"""
from __future__ import annotations

import numpy as np
from scipy import special

KAISER_BESSEL = 0
GAUSSIAN = 1
B_SPLINE = 2
SINC_POWER = 3


def bspline(u, p: int) -> np.ndarray:
    """Centred cardinal B-spline M_p(u) by the Cox-de Boor recursion (stable, no cancellation)."""
    u = np.asarray(u, dtype=np.float64)
    # level 1 at the p points u - (p-1)/2 + j, j = 0 .. p-1; level k keeps p - k + 1 points
    offs = np.arange(p, dtype=np.float64) - (p - 1) / 2.0
    y = u[..., None] + offs
    v = ((y >= -0.5) & (y < 0.5)).astype(np.float64)
    for k in range(2, p + 1):
        r = p - k
        yk = u[..., None] + (np.arange(r + 1, dtype=np.float64) - r / 2.0)
        v = ((k / 2.0 + yk) * v[..., 1:] + (k / 2.0 - yk) * v[..., :-1]) / (k - 1)
    return v[..., 0]


def sinc_beta(sigma: float, m: int) -> float:
    return (2.0 * sigma - 1.0) / (2.0 * m * sigma)


def _sinc(y):
    y = np.asarray(y, dtype=np.float64)
    out = np.ones_like(y)
    nz = y != 0
    out[nz] = np.sin(y[nz]) / y[nz]
    return out


def kb_b(sigma: float) -> float:
    return np.pi * (2.0 - 1.0 / sigma)


def gauss_b(sigma: float, m: int) -> float:
    return 2.0 * sigma / (2.0 * sigma - 1.0) * m / np.pi


def phi(u, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """Window Phi(u), u in grid cells, strict support |u| < m."""
    u = np.asarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    inside = np.abs(u) < m
    ui = u[inside]
    if window == KAISER_BESSEL:
        b = kb_b(sigma)
        s = np.sqrt(m * m - ui * ui)
        # sinh(b s)/(pi s); s > 0 strictly inside the support
        out[inside] = np.sinh(b * s) / (np.pi * s)
    elif window == GAUSSIAN:
        b = gauss_b(sigma, m)
        out[inside] = np.exp(-ui * ui / b) / np.sqrt(np.pi * b)
    elif window == B_SPLINE:
        out[inside] = bspline(ui, 2 * m)
    elif window == SINC_POWER:
        out[inside] = _sinc(np.pi * sinc_beta(sigma, m) * ui) ** (2 * m)
    else:
        raise ValueError("unknown window")
    return out


def phi_hat(xi, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """Fourier transform of the untruncated window at frequency xi (cycles per cell)."""
    xi = np.asarray(xi, dtype=np.float64)
    if window == KAISER_BESSEL:
        b = kb_b(sigma)
        arg = b * b - (2.0 * np.pi * xi) ** 2
        if np.any(arg < 0):
            raise ValueError("KB Phi_hat evaluated outside |2 pi xi| <= b")
        return special.i0(m * np.sqrt(arg))
    if window == GAUSSIAN:
        b = gauss_b(sigma, m)
        return np.exp(-b * np.pi ** 2 * xi * xi)
    if window == B_SPLINE:
        return _sinc(np.pi * xi) ** (2 * m)
    if window == SINC_POWER:
        beta = sinc_beta(sigma, m)
        return bspline(xi / beta, 2 * m) / beta
    raise ValueError("unknown window")


def deconv_factors(N: int, n: int, m: int, sigma: float, window: int = KAISER_BESSEL) -> np.ndarray:
    """c_k for k = -N/2 .. N/2-1 (index k + N/2): Phi_hat(k/n)."""
    k = np.arange(-N // 2, N // 2, dtype=np.float64)
    c = phi_hat(k / n, m, sigma, window)
    if np.any(~np.isfinite(c)) or np.any(np.abs(c) < 1e-300):
        raise ValueError("degenerate window weight")
    return c
