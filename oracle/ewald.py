"""Oracle O4: Madelung constant through the ENUF Ewald split, Eqs. (10)-(12) of
PAPER.md:290-304 (§5).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  Madelung = U^E * m / (N Z+ Z-)                                   Eq. (10)
  U^{E,R}  = 1/2 sum_n sum_{i,j}' q_i q_j erfc(alpha|r_ij + nL|)/|r_ij + nL|
                                                                    Eq. (11)
  U^{E,K}  = 1/(2 pi L) sum_{n != 0} exp(-pi^2 |n|^2/(alpha L)^2)/|n|^2 S(n) S(-n)
             - alpha/sqrt(pi) sum_i q_i^2                           Eq. (12)
  S(n)     = sum_i q_i exp(-2 pi i n.r_i / L)

Readings (Q19/Q20): erfc is the textbook complementary error function
(the printed lower limit 0 is a typo); Eq. 10 yields a negative U for an ionic
crystal, we report |U|; alpha is in units of 1/r0 and chosen so that both sums
converge at the grid's k-range and with the minimum-image real-space cutoff L/2.

S(n) is taken over n in I_N from any NDFT provider `fhat_fn(x, f, N)` that
returns Eq. (5) for x_i = r_i/L - 1/2, f_i = q_i: then S(n) = (-1)^{n0+n1+n2}
fhat(n) and S(n)S(-n) = |fhat(n)|^2 for real charges.
"""
from __future__ import annotations

import numpy as np
from scipy import special

from . import index_set, ndft_direct


def real_space_energy(r: np.ndarray, q: np.ndarray, L: float, alpha: float, block: int = 512) -> float:
    """Eq. (11) with the minimum image convention (cut-off L/2; erfc(alpha L/2) negligible)."""
    M = r.shape[0]
    tot = 0.0
    for a in range(0, M, block):
        d = r[a:a + block, None, :] - r[None, :, :]
        d -= L * np.round(d / L)
        dist = np.sqrt(np.sum(d * d, axis=-1))
        qq = q[a:a + block, None] * q[None, :]
        with np.errstate(divide="ignore", invalid="ignore"):
            term = qq * special.erfc(alpha * dist) / dist
        # the i == j, n = 0 term is omitted (the dagger in Eq. 11); pairs beyond L/2 dropped
        mask = (dist > 0) & (dist <= L / 2)
        tot += float(np.sum(term[mask]))
    return 0.5 * tot


def reciprocal_energy(fhat: np.ndarray, q: np.ndarray, L: float, alpha: float) -> float:
    """Eq. (12) given fhat(n) on I_N (shape N, index n + N/2)."""
    N = fhat.shape
    ks = index_set(N).astype(np.float64)
    n2 = np.sum(ks * ks, axis=1)
    s2 = np.abs(fhat.reshape(-1)) ** 2
    nz = n2 > 0
    e = np.exp(-np.pi ** 2 * n2[nz] / (alpha * L) ** 2) / n2[nz]
    return float(np.sum(e * s2[nz]) / (2.0 * np.pi * L) - alpha / np.sqrt(np.pi) * np.sum(q * q))


def madelung(kind: str, cells: int, N, alpha: float, fhat_fn=None) -> float:
    """Madelung constant of a crystal (Eq. 10) with S(n) from `fhat_fn` (default: O1 direct NDFT)."""
    from inputs import crystal  # seeded structure builder (no method arithmetic)

    r, q, L = crystal(kind, cells)
    x = r / L - 0.5
    f = q.astype(np.complex128)
    if fhat_fn is None:
        fhat = ndft_direct(x, f, N)
    else:
        fhat = np.asarray(fhat_fn(x, f, N)).reshape(tuple(N))
    U = real_space_energy(r, q, L, alpha) + reciprocal_energy(fhat, q, L, alpha)
    nions = r.shape[0]
    if kind == "caf2":
        m_ions, zp, zm = 3, 2.0, 1.0
    else:
        m_ions, zp, zm = 2, 1.0, 1.0
    return abs(U) * m_ions / (nions * zp * zm)
