"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no window, spread, FFT or
deconvolution).  It only draws random numbers and builds the point sets the
paper's workloads are shaped like:

* uniform points x_j ~ U[-0.5, 0.5)^3, values f_j ~ U[-0.5,0.5) + i U[-0.5,0.5)
  ("randomly scattered in the spatial domain", §1);
* Gaussian-clustered points (Irwin-Hall normal around K centres, periodically
  wrapped) for the load-balance cases of SURVEY.md §8(d);
* equispaced points x_j = N^{-1} ⊙ j (§1 Eq. 3);
* the fluorite CaF2 crystal of PAPER.md:306 (§5, Fig. 14).

The generator is counter based (splitmix64 of (seed, stream, j)), so element j
of any stream can be produced independently on the host (this file, numpy) and
on the device (inputs/gen.cu, a separate library that is NOT part of the
product path).  Both produce bit-identical doubles: the only floating-point
operations are an exact int->double conversion, one exact multiply by 2^-53
and a fixed sequence of additions.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)
STREAM_MUL = np.uint64(0xD1B54A32D192ED03)

# stream ids (kept identical in inputs/gen.cu)
STREAM_X = 0          # x_t uses STREAM_X + t, t = 0,1,2
STREAM_F_RE = 3
STREAM_F_IM = 4
STREAM_CENTER = 8     # cluster centres: STREAM_CENTER + t
STREAM_IRWIN = 16     # Irwin-Hall draws: STREAM_IRWIN + 12*t + r, r = 0..11

SEED_UNIFORM = 2001
SEED_CENTERS = 2002


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return np.uint64(seed) * GOLDEN ^ np.uint64(stream) * STREAM_MUL


def u64(seed: int, stream: int, j: np.ndarray) -> np.ndarray:
    """splitmix64 output for counters j (uint64 array) of (seed, stream)."""
    j = np.asarray(j, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _key(seed, stream) + (j + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, j: np.ndarray) -> np.ndarray:
    """Double in [0,1) from the top 53 bits (exact conversion and scaling)."""
    return (u64(seed, stream, j) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def wrap(x: np.ndarray) -> np.ndarray:
    """Periodic wrap into [-0.5, 0.5): x - floor(x + 0.5)."""
    return x - np.floor(x + 0.5)


def uniform_points(M: int, seed: int = SEED_UNIFORM, start: int = 0, d: int = 3) -> np.ndarray:
    j = np.arange(start, start + M, dtype=np.uint64)
    x = np.empty((M, d), dtype=np.float64)
    for t in range(d):
        x[:, t] = uniform01(seed, STREAM_X + t, j) - 0.5
    return x


def uniform_values(M: int, seed: int = SEED_UNIFORM, start: int = 0) -> np.ndarray:
    j = np.arange(start, start + M, dtype=np.uint64)
    re = uniform01(seed, STREAM_F_RE, j) - 0.5
    im = uniform01(seed, STREAM_F_IM, j) - 0.5
    return re + 1j * im


def cluster_centers(K: int = 16, seed: int = SEED_CENTERS, d: int = 3) -> np.ndarray:
    j = np.arange(K, dtype=np.uint64)
    c = np.empty((K, d), dtype=np.float64)
    for t in range(d):
        c[:, t] = uniform01(seed, STREAM_CENTER + t, j) - 0.5
    return c


def clustered_points(M: int, K: int = 16, s: float = 0.05, seed: int = SEED_UNIFORM,
                     center_seed: int = SEED_CENTERS, start: int = 0, d: int = 3) -> np.ndarray:
    """x = wrap(c_{j mod K} + s * z), z = sum_{r<12} U_r - 6 (Irwin-Hall, additions only)."""
    j = np.arange(start, start + M, dtype=np.uint64)
    c = cluster_centers(K, center_seed, d)
    x = np.empty((M, d), dtype=np.float64)
    cj = (j % np.uint64(K)).astype(np.int64)
    for t in range(d):
        z = np.zeros(M, dtype=np.float64)
        for r in range(12):
            z = z + uniform01(seed, STREAM_IRWIN + 12 * t + r, j)
        z = z - 6.0
        x[:, t] = wrap(c[cj, t] + s * z)
    return x


def equispaced_points(N) -> np.ndarray:
    """x_j = N^{-1} ⊙ j for j in I_N, lexicographic (§1)."""
    N = tuple(int(v) for v in N)
    axes = [np.arange(-n // 2, n // 2, dtype=np.float64) / n for n in N]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in mesh], axis=1)


# ---------------------------------------------------------------- crystals --
# Fluorite (CaF2), PAPER.md:306 (§5, Fig. 14): 4 Ca2+ (fcc) + 8 F- (the
# (1/4,3/4)^3 sublattice) per cubic cell of side l; unit length r0 = sqrt(3) l/4
# so l = 4/sqrt(3) in units of r0.
CAF2_CATIONS = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]])
CAF2_ANIONS = np.array([[a, b, c] for a in (0.25, 0.75) for b in (0.25, 0.75) for c in (0.25, 0.75)])
# Rock salt (NaCl): shortest cation-anion distance r0 = l/2.
NACL_CATIONS = np.array([[0, 0, 0], [0.5, 0.5, 0], [0.5, 0, 0.5], [0, 0.5, 0.5]])
NACL_ANIONS = NACL_CATIONS + np.array([0.5, 0.0, 0.0])


def crystal(kind: str, cells: int):
    """Return (positions r_i in units of r0, in [0, L)^3; charges q_i; side L)."""
    if kind == "caf2":
        cat, an, qc, qa, l = CAF2_CATIONS, CAF2_ANIONS, 2.0, -1.0, 4.0 / np.sqrt(3.0)
    elif kind == "nacl":
        cat, an, qc, qa, l = NACL_CATIONS, NACL_ANIONS, 1.0, -1.0, 2.0
    else:
        raise ValueError(kind)
    base = np.concatenate([cat, an % 1.0])
    q = np.concatenate([np.full(len(cat), qc), np.full(len(an), qa)])
    g = np.arange(cells, dtype=np.float64)
    shifts = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    frac = (shifts[:, None, :] + base[None, :, :]).reshape(-1, 3)   # in cell units
    L = cells * l
    r = frac * l
    qq = np.tile(q, len(shifts))
    return r, qq, L


def crystal_nfft_inputs(kind: str, cells: int):
    """NFFT inputs for the structure factor S(n) of Eq. 12: x_i = r_i/L - 1/2, f_i = q_i."""
    r, q, L = crystal(kind, cells)
    x = r / L - 0.5
    return x, q.astype(np.complex128), L
