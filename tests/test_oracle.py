"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test names the oracle part it pins and the passage
it follows.  None of them compares the oracle with itself: expected values come
from mpmath brute force, numpy.fft on the equispaced reduction (Eq. 3), closed
forms, exact symmetries, quadrature, the paper's Madelung constant and textbook
values.
"""
import json
import os

import mpmath
import numpy as np
import pytest
from scipy import integrate

import inputs
import oracle
from oracle import ewald, windows

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
N16 = (16, 16, 16)


# ------------------------------------------------------------------ O1 --
def test_O1_mpmath_brute_force():
    """O1 vs 50-digit brute force of Eq. 5, M=8, N=4^3."""
    x = inputs.uniform_points(8, seed=11)
    f = inputs.uniform_values(8, seed=11)
    got = oracle.ndft_direct(x, f, (4, 4, 4))
    mpmath.mp.dps = 50
    ks = oracle.index_set((4, 4, 4))
    ref = np.zeros(len(ks), dtype=np.complex128)
    for q, k in enumerate(ks):
        s = mpmath.mpc(0)
        for j in range(8):
            arg = sum(int(k[t]) * mpmath.mpf(float(x[j, t])) for t in range(3))
            s += mpmath.mpc(float(f[j].real), float(f[j].imag)) * mpmath.expjpi(-2 * arg)
        ref[q] = complex(s)
    assert oracle.rel_l2_error(got.reshape(-1), ref) < 1e-15


def test_O1_zero_frequency_and_origin():
    """fhat(0) = sum_j f_j; a single point at the origin gives fhat = f_0 for all k."""
    x = inputs.uniform_points(300, seed=5)
    f = inputs.uniform_values(300, seed=5)
    fh = oracle.ndft_direct(x, f, (8, 8, 8))
    assert abs(fh[4, 4, 4] - np.sum(f)) < 1e-13
    one = oracle.ndft_direct(np.zeros((1, 3)), np.array([0.7 - 0.2j]), (6, 4, 8))
    assert np.max(np.abs(one - (0.7 - 0.2j))) == 0.0
    empty = oracle.ndft_direct(np.zeros((0, 3)), np.zeros(0, dtype=complex), (4, 4, 4))
    assert np.all(empty == 0)


def test_O1_equispaced_reduces_to_dft():
    """x_j = N^{-1} ⊙ j, M = |I_N|: Eq. 5 is Eq. 3, i.e. numpy.fft.fftn up to the
    index shift j -> j + N/2, which multiplies fhat(k) by (-1)^(k0+k1+k2)."""
    N = (8, 6, 10)
    x = inputs.equispaced_points(N)
    f = inputs.uniform_values(x.shape[0], seed=3)
    got = oracle.ndft_direct(x, f, N)
    F = f.reshape(N)
    X = np.fft.fftn(F)
    ks = oracle.index_set(N)
    ref = np.array([(-1.0) ** int(np.sum(k)) * X[tuple(k % np.array(N))] for k in ks]).reshape(N)
    assert oracle.rel_l2_error(got, ref) < 1e-14


def test_O1_linearity_translation_conjugate():
    x = inputs.uniform_points(200, seed=21)
    f = inputs.uniform_values(200, seed=21)
    g = inputs.uniform_values(200, seed=22)
    N = (8, 8, 8)
    a, b = 0.3 - 1.1j, -2.0 + 0.5j
    lhs = oracle.ndft_direct(x, a * f + b * g, N)
    rhs = a * oracle.ndft_direct(x, f, N) + b * oracle.ndft_direct(x, g, N)
    assert oracle.rel_l2_error(lhs, rhs) < 1e-13
    # translation x -> x + delta multiplies by exp(-2 pi i k.delta)
    delta = np.array([0.0123, -0.2, 0.31])
    sh = oracle.ndft_direct(x + delta, f, N)
    k = oracle.index_set(N).astype(float)
    ph = np.exp(-2j * np.pi * (k @ delta)).reshape(N)
    assert oracle.rel_l2_error(sh, ph * oracle.ndft_direct(x, f, N)) < 1e-13
    # real values: fhat(-k) = conj fhat(k) for k, -k in I_N
    fr = oracle.ndft_direct(x, f.real.astype(complex), N)
    inner = fr[1:, 1:, 1:]
    assert np.max(np.abs(inner - np.conj(inner[::-1, ::-1, ::-1]))) < 1e-12


def test_O1_sampled_matches_full():
    x = inputs.uniform_points(100, seed=7)
    f = inputs.uniform_values(100, seed=7)
    N = (8, 8, 8)
    full = oracle.ndft_direct(x, f, N)
    ks = np.array([[-4, 0, 3], [0, 0, 0], [3, -1, -4]])
    s = oracle.ndft_direct(x, f, N, ks=ks)
    for q, k in enumerate(ks):
        assert s[q] == full[tuple(k + 4)]


def test_O1_rejects_odd_bandwidth():
    with pytest.raises(ValueError):
        oracle.ndft_direct(np.zeros((1, 3)), np.ones(1), (3, 4, 4))


# ------------------------------------------------------------------ O3 --
@pytest.mark.parametrize("m", [2, 4, 6, 8])
def test_O3_kaiser_bessel_fourier_pair_quadrature(m):
    """Phi_hat(xi) = I0(m sqrt(b^2 - (2 pi xi)^2)) vs quadrature of the truncated Phi over [-m, m]
    (reading Q5).  Agreement to the truncation level (survey: 7.7e-13 at m=6)."""
    sigma = 2.0
    for xi in [0.0, 0.05, 0.125, 0.2, 0.25]:
        val, _ = integrate.quad(lambda u: windows.phi(np.array([u]), m, sigma)[0] * np.cos(2 * np.pi * xi * u),
                                -m, m, epsabs=0, epsrel=2e-14, limit=200)
        ref = windows.phi_hat(xi, m, sigma)
        tol = {2: 2e-3, 4: 2e-7, 6: 3e-11, 8: 1e-13}[m]
        assert abs(val - ref) / ref < tol


def test_O3_gaussian_fourier_pair_quadrature():
    sigma, m = 2.0, 6
    b = windows.gauss_b(sigma, m)
    for xi in [0.0, 0.1, 0.25]:
        val, _ = integrate.quad(lambda u: np.exp(-u * u / b) / np.sqrt(np.pi * b) * np.cos(2 * np.pi * xi * u),
                                -np.inf, np.inf, epsabs=0, epsrel=2e-14)
        assert abs(val - windows.phi_hat(xi, m, sigma, windows.GAUSSIAN)) < 1e-13


def test_O3_window_shape():
    m, sigma = 6, 2.0
    u = np.linspace(-5.9, 5.9, 101)
    assert np.allclose(windows.phi(u, m, sigma), windows.phi(-u, m, sigma), rtol=1e-15, atol=0)
    assert np.all(windows.phi(np.array([6.0, -6.0, 7.5]), m, sigma) == 0)
    b = windows.kb_b(sigma)
    assert windows.phi(np.array([0.0]), m, sigma)[0] == pytest.approx(np.sinh(b * m) / (np.pi * m), rel=1e-15)
    c = windows.deconv_factors(16, 32, m, sigma)
    assert np.all(c > 0) and np.allclose(c[1:], c[1:][::-1], rtol=1e-15)


def test_O3_taps_strict_truncation():
    """2m taps l = floor(u)-m+1 .. floor(u)+m; on a node the last tap (|u-l| = m) is zero."""
    w, idx = oracle.taps_1d(32, 6, 2.0, 0, 0.0)
    assert list(idx) == [(l % 32) for l in range(-5, 7)]
    assert w[-1] == 0.0 and w[0] > 0
    w2, idx2 = oracle.taps_1d(32, 6, 2.0, 0, 0.49)   # u = 15.68: wraps across the boundary
    assert list(idx2) == [(l % 32) for l in range(10, 22)]
    assert np.all(w2 > 0)
    ref = windows.phi(15.68 - np.arange(10, 22), 6, 2.0)
    assert np.allclose(w2, ref, rtol=1e-13, atol=0)


def test_O3_bspline_closed_forms_and_partition_of_unity():
    """NEXT #3 B-spline window M_{2m} (Cox-de Boor): textbook values of M_2 (hat) and M_4 (cubic:
    M_4(0) = 2/3, M_4(1) = 1/6, M_4(1/2) = 23/48), symmetry, unit integral, and the partition of
    unity sum_l M_p(u - l) = 1; the C oracle's taps (a separate implementation) agree."""
    u = np.linspace(-1, 1, 41)
    assert np.allclose(windows.bspline(u, 2), 1 - np.abs(u), atol=1e-15, rtol=0)
    assert windows.bspline(np.array([0.0, 1.0, -1.0, 0.5]), 4) == pytest.approx([2 / 3, 1 / 6, 1 / 6, 23 / 48], abs=1e-15)
    for p in (4, 12, 16):
        uu = np.random.default_rng(p).uniform(-3, 3, 25)
        tot = sum(windows.bspline(uu - l, p) for l in range(-p, p + 1))
        assert np.allclose(tot, 1.0, atol=1e-14, rtol=0)
        assert np.allclose(windows.bspline(uu, p), windows.bspline(-uu, p), atol=1e-16, rtol=1e-14)
        val, _ = integrate.quad(lambda v: windows.bspline(np.array([v]), p)[0], -p / 2, p / 2, points=list(range(-p // 2, p // 2 + 1)),
                                epsabs=0, epsrel=1e-13, limit=200)
        assert val == pytest.approx(1.0, abs=1e-13)
    w, idx = oracle.taps_1d(32, 6, 2.0, windows.B_SPLINE, 0.123)
    u0 = 32 * 0.123
    assert np.allclose(w, windows.phi(u0 - np.arange(int(np.floor(u0)) - 5, int(np.floor(u0)) + 7), 6, 2.0,
                                      windows.B_SPLINE), rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("m", [2, 3, 6])
def test_O3_bspline_fourier_pair_quadrature(m):
    """Phi_hat(xi) = sinc(pi xi)^{2m} vs quadrature of M_{2m} (no truncation: support [-m, m])."""
    for xi in [0.0, 0.07, 0.125, 0.25]:
        val, _ = integrate.quad(lambda v: windows.phi(np.array([v]), m, 2.0, windows.B_SPLINE)[0] * np.cos(2 * np.pi * xi * v),
                                -m, m, points=list(range(-m, m + 1)), epsabs=1e-15, epsrel=1e-13, limit=400)
        ref = windows.phi_hat(xi, m, 2.0, windows.B_SPLINE)
        assert abs(val - ref) <= 1e-13 * max(1.0, ref)


@pytest.mark.parametrize("m", [2, 3])
def test_O3_sinc_power_fourier_pair_quadrature(m):
    """Phi_hat(xi) = M_{2m}(xi / beta) / beta, beta = (2 sigma - 1)/(2 m sigma), vs quadrature of the
    untruncated sinc^{2m}(pi beta u) (the transform of sinc is a box: a 2m-fold box convolution)."""
    sigma = 2.0
    beta = windows.sinc_beta(sigma, m)
    f = lambda v: (np.sinc(beta * v)) ** (2 * m)   # np.sinc(y) = sin(pi y)/(pi y)
    for xi in [0.0, 0.05, 0.1, 0.2]:
        L = 4000.0
        val, _ = integrate.quad(f, -L, L, weight="cos", wvar=2 * np.pi * xi, limit=4000) if xi else \
            integrate.quad(f, -L, L, limit=4000, epsabs=0, epsrel=1e-13)
        ref = windows.phi_hat(xi, m, sigma, windows.SINC_POWER)
        assert abs(val - ref) <= 2e-7 * ref + 1e-12


@pytest.mark.parametrize("m", [2, 4, 6])
def test_O3_sinc_power_taps_poisson_sum(m):
    """Value pin of the sinc-power window's TAPS (the C oracle's oracle_taps): the transform of
    sinc^{2m}(pi beta u) is supported in |xi| <= m beta = (2 sigma - 1)/(2 sigma) < 1, so by Poisson
    summation sum_{l in Z} Phi(u - l) = Phi_hat(0) = M_2m(0)/beta exactly, for every u.  The 2m taps
    are the terms with |u - l| < m; the rest (the truncated tail) is summed here with numpy's sinc
    over 2e5 periods.  A wrong exponent, beta, tap offset or truncation breaks the identity."""
    sigma = 2.0
    beta = windows.sinc_beta(sigma, m)
    ref = windows.bspline(np.array([0.0]), 2 * m)[0] / beta
    n = 64
    ls = np.arange(-200000, 200001, dtype=np.float64)
    for x in np.random.default_rng(m).uniform(-0.5, 0.5, 5):
        w, _ = oracle.taps_1d(n, m, sigma, windows.SINC_POWER, float(x))
        d = n * float(x) - ls
        far = np.abs(d) >= m
        tail = np.sum(np.sinc(beta * d[far]) ** (2 * m))
        assert abs(w.sum() + tail - ref) <= 1e-13 * ref, (m, x, w.sum() + tail, ref)
    assert windows.phi_hat(0.0, m, sigma, windows.SINC_POWER) == pytest.approx(ref, rel=1e-14)


def test_O2_windows_accuracy_fig12_shape():
    """Fig. 12's shape (values unpinned): on the §4 setup (M = 4096, N = 16^3,
    sigma = 2) E2 of the CPU NFFT against the direct NDFT falls with m for all four windows, and
    Kaiser-Bessel is the most accurate at every m >= 3."""
    setup = json.load(open(os.path.join(GOLDEN, "paper_section4_setup.json")))
    M, N, sigma = setup["M"], tuple(setup["N"]), setup["sigma"]
    x, f = inputs.uniform_points(M), inputs.uniform_values(M)
    s = oracle.ndft_direct(x, f, N)
    E = {}
    for win in (windows.KAISER_BESSEL, windows.GAUSSIAN, windows.B_SPLINE, windows.SINC_POWER):
        E[win] = [oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N, m=m, sigma=sigma, window=win), s) for m in range(2, 7)]
        assert all(a > b for a, b in zip(E[win][:-1], E[win][1:])), (win, E[win])
    for i in range(1, 5):
        assert E[windows.KAISER_BESSEL][i] < min(E[w][i] for w in (windows.GAUSSIAN, windows.B_SPLINE, windows.SINC_POWER))
    # B-spline: the classical (2 sigma - 1)^(-2m) decay
    assert E[windows.B_SPLINE][4] < 4 * (2 * sigma - 1) ** (-12)


# ------------------------------------------------------------------ O2 --
def test_O2_spread_equals_lattice_gather():
    """oracle_spread (point-centric scatter) == per-lattice gather."""
    x = inputs.uniform_points(20, seed=31)
    x[0] = [0.5, -0.5, 0.0]        # boundary and on-node coordinates
    f = inputs.uniform_values(20, seed=31)
    n = (16, 8, 16)
    for win in (windows.KAISER_BESSEL, windows.GAUSSIAN, windows.B_SPLINE, windows.SINC_POWER):
        a = oracle.spread(x, f, n, 3, 2.0, win)
        b = oracle.spread_naive_gather(x, f, n, 3, 2.0, win)
        assert oracle.rel_l2_error(a, b) < 1e-13


def test_O2_fft_convention_is_eq3():
    """The FFT stage computes ghat(k) = sum_l g(l) exp(-2 pi i k.l/n), unnormalised (Eq. 3 on I_n)."""
    rng = np.random.default_rng(0)
    g = rng.standard_normal((4, 6, 8)) + 1j * rng.standard_normal((4, 6, 8))
    got = oracle.fft_grid(g)
    l = np.stack(np.meshgrid(*[np.arange(s) for s in g.shape], indexing="ij"), -1).reshape(-1, 3)
    ref = np.zeros(g.size, dtype=complex)
    for q, k in enumerate(l):
        ph = np.exp(-2j * np.pi * np.sum(k * l / np.array(g.shape), axis=1))
        ref[q] = np.sum(g.reshape(-1) * ph)
    assert oracle.rel_l2_error(got.reshape(-1), ref) < 1e-14


def test_O2_accuracy_decay_paper_section4():
    """§4 setup: E2 of O2 against O1 decays geometrically in m, like the KB bound
    4 pi (sqrt m + m)(1-1/sigma)^(1/4) exp(-2 pi m sqrt(1-1/sigma)), and meets the
    north_star bar 1e-9 at m=6."""
    setup = json.load(open(os.path.join(GOLDEN, "paper_section4_setup.json")))
    M, N = setup["M"], tuple(setup["N"])
    x = inputs.uniform_points(M)
    f = inputs.uniform_values(M)
    s = oracle.ndft_direct(x, f, N)
    errs = []
    sigma = setup["sigma"]
    for m in range(1, 8):
        e = oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N, m=m, sigma=sigma), s)
        bound = 4 * np.pi * (np.sqrt(m) + m) * (1 - 1 / sigma) ** 0.25 * np.exp(-2 * np.pi * m * np.sqrt(1 - 1 / sigma))
        assert e < bound and e > bound / 1e3
        errs.append(e)
    ratios = np.array(errs[:-1]) / np.array(errs[1:])
    assert np.all(ratios > setup["kb_e2_decay_per_m_min"])
    assert errs[5] < setup["north_star_e2_bar_m6"]


def test_O2_gaussian_cannot_meet_bar_at_m6():
    x = inputs.uniform_points(1000)
    f = inputs.uniform_values(1000)
    s = oracle.ndft_direct(x, f, N16)
    e = oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N16, m=6, window=windows.GAUSSIAN), s)
    assert 1e-7 < e < 1e-5


def test_O2_grid_shift_covariance():
    """x -> x + s/n (integer s) shifts the grid exactly: fhat -> fhat exp(-2 pi i k.s/n)."""
    x = inputs.uniform_points(500, seed=41)
    f = inputs.uniform_values(500, seed=41)
    N = N16
    s = np.array([3, -7, 12])
    a = oracle.nfft_adjoint(x, f, N)
    b = oracle.nfft_adjoint(x + s / 32.0, f, N)
    k = oracle.index_set(N).astype(float)
    ph = np.exp(-2j * np.pi * (k @ (s / 32.0))).reshape(N)
    assert oracle.rel_l2_error(b, ph * a) < 1e-14


def test_O2_partition_invariance_eq8():
    """Eq. 8: the NFFT of a partition sums to the NFFT of the whole set."""
    x = inputs.uniform_points(900, seed=51)
    f = inputs.uniform_values(900, seed=51)
    whole = oracle.nfft_adjoint(x, f, N16)
    slab = np.floor((x[:, 0] + 0.5) * 4).astype(int)   # 4 equal-size x-slabs
    parts = sum(oracle.nfft_adjoint(x[slab == r], f[slab == r], N16) for r in range(4))
    assert oracle.rel_l2_error(parts, whole) < 1e-14


def test_O2_real_values_conjugate_symmetry():
    x = inputs.uniform_points(300, seed=61)
    f = inputs.uniform_values(300, seed=61).real.astype(complex)
    a = oracle.nfft_adjoint(x, f, N16)
    inner = a[1:, 1:, 1:]
    assert np.max(np.abs(inner - np.conj(inner[::-1, ::-1, ::-1]))) < 1e-12 * np.max(np.abs(a))


def test_O2_on_node_points_and_boundary():
    """Equispaced on-node inputs (t = 0, strict truncation) still meet the bar; x = 0.5 == x = -0.5."""
    N = (8, 8, 8)
    x = inputs.equispaced_points(N)
    f = inputs.uniform_values(x.shape[0], seed=71)
    e = oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N), oracle.ndft_direct(x, f, N))
    assert e < 1e-9
    xb = np.array([[0.5, 0.1, -0.2]])
    xa = np.array([[-0.5, 0.1, -0.2]])
    one = np.array([1.0 + 0j])
    assert np.array_equal(oracle.nfft_adjoint(xb, one, N), oracle.nfft_adjoint(xa, one, N))


# ------------------------------------------------------------------ O4 --
def test_O4_madelung_caf2_paper_value_via_O1():
    """Fluorite Madelung constant 2.5194 with S(n) from the direct NDFT (O1)."""
    gold = json.load(open(os.path.join(GOLDEN, "madelung.json")))["caf2"]
    v = ewald.madelung("caf2", 8, (64, 64, 64), 0.85)
    assert abs(v - gold["value"]) < gold["tolerance"]


def test_O4_madelung_alpha_invariance_via_O2():
    """alpha does not affect U^E; O2 S(n) at alpha in [0.7, 1.0]."""
    gold = json.load(open(os.path.join(GOLDEN, "madelung.json")))["caf2"]
    fn = lambda x, f, N: oracle.nfft_adjoint(x, f, N, m=6)
    vals = [ewald.madelung("caf2", 8, (64, 64, 64), a, fhat_fn=fn) for a in (0.7, 1.0)]
    assert abs(vals[0] - vals[1]) < 1e-9
    assert abs(vals[0] - gold["value"]) < gold["tolerance"]


def test_O4_madelung_nacl_textbook():
    gold = json.load(open(os.path.join(GOLDEN, "madelung.json")))["nacl"]
    fn = lambda x, f, N: oracle.nfft_adjoint(x, f, N, m=6)
    v = ewald.madelung("nacl", 4, (32, 32, 32), 1.0, fhat_fn=fn)
    assert abs(v - gold["value"]) < gold["tolerance"]


def test_O4_crystal_sizes():
    """12 * 32^3 = 393,216 ions and L = 73.9 r0 for 32^3 fluorite cells."""
    r, q, L = inputs.crystal("caf2", 32)
    assert r.shape[0] == 393216 and abs(L - 73.9) < 0.01
    assert abs(np.sum(q)) == 0
    # shortest Ca-F distance is r0 = 1
    r1, q1, L1 = inputs.crystal("caf2", 1)
    d = r1[q1 > 0][:, None, :] - r1[q1 < 0][None, :, :]
    assert np.min(np.sqrt(np.sum(d * d, -1))) == pytest.approx(1.0, rel=1e-15)


# ------------------------------------------------------------------ O5 --
def test_O5_rel_l2_error():
    assert oracle.rel_l2_error([1, 2, 3], [1, 2, 3]) == 0.0
    assert oracle.rel_l2_error([1, 1], [1, 0]) == 1.0
    with pytest.raises(ValueError):
        oracle.rel_l2_error([1.0], [0.0])
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal(100), rng.standard_normal(100)
    ref = np.sqrt(sum((ai - bi) ** 2 for ai, bi in zip(a, b)) / sum(bi * bi for bi in b))
    assert abs(oracle.rel_l2_error(a, b) - ref) < 1e-15


# --------------------------------------------------------------- inputs --
def test_inputs_generator_properties():
    x = inputs.uniform_points(100000)
    assert x.min() >= -0.5 and x.max() < 0.5
    assert abs(x.mean()) < 5e-3 and abs(x.var() - 1 / 12) < 2e-3
    # counter-based: a window of the stream equals the slice of the full stream
    assert np.array_equal(inputs.uniform_points(10, start=500), x[500:510])
    c = inputs.clustered_points(50000, s=0.05)
    assert c.min() >= -0.5 and c.max() < 0.5
    assert np.array_equal(inputs.clustered_points(7, start=100), c[100:107])


# ------------------------------------------------------- O1i / O2i (Eq. 6) --
def test_O1i_mpmath_brute_force():
    """O1i vs 50-digit brute force of Eq. 6, M = 5, N = 4^3."""
    x = inputs.uniform_points(5, seed=12)
    rng = np.random.default_rng(12)
    fh = rng.standard_normal((4, 4, 4)) + 1j * rng.standard_normal((4, 4, 4))
    got = oracle.ndft_inverse_direct(x, fh, (4, 4, 4))
    mpmath.mp.dps = 50
    ks = oracle.index_set((4, 4, 4))
    ref = np.zeros(5, dtype=np.complex128)
    for j in range(5):
        s = mpmath.mpc(0)
        for q, k in enumerate(ks):
            arg = sum(int(k[t]) * mpmath.mpf(float(x[j, t])) for t in range(3))
            v = fh.reshape(-1)[q]
            s += mpmath.mpc(float(v.real), float(v.imag)) * mpmath.expjpi(2 * arg)
        ref[j] = complex(s)
    assert oracle.rel_l2_error(got, ref) < 1e-15


def test_O1i_equispaced_reduces_to_idft_and_origin():
    """x_j = N^{-1} ⊙ j (j in I_N): Eq. 6 is the inverse DFT (Eq. 4) up to the index shift,
    i.e. prod N_t * numpy.fft.ifftn; a point at the origin gives sum_k fhat(k)."""
    N = (8, 6, 4)
    x = inputs.equispaced_points(N)
    rng = np.random.default_rng(7)
    fh = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    got = oracle.ndft_inverse_direct(x, fh, N).reshape(N)
    # fhat index k + N/2 -> numpy index k mod N; output j + N/2 <- numpy index j mod N
    G = np.fft.ifftn(np.fft.ifftshift(fh)) * np.prod(N)
    ref = np.fft.fftshift(G)
    assert oracle.rel_l2_error(got, ref) < 1e-14
    o = oracle.ndft_inverse_direct(np.zeros((1, 3)), fh, N)
    assert abs(o[0] - fh.sum()) < 1e-12


def test_O1i_is_the_adjoint_of_O1():
    """Eq. 6 is A^H of Eq. 5's matrix A: <A f, g> = <f, A^H g> for any f, g."""
    N = (8, 8, 6)
    x = inputs.uniform_points(200, seed=21)
    f = inputs.uniform_values(200, seed=21)
    rng = np.random.default_rng(21)
    g = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    lhs = np.vdot(g, oracle.ndft_direct(x, f, N))
    rhs = np.vdot(oracle.ndft_inverse_direct(x, g, N), f)
    assert abs(lhs - rhs) / abs(lhs) < 1e-13


def test_O2i_is_the_transpose_of_O2():
    """The inverse CUNFFT (subdivide, inverse FFT, interpolate) is exactly the
    adjoint of the pinned O2 chain (spread, FFT, deconvolve/crop): <O2 f, g> = <f, O2i g> to
    rounding, for both windows and odd/boundary points.  A dropped factor, a wrong sign or a
    transposed index in any O2i step breaks this identity."""
    N = (8, 16, 4)
    x = inputs.uniform_points(300, seed=23)
    x[0] = [0.5, -0.5, 0.0]
    x[1] = [0.25, 0.125, -0.375]   # on grid nodes
    f = inputs.uniform_values(300, seed=23)
    rng = np.random.default_rng(23)
    g = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    for win, m in ((windows.KAISER_BESSEL, 4), (windows.KAISER_BESSEL, 6), (windows.GAUSSIAN, 3)):
        lhs = np.vdot(g, oracle.nfft_adjoint(x, f, N, m=m, window=win))
        rhs = np.vdot(oracle.nfft_inverse(x, g, N, m=m, window=win), f)
        assert abs(lhs - rhs) / abs(lhs) < 1e-13


def test_O2i_accuracy_vs_O1i_paper_section4():
    """§4 setup ("the obtained precision data of HP-NFFT and its inverse process"):
    E2(O2i vs O1i) decays with m and meets 1e-9 at m = 6, like the forward direction."""
    setup = json.load(open(os.path.join(GOLDEN, "paper_section4_setup.json")))
    M, N = setup["M"], tuple(setup["N"])
    x = inputs.uniform_points(M)
    rng = np.random.default_rng(4)
    fh = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    s = oracle.ndft_inverse_direct(x, fh, N)
    errs = [oracle.rel_l2_error(oracle.nfft_inverse(x, fh, N, m=m), s) for m in (2, 4, 6)]
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < setup["north_star_e2_bar_m6"]


# ------------------------------------------------ O2 parallel spread, d = 1 and 2 (NEXT #4) --
def test_O2_spread_thread_count_invariant():
    """The plane-ownership OpenMP spread gives every node its
    contributions in the serial order: bit-identical results for 1, 3 and 8 threads, also on a
    grid smaller than the stencil (n = 4 < 2m: the taps wrap onto the same planes)."""
    for n, m, M in [((32, 16, 8), 6, 3000), ((4, 8, 16), 3, 500)]:
        x = inputs.clustered_points(M, s=0.05, seed=32)
        f = inputs.uniform_values(M, seed=32)
        ref = oracle.spread(x, f, n, m, 2.0, nthreads=1)
        for T in (3, 8):
            assert np.array_equal(oracle.spread(x, f, n, m, 2.0, nthreads=T), ref)


def _gather_low_dim(x, f, n, m, sigma, window):
    """Spreading per lattice node as a gather over all points and periodic images,
    for any d, written independently of oracle.c."""
    d = len(n)
    g = np.zeros(n, dtype=complex)
    for j in range(x.shape[0]):
        tot = []
        for t in range(d):
            u = n[t] * x[j, t]
            l = np.arange(n[t])
            tot.append(sum(windows.phi(u - (l + r * n[t]), m, sigma, window) for r in range(-3, 4)))
        w = tot[0]
        for t in range(1, d):
            w = np.multiply.outer(w, tot[t])
        g += f[j] * w
    return g


@pytest.mark.parametrize("d", [1, 2])
def test_O2_low_dim_spread_equals_lattice_gather(d):
    """d = 1, 2 (I_N and Eq. 5 are defined for any d): the oracle's spread,
    whose missing dimensions are a single tap of weight exactly 1, equals the per-node gather."""
    n = (32,) if d == 1 else (16, 8)
    x = inputs.uniform_points(25, seed=33, d=d)
    x[0, 0] = 0.5
    f = inputs.uniform_values(25, seed=33)
    for win in (windows.KAISER_BESSEL, windows.GAUSSIAN):
        a = oracle.spread(x, f, n, 3, 2.0, win)
        assert a.shape == n
        assert oracle.rel_l2_error(a, _gather_low_dim(x, f, n, 3, 2.0, win)) < 1e-13


@pytest.mark.parametrize("d,N,M", [(1, (256,), 700), (2, (32, 64), 3000)])
def test_O2_low_dim_accuracy_and_adjoint_identity(d, N, M):
    """d = 1, 2: O2 against the direct NDFT within the KB error bound (and <= 1e-9 at m = 6,
    north_star), exact grid-shift covariance, and the adjoint identity <A f, g> = <f, A^H g>
    between the O2 and O2i chains."""
    x = inputs.uniform_points(M, seed=34, d=d)
    f = inputs.uniform_values(M, seed=34)
    s = oracle.ndft_direct(x, f, N)
    sigma = 2.0
    for m in (2, 4, 6):
        e = oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N, m=m), s)
        bound = 4 * np.pi * (np.sqrt(m) + m) * (1 - 1 / sigma) ** 0.25 * np.exp(-2 * np.pi * m * np.sqrt(1 - 1 / sigma))
        assert bound / 1e3 < e < bound
    assert oracle.rel_l2_error(oracle.nfft_adjoint(x, f, N), s) < 1e-9
    n = oracle.grid_size(N, sigma)
    shift = np.array([3.0 / n[t] for t in range(d)])
    a = oracle.nfft_adjoint(inputs.wrap(x + shift), f, N)
    k = np.meshgrid(*[np.arange(-v // 2, v // 2) for v in N], indexing="ij")
    ph = np.exp(-2j * np.pi * sum(k[t] * shift[t] for t in range(d)))
    assert oracle.rel_l2_error(a, oracle.nfft_adjoint(x, f, N) * ph) < 1e-14
    rng = np.random.default_rng(d)
    gh = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    lhs = np.vdot(gh, oracle.nfft_adjoint(x, f, N))
    rhs = np.vdot(oracle.nfft_inverse(x, gh, N), f)
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
