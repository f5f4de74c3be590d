/*
 * oracle.c -- plain CPU oracle for the HP-NFFT adjoint path (TEST INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference)
 * may load this library.  It shares no code, header, table or constant generator with
 * the CUDA path (paper_2001_01583_b200/csrc/).
 *
 * O1  oracle_ndft    : direct NDFT, Eq. (5) of PAPER.md:37 (§1),
 *                      fhat(k) = sum_{j<M} f_j exp(-2 pi i k.x_j), k in I_N,
 *                      Kahan-compensated complex accumulation in float64, one output at a
 *                      time (OpenMP over independent outputs only; every sum is serial).
 * O2a oracle_spread  : the "Spreading" step of CUNFFT (§2 Fig. 1 and
 *                      PAPER.md:162, §3): g(l) += f_j * prod_t Phi(u_t - l_t) over the
 *                      truncated neighbourhood J(x_j), l taken modulo n (periodic grid).
 *                      Loop over points in order, taps in natural order; OpenMP threads own
 *                      disjoint dimension-0 grid planes (bit-identical to the serial loop).
 * O1i oracle_ndft_inverse : direct inverse NDFT, Eq. (6) of PAPER.md:43 (§1),
 *                      f(x_j) = sum_{k in I_N} fhat(k) exp(+2 pi i k.x_j), Kahan-summed, one
 *                      output point at a time (OpenMP over points only).
 * O2i oracle_interp  : the "Interpolating" step of inverse CUNFFT (§2 Fig. 2 and
 *                      PAPER.md:242, §3): f_j = sum_l g(l) prod_t Phi(u_t - l_t) over the same
 *                      truncated neighbourhood as oracle_spread (its transpose).
 *
 * Conventions (readings Q1-Q10):
 *   u_t = n_t x_t (exact: n_t a power of two), c_t = floor(u_t), t_t = u_t - c_t (exact),
 *   taps l_t = c_t - m + 1 + i, i = 0..2m-1, u_t - l_t = t_t + (m - 1 - i).
 *   Strict truncation |u - l| < m: all taps are inside except i = 2m-1 when t_t == 0
 *   (then u - l = -m exactly).  Kaiser-Bessel b = pi(2 - 1/sigma); Gaussian
 *   b = 2 sigma/(2 sigma - 1) m / pi (see oracle/windows.py for the formulas).
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_KB 0
#define ORACLE_GAUSS 1
#define ORACLE_BSPLINE 2
#define ORACLE_SINC_POWER 3

static const double PI = 3.14159265358979323846264338327950288;

/* exp(-2 pi i k x) with the argument k*x reduced exactly: k*x = p + e (fma gives the
 * exact product error e), r = (p - nearbyint(p)) + e, phase = exp(-2 pi i r). */
static inline void phase(int64_t k, double x, double* re, double* im) {
  double kd = (double)k;
  double p = kd * x;
  double e = fma(kd, x, -p);
  double r = (p - nearbyint(p)) + e;
  double s, c;
  sincos(2.0 * PI * r, &s, &c);
  *re = c;
  *im = -s;
}

/* O1: direct NDFT.  x: [M][d], f: [M][2] (re,im), ks: [K][d] integer frequencies
 * (or NULL: all of I_N in row-major order, last dimension fastest, index k_t + N_t/2).
 * out: [K][2].  Returns 0 on success. */
int oracle_ndft(int d, const int64_t* N, int64_t M, const double* x, const double* f,
                int64_t K, const int64_t* ks, double* out, int nthreads) {
  if (d < 1 || d > 3) return -1;
  int64_t total = 1;
  for (int t = 0; t < d; ++t) total *= N[t];
  if (ks == NULL) K = total;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t q = 0; q < K; ++q) {
    int64_t k[3] = {0, 0, 0};
    if (ks) {
      for (int t = 0; t < d; ++t) k[t] = ks[q * d + t];
    } else {
      int64_t r = q;
      for (int t = d - 1; t >= 0; --t) {
        k[t] = (r % N[t]) - N[t] / 2;
        r /= N[t];
      }
    }
    double sr = 0.0, si = 0.0, cr = 0.0, ci = 0.0; /* Kahan sums and compensations */
    for (int64_t j = 0; j < M; ++j) {
      double er = 1.0, ei = 0.0;
      for (int t = 0; t < d; ++t) {
        double pr, pi_;
        phase(k[t], x[j * d + t], &pr, &pi_);
        double nr = er * pr - ei * pi_;
        double ni = er * pi_ + ei * pr;
        er = nr;
        ei = ni;
      }
      double fr = f[2 * j], fi = f[2 * j + 1];
      double vr = fr * er - fi * ei;
      double vi = fr * ei + fi * er;
      double y, tt;
      y = vr - cr; tt = sr + y; cr = (tt - sr) - y; sr = tt;
      y = vi - ci; tt = si + y; ci = (tt - si) - y; si = tt;
    }
    out[2 * q] = sr;
    out[2 * q + 1] = si;
  }
  return 0;
}

/* Window Phi(a) for a strictly inside the support (|a| < m). */
/* centred cardinal B-spline M_p(u), Cox-de Boor: M_1 = [-1/2 <= u < 1/2],
 * M_k(y) = ((k/2 + y) M_{k-1}(y + 1/2) + (k/2 - y) M_{k-1}(y - 1/2)) / (k - 1)  (windows.py) */
static double bspline(double u, int p) {
  double v[64];
  for (int j = 0; j < p; ++j) {
    double y = u - 0.5 * (double)(p - 1) + (double)j;
    v[j] = (y >= -0.5 && y < 0.5) ? 1.0 : 0.0;
  }
  for (int k = 2; k <= p; ++k) {
    int r = p - k;
    for (int j = 0; j <= r; ++j) {
      double y = u - 0.5 * (double)r + (double)j;
      v[j] = ((0.5 * k + y) * v[j + 1] + (0.5 * k - y) * v[j]) / (double)(k - 1);
    }
  }
  return v[0];
}

static inline double window_value(double a, int m, double sigma, int window) {
  if (window == ORACLE_KB) {
    double b = PI * (2.0 - 1.0 / sigma);
    double s = sqrt((double)m * (double)m - a * a);
    return sinh(b * s) / (PI * s);
  } else if (window == ORACLE_GAUSS) {
    double b = 2.0 * sigma / (2.0 * sigma - 1.0) * (double)m / PI;
    return exp(-a * a / b) / sqrt(PI * b);
  } else if (window == ORACLE_BSPLINE) {
    return bspline(a, 2 * m);
  } else {
    double beta = (2.0 * sigma - 1.0) / (2.0 * m * sigma);
    double y = PI * beta * a;
    double sc = (y == 0.0) ? 1.0 : sin(y) / y;
    return pow(sc, 2 * m);
  }
}

/* The 2m taps of one coordinate: weights w[i] = Phi(u - l_i) and grid indices l_i mod n,
 * l_i = floor(u) - m + 1 + i (strict truncation |u - l| < m, Q4).  A dimension t >= d
 * of a d < 3 problem is the trivial one (n = 1): a single tap of weight exactly 1. */
static int taps_of(int trivial, double xt, int64_t n, int m, double sigma, int window, double* w, int64_t* idx) {
  if (trivial) {
    w[0] = 1.0;
    idx[0] = 0;
    return 1;
  }
  const int taps = 2 * m;
  double u = (double)n * xt;
  double c = floor(u);
  double tt = u - c;
  int64_t ci = (int64_t)c;
  for (int i = 0; i < taps; ++i) {
    int64_t l = ci - m + 1 + i;
    /* |u - l| < m  <=>  not (i == 2m-1 and tt == 0) */
    int inside = !(i == taps - 1 && tt == 0.0);
    w[i] = inside ? window_value(tt + (double)(m - 1 - i), m, sigma, window) : 0.0;
    int64_t lm = l % n;
    if (lm < 0) lm += n;
    idx[i] = lm;
  }
  return taps;
}

/* O2a: spread.  d in 1..3; n: grid sizes [d]; x: [M][d]; f: [M][2]; g: [n0][n1][n2][2] (the
 * d given dimensions, row-major), accumulated into (caller zeroes it).  Returns 0 on success.
 * Parallel by grid-plane ownership: thread r owns the dimension-0 planes
 * [r n0 / T, (r+1) n0 / T) and visits every point in input order, applying only the taps whose
 * plane it owns.  Every grid node therefore receives its contributions in exactly the order of
 * the serial loop (points in order, taps in natural order): no atomics, no private grids, the
 * result is bit-identical to the serial loop for any thread count. */
int oracle_spread(int d, const int64_t* n, int m, double sigma, int window, int64_t M,
                  const double* x, const double* f, double* g, int nthreads) {
  if (m < 1 || m > 16 || d < 1 || d > 3) return -1;
  int64_t nn[3] = {1, 1, 1};
  for (int t = 0; t < d; ++t) nn[t] = n[t];
  int T = 1;
#ifdef _OPENMP
  T = nthreads > 0 ? nthreads : omp_get_max_threads();
  if (T > nn[0]) T = (int)nn[0];
#pragma omp parallel num_threads(T)
#endif
  {
    int r = 0;
#ifdef _OPENMP
    r = omp_get_thread_num();
#endif
    const int64_t p_lo = nn[0] * r / T, p_hi = nn[0] * (r + 1) / T;
    double w[3][32];
    int64_t idx[3][32];
    int nt[3];
    for (int64_t j = 0; j < M; ++j) {
      /* ownership test on the plane indices alone (no window evaluation for foreign points) */
      const int64_t c0 = (int64_t)floor((double)nn[0] * x[j * d]);
      int mine = 0;
      for (int i0 = 0; i0 < 2 * m; ++i0) {
        int64_t l = (c0 - m + 1 + i0) % nn[0];
        if (l < 0) l += nn[0];
        mine |= l >= p_lo && l < p_hi;
      }
      if (!mine) continue;
      nt[0] = taps_of(0, x[j * d], nn[0], m, sigma, window, w[0], idx[0]);
      for (int t = 1; t < 3; ++t) nt[t] = taps_of(t >= d, t < d ? x[j * d + t] : 0.0, nn[t], m, sigma, window, w[t], idx[t]);
      const double fr = f[2 * j], fi = f[2 * j + 1];
      for (int i0 = 0; i0 < nt[0]; ++i0) {
        if (idx[0][i0] < p_lo || idx[0][i0] >= p_hi) continue;
        for (int i1 = 0; i1 < nt[1]; ++i1) {
          for (int i2 = 0; i2 < nt[2]; ++i2) {
            double wt = w[0][i0] * w[1][i1] * w[2][i2];
            int64_t off = ((idx[0][i0] * nn[1] + idx[1][i1]) * nn[2] + idx[2][i2]) * 2;
            g[off] += fr * wt;
            g[off + 1] += fi * wt;
          }
        }
      }
    }
  }
  return 0;
}

/* 1-D weights of one coordinate (exposed for the window/tap pins in tests). */
int oracle_taps(int64_t n, int m, double sigma, int window, double x, double* w, int64_t* idx) {
  taps_of(0, x, n, m, sigma, window, w, idx);
  return 0;
}

/* O1i: direct inverse NDFT.  x: [M][d]; fhat: all of I_N in row-major order (index k_t + N_t/2),
 * [|I_N|][2]; out: [M][2].  exp(+2 pi i k x) = conj(phase(k, x)).  Returns 0 on success. */
int oracle_ndft_inverse(int d, const int64_t* N, int64_t M, const double* x, const double* fhat, double* out,
                        int nthreads) {
  if (d < 1 || d > 3) return -1;
  int64_t total = 1;
  for (int t = 0; t < d; ++t) total *= N[t];
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t j = 0; j < M; ++j) {
    double sr = 0.0, si = 0.0, cr = 0.0, ci = 0.0;
    for (int64_t q = 0; q < total; ++q) {
      int64_t k[3] = {0, 0, 0};
      int64_t r = q;
      for (int t = d - 1; t >= 0; --t) {
        k[t] = (r % N[t]) - N[t] / 2;
        r /= N[t];
      }
      double er = 1.0, ei = 0.0;
      for (int t = 0; t < d; ++t) {
        double pr, pi_;
        phase(k[t], x[j * d + t], &pr, &pi_);
        pi_ = -pi_; /* exp(+2 pi i k x) */
        double nr = er * pr - ei * pi_;
        double ni = er * pi_ + ei * pr;
        er = nr;
        ei = ni;
      }
      double fr = fhat[2 * q], fi = fhat[2 * q + 1];
      double vr = fr * er - fi * ei;
      double vi = fr * ei + fi * er;
      double y, tt;
      y = vr - cr; tt = sr + y; cr = (tt - sr) - y; sr = tt;
      y = vi - ci; tt = si + y; ci = (tt - si) - y; si = tt;
    }
    out[2 * j] = sr;
    out[2 * j + 1] = si;
  }
  return 0;
}

/* O2i: interpolate.  d in 1..3; n: grid sizes [d]; g: [n0][n1][n2][2]; x: [M][d]; out f: [M][2].
 * Same taps and weights as oracle_spread (the interpolation is the spread's transpose); every
 * output is an independent serial sum (OpenMP over points only). */
int oracle_interp(int d, const int64_t* n, int m, double sigma, int window, int64_t M, const double* x,
                  const double* g, double* f, int nthreads) {
  if (m < 1 || m > 16 || d < 1 || d > 3) return -1;
  int64_t nn[3] = {1, 1, 1};
  for (int t = 0; t < d; ++t) nn[t] = n[t];
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t j = 0; j < M; ++j) {
    double w[3][32];
    int64_t idx[3][32];
    int nt[3];
    for (int t = 0; t < 3; ++t) nt[t] = taps_of(t >= d, t < d ? x[j * d + t] : 0.0, nn[t], m, sigma, window, w[t], idx[t]);
    double sr = 0.0, si = 0.0;
    for (int i0 = 0; i0 < nt[0]; ++i0) {
      for (int i1 = 0; i1 < nt[1]; ++i1) {
        for (int i2 = 0; i2 < nt[2]; ++i2) {
          double wt = w[0][i0] * w[1][i1] * w[2][i2];
          int64_t off = ((idx[0][i0] * nn[1] + idx[1][i1]) * nn[2] + idx[2][i2]) * 2;
          sr += g[off] * wt;
          si += g[off + 1] * wt;
        }
      }
    }
    f[2 * j] = sr;
    f[2 * j + 1] = si;
  }
  return 0;
}
