// spread_common.cuh -- per-point cell/tap arithmetic shared by the spread kernels (A3).
//   u = n x (exact, n a power of two), c = floor(u), t = u - c in [0,1) (exact),
//   tap i in [0, 2m) is grid node l = c - m + 1 + i with weight Phi(t + m - 1 - i);
//   strict truncation |u - l| < m removes only tap 2m-1 when t == 0 (Q4).
// Phi on each tap interval is the degree-kPolyDeg polynomial in s = 2t - 1 built by
// k_window_poly (tables.cu).
#pragma once

#include "common.cuh"
#include "window.cuh"

namespace hpnfft {

struct CellT {
  int c;      // floor(n x) mod n
  double t;   // fractional offset in [0, 1)
};

__device__ __forceinline__ CellT cell_of(double x, int64_t n) {
  double u = __dmul_rn((double)n, x);
  double c = floor(u);
  CellT r;
  r.t = u - c;
  r.c = (int)((int64_t)c & (n - 1));
  return r;
}

// Weight of tap i for fractional offset t; poly points at [2m][kPolyDeg+1] coefficients.
__device__ __forceinline__ double tap_weight(const double* poly, int i, double t, int m) {
  const double* a = poly + i * (kPolyDeg + 1);
  double s = fma(2.0, t, -1.0);
  double v = a[kPolyDeg];
#pragma unroll
  for (int j = kPolyDeg - 1; j >= 0; --j) v = fma(v, s, a[j]);
  return (i == 2 * m - 1 && t == 0.0) ? 0.0 : v;
}

// Tap weight of the generic kernels (atomic spread, warp gather).  m <= kMaxSweepM: the plan's
// tap polynomial (<= 2e-14 of Phi(0)).  m = 9..15: the window evaluated directly -- at large m
// the deconvolution 1/c_k amplifies a tap error by up to ~1e2 at the spectrum's edge (sinc
// power, B-spline: c(xi) decays fast), so the generic path uses the closed forms (ulp-level).
template <int M_>
__device__ __forceinline__ double tap_w(const double* poly, int i, double t, double sigma, int window) {
  if constexpr (M_ > kMaxSweepM) {
    if (i == 2 * M_ - 1 && t == 0.0) return 0.0;   // strict truncation |u - l| < m
    return window_exact(t + (double)(M_ - 1 - i), M_, sigma, window);
  } else {
    (void)sigma;
    (void)window;
    return tap_weight(poly, i, t, M_);
  }
}

}  // namespace hpnfft
