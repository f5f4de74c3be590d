// window.cuh -- device-side window functions of the CUDA path (A3 in SURVEY.md §8(a)).
//
// Kaiser-Bessel in the NFFT convention with the window measured in grid cells u = n x
// (reading Q3; the paper only names the window, and defers the
// formula to its Ref. [28]):
//   b = pi (2 - 1/sigma),  Phi(u) = sinh(b sqrt(m^2-u^2)) / (pi sqrt(m^2-u^2)),  |u| < m
//   c(xi) = I0(m sqrt(b^2 - (2 pi xi)^2))        (Fourier weight, "Scaling")
// Gaussian: b = 2 sigma/(2 sigma - 1) m/pi, Phi(u) = exp(-u^2/b)/sqrt(pi b), c(xi) = exp(-b pi^2 xi^2).
// B-spline: Phi(u) = M_2m(u), the centred cardinal
//   B-spline of order 2m (exact support [-m, m]), c(xi) = sinc(pi xi)^2m.
// Sinc power (NEXT #3): beta = (2 sigma - 1)/(2 m sigma), Phi(u) = sinc(pi beta u)^2m (|u| < m),
//   c(xi) = M_2m(xi / beta) / beta (the 2m-fold convolution of the box transform of sinc).
// These evaluate only at plan time (tap polynomials, deconvolution tables), never per point.
#pragma once

#include <cuda_runtime.h>

namespace hpnfft {

// M_p(u) by the de Boor triangle: level-1 boxes at u - (p-1)/2 + j, each level k combines
// neighbours: M_k(y) = ((k/2 + y) M_{k-1}(y + 1/2) + (k/2 - y) M_{k-1}(y - 1/2)) / (k - 1).
__device__ inline double cardinal_bspline(double u, int p) {
  double v[32];
  for (int j = 0; j < p; ++j) {
    const double y = u - 0.5 * (double)(p - 1) + (double)j;
    v[j] = (y >= -0.5 && y < 0.5) ? 1.0 : 0.0;
  }
  for (int k = 2; k <= p; ++k) {
    const int r = p - k;
    for (int j = 0; j <= r; ++j) {
      const double y = u - 0.5 * (double)r + (double)j;
      v[j] = ((0.5 * k + y) * v[j + 1] + (0.5 * k - y) * v[j]) / (double)(k - 1);
    }
  }
  return v[0];
}

__device__ inline double sinc_of(double y) { return y == 0.0 ? 1.0 : sin(y) / y; }

__device__ __forceinline__ double window_exact(double a, int m, double sigma, int window) {
  const double kPi = 3.141592653589793238462643383279502884;
  if (window == 2) return cardinal_bspline(a, 2 * m);
  if (window == 3) {
    const double beta = (2.0 * sigma - 1.0) / (2.0 * m * sigma);
    return pow(sinc_of(kPi * beta * a), (double)(2 * m));   // one rounding, not 2m (m up to 15)
  }
  if (window == 0) {
    double b = kPi * (2.0 - 1.0 / sigma);
    double s = sqrt((double)m * (double)m - a * a);
    return sinh(b * s) / (kPi * s);
  }
  double b = 2.0 * sigma / (2.0 * sigma - 1.0) * (double)m / kPi;
  return exp(-a * a / b) / sqrt(kPi * b);
}

__device__ __forceinline__ double window_fourier(double xi, int m, double sigma, int window) {
  const double kPi = 3.141592653589793238462643383279502884;
  if (window == 2) {
    const double sc = sinc_of(kPi * xi);
    double r = 1.0;
    for (int i = 0; i < 2 * m; ++i) r *= sc;
    return r;
  }
  if (window == 3) {
    const double beta = (2.0 * sigma - 1.0) / (2.0 * m * sigma);
    return cardinal_bspline(xi / beta, 2 * m) / beta;
  }
  if (window == 0) {
    double b = kPi * (2.0 - 1.0 / sigma);
    double w = 2.0 * kPi * xi;
    return cyl_bessel_i0((double)m * sqrt(b * b - w * w));
  }
  double b = 2.0 * sigma / (2.0 * sigma - 1.0) * (double)m / kPi;
  return exp(-b * kPi * kPi * xi * xi);
}

}  // namespace hpnfft
