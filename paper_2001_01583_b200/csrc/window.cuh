// window.cuh -- device-side window functions of the CUDA path (A3 in SURVEY.md §8(a)).
//
// Kaiser-Bessel in the NFFT convention with the window measured in grid cells u = n x
// (reading Q3; the paper only names the window, and defers the
// formula to its Ref. [28]):
//   b = pi (2 - 1/sigma),  Phi(u) = sinh(b sqrt(m^2-u^2)) / (pi sqrt(m^2-u^2)),  |u| < m
//   c(xi) = I0(m sqrt(b^2 - (2 pi xi)^2))        (Fourier weight, "Scaling")
// Gaussian: b = 2 sigma/(2 sigma - 1) m/pi, Phi(u) = exp(-u^2/b)/sqrt(pi b), c(xi) = exp(-b pi^2 xi^2).
#pragma once

#include <cuda_runtime.h>

namespace hpnfft {

__device__ __forceinline__ double window_exact(double a, int m, double sigma, int window) {
  const double kPi = 3.141592653589793238462643383279502884;
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
  if (window == 0) {
    double b = kPi * (2.0 - 1.0 / sigma);
    double w = 2.0 * kPi * xi;
    return cyl_bessel_i0((double)m * sqrt(b * b - w * w));
  }
  double b = 2.0 * sigma / (2.0 * sigma - 1.0) * (double)m / kPi;
  return exp(-b * kPi * kPi * xi * xi);
}

}  // namespace hpnfft
