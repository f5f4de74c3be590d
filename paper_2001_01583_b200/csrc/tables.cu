// tables.cu -- plan-time device tables (A0 in SURVEY.md §8(a)).
//   * 1/c_k per dimension for the deconvolution ("Scaling", §3),
//   * FFT twiddles exp(-2 pi i q/n) from sincospi on exact arguments,
//   * window tap polynomials: tap i of a point with fractional cell offset t = u - floor(u)
//     has weight Phi(t + m - 1 - i); on t in [0,1) it is replaced by a degree-kPolyDeg
//     polynomial in s = 2t - 1 obtained by Chebyshev interpolation (DESIGN.md "Window
//     evaluation": max error ~1e-14 of Phi(0) for KB m = 6).
#include <math.h>

#include "common.cuh"
#include "window.cuh"

namespace hpnfft {

// inv_c[q] = 1 / c(k / n) for k = q - koff, q < count (koff = N/2: k in I_N; the extended tables
// of the real-charge path: count N + 2, koff N/2 + 1)
__global__ void k_deconv_table(double* inv_c, int64_t count, int64_t koff, int64_t n, int m, double sigma, int window,
                               int* bad) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= count) return;
  if (n == 1) {   // a trivial dimension of a d < 3 plan: no deconvolution
    inv_c[q] = 1.0;
    return;
  }
  double k = (double)(q - koff);
  double c = window_fourier(k / (double)n, m, sigma, window);
  if (!isfinite(c) || !(fabs(c) >= 1e-300)) atomicExch(bad, 1);
  inv_c[q] = 1.0 / c;
}

__global__ void k_twiddle_table(double* tw, int64_t n) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  double s, c;
  sincospi(2.0 * (double)q / (double)n, &s, &c);   // exact argument 2q/n
  tw[2 * q] = c;
  tw[2 * q + 1] = -s;
}

// One thread per tap: Chebyshev interpolation at D+1 first-kind nodes, then conversion of the
// Chebyshev series to power-basis coefficients in s (Horner on the device).
__global__ void k_window_poly(double* poly, int m, double sigma, int window) {
  const int D = kPolyDeg;
  int i = threadIdx.x;
  if (i >= 2 * m) return;
  const double kPi = 3.141592653589793238462643383279502884;
  double fv[D + 1], ch[D + 1];
  for (int j = 0; j <= D; ++j) {
    double sj = cospi((j + 0.5) / (D + 1));
    double a = (sj + 1.0) * 0.5 + (double)(m - 1 - i);   // u - l for t = (s+1)/2
    fv[j] = (fabs(a) < m) ? window_exact(a, m, sigma, window) : 0.0;
  }
  for (int k = 0; k <= D; ++k) {
    double acc = 0.0;
    for (int j = 0; j <= D; ++j) acc += fv[j] * cospi((double)k * (j + 0.5) / (D + 1));
    ch[k] = acc * 2.0 / (D + 1);
  }
  ch[0] *= 0.5;
  // power basis: sum_k ch[k] T_k(s); T_k built by T_{k+1} = 2 s T_k - T_{k-1}
  double Tm1[D + 1], T0[D + 1], T1[D + 1], out[D + 1];
  for (int j = 0; j <= D; ++j) { Tm1[j] = 0; T0[j] = 0; out[j] = 0; }
  T0[0] = 1.0;                   // T_0
  for (int j = 0; j <= D; ++j) out[j] += ch[0] * T0[j];
  for (int j = 0; j <= D; ++j) Tm1[j] = T0[j];
  for (int j = 0; j <= D; ++j) T0[j] = (j == 1) ? 1.0 : 0.0;   // T_1 = s
  for (int j = 0; j <= D; ++j) out[j] += ch[1] * T0[j];
  for (int k = 2; k <= D; ++k) {
    for (int j = 0; j <= D; ++j) T1[j] = (j > 0 ? 2.0 * T0[j - 1] : 0.0) - Tm1[j];
    for (int j = 0; j <= D; ++j) { out[j] += ch[k] * T1[j]; Tm1[j] = T0[j]; T0[j] = T1[j]; }
  }
  (void)kPi;
  for (int j = 0; j <= D; ++j) poly[i * (D + 1) + j] = out[j];
}

int build_tables(Plan* p) {
  int* bad = nullptr;
  HPNFFT_CUDA_TRY(p, cudaMallocAsync(&bad, sizeof(int), p->stream), "alloc flag");
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(bad, 0, sizeof(int), p->stream), "memset flag");
  for (int t = 0; t < 3; ++t) {
    int64_t N = p->N[t];
    k_deconv_table<<<(unsigned)((N + 255) / 256), 256, 0, p->stream>>>(p->inv_c[t], N, N / 2, p->n[t], p->m, p->sigma,
                                                                     p->window, bad);
    k_twiddle_table<<<(unsigned)((p->n[t] + 255) / 256), 256, 0, p->stream>>>(p->twiddle[t], p->n[t]);
    if (t < 2)
      k_deconv_table<<<(unsigned)((N + 2 + 255) / 256), 256, 0, p->stream>>>(p->inv_c_ext[t], N + 2, N / 2 + 1, p->n[t],
                                                                           p->m, p->sigma, p->window, bad);
  }
  if (p->n[2] >= 2)
    k_twiddle_table<<<(unsigned)((p->n[2] / 2 + 255) / 256), 256, 0, p->stream>>>(p->twiddle_half, p->n[2] / 2);
  k_window_poly<<<1, 32, 0, p->stream>>>(p->poly, p->m, p->sigma, p->window);
  int rc = check_launch(p, "table kernels");
  if (rc) return rc;
  int hbad = 0;
  HPNFFT_CUDA_TRY(p, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, p->stream), "flag d2h");
  HPNFFT_CUDA_TRY(p, cudaStreamSynchronize(p->stream), "plan sync");
  cudaFreeAsync(bad, p->stream);
  if (hbad) {
    set_error("degenerate window weight: a Fourier weight c_k is not finite or below 1e-300");
    return HPNFFT_E_DEGENERATE_WINDOW;
  }
  return HPNFFT_OK;
}

}  // namespace hpnfft
