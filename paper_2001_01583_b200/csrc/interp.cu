// interp.cu -- the inverse direction (Eq. 6):
//     f(x_j) = sum_{k in I_N} fhat(k) exp(+2 pi i k.x_j),
// by the inverse CUNFFT of Alg. 5: Subdividing + Inverse FFT (fft.cu,
// subdivide_and_ifft) and the Interpolating step here:
//     f_j = sum_l g(l) prod_t Phi(n_t x_jt - l_t)      (the spread's transpose, same 2m taps)
// No atomics ("the mutex error ... is not available"): every point is a
// gather.  One warp per point, points in bin-sorted order (set_points) so that the warps of a CTA
// gather overlapping footprints from L1/L2.  Lanes (r, i2), r = lane / 12 in {0, 1}, i2 = lane
// mod 12 (24 of 32 lanes; i2 runs along the contiguous l2, 192-byte rows): lane (r, i2) sums
// the rows i1 = r, r + 2, ... of every plane i0, weighted by w0[i0] w1[i1]; times w2[i2] and a
// warp reduction at the end.  The 3 x 2m tap weights come from the window polynomials
// (tables.cu), one per lane, exchanged by shuffles.
#include "spread_common.cuh"

namespace hpnfft {

namespace {

constexpr int kPointsPerCta = 1024;

template <int M_>
__global__ void __launch_bounds__(256) k_interpolate(const double2* __restrict__ g, const double* __restrict__ xs,
                                                      const uint32_t* __restrict__ perm,
                                                      const double* __restrict__ poly_g, double2* __restrict__ f,
                                                      int64_t M, int n0, int n1, int n2, int lead, double sigma,
                                                      int window) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  // lanes (r, i2): R row groups of W lanes (R = 2 for 2m <= 16; m = 9..15: one group of 2m lanes)
  constexpr int R = 2 * W <= 32 ? 2 : 1;
  constexpr int NR = W / R;                 // rows i1 per lane
  constexpr int TR = (3 * W + 31) / 32;     // shuffle rounds holding the 3 x 2m tap weights
  static_assert(W <= 32, "one lane per tap along l2");
  __shared__ double poly[W * PD];
  for (int e = threadIdx.x; e < W * PD; e += blockDim.x) poly[e] = poly_g[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  // A CTA walks one run of kPointsPerCta consecutive sorted points (its warps interleaved), so
  // the footprints it gathers stay close together and are partly served from the SM's L1.
  // (Measured: persistent grid-stride runs of 64 / 256 points raise the L2 hit rate to 92 % but
  // run slower, 38.8 / 34.5 ms vs 27.7 ms at config 4: the gather is bound by L1 wavefronts.)
  {
  const int64_t k_begin = (int64_t)blockIdx.x * kPointsPerCta;
  const int64_t k_end = min(M, k_begin + (int64_t)kPointsPerCta);
  for (int64_t k = k_begin + (threadIdx.x >> 5); k < k_end; k += nwarps) {
  const CellT a0 = cell_of(xs[3 * k], n0), a1 = cell_of(xs[3 * k + 1], n1), a2 = cell_of(xs[3 * k + 2], n2);
  // tap weights: value q = 32 * round + lane is tap q % W of dimension q / W
  auto tap = [&](int q) -> double {
    const int d = q / W, i = q - d * W;
    const double tt = d == 0 ? a0.t : (d == 1 ? a1.t : a2.t);
    if (d < lead) return i == M_ - 1 ? 1.0 : 0.0;   // trivial dimension of a d < 3 plan: the tap l = c = 0
    return q < 3 * W ? tap_w<M_>(poly, i, tt, sigma, window) : 0.0;
  };
  double tv[TR];
#pragma unroll
  for (int u = 0; u < TR; ++u) tv[u] = tap(32 * u + lane);
  auto weight = [&](int q) -> double {   // warp-uniform q; every lane takes part in the shuffles
    double v = 0.0;
#pragma unroll
    for (int u = 0; u < TR; ++u) {
      const double s = __shfl_sync(0xffffffffu, tv[u], q & 31);
      if ((q >> 5) == u) v = s;
    }
    return v;
  };
  const int r = lane / W, i2 = lane - r * W;     // r in [0, R) for the R W active lanes
  const bool act = lane < R * W;
  const int l2 = (a2.c - M_ + 1 + (act ? i2 : 0)) & (n2 - 1);
  // this lane's rows i1 = r, r + R, ...: their w1 and grid row offsets, fetched once per point
  double w1r[NR];
  int row[NR];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    double wq = 0.0;
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const double w = weight(W + R * q + rr);   // all lanes shuffle
      if (rr == r) wq = w;
    }
    w1r[q] = wq;
    row[q] = ((a1.c - M_ + 1 + R * q + r) & (n1 - 1)) * n2 + l2;
  }
  double sr = 0.0, si = 0.0, tr = 0.0, ti = 0.0;   // two accumulator pairs: shorter FMA chains
  const int i0lo = lead >= 1 ? M_ - 1 : 0, i0hi = lead >= 1 ? M_ : W;
#pragma unroll 2
  for (int i0 = i0lo; i0 < i0hi; ++i0) {
    const double w0 = weight(i0);
    const int l0 = (a0.c - M_ + 1 + i0) & (n0 - 1);
    const double2* plane = g + (size_t)l0 * n1 * n2;
    if (act) {
      double2 v[NR];
#pragma unroll
      for (int q = 0; q < NR; ++q) v[q] = __ldg(plane + row[q]);
#pragma unroll
      for (int q = 0; q < NR; q += 2) {
        const double wa = w0 * w1r[q];
        sr = fma(wa, v[q].x, sr);
        si = fma(wa, v[q].y, si);
        if (q + 1 < NR) {
          const double wb = w0 * w1r[q + 1];
          tr = fma(wb, v[q + 1].x, tr);
          ti = fma(wb, v[q + 1].y, ti);
        }
      }
    }
  }
  sr += tr;
  si += ti;
  const double w2raw = weight(2 * W + (act ? i2 : 0));
  const double w2 = act ? w2raw : 0.0;
  sr *= w2;
  si *= w2;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  if (lane == 0) f[perm[k]] = make_double2(sr, si);
  }
  }
}

template <int M_>
int launch_interp(Plan* p, double* f) {
  const int64_t M = p->M;
  if (M == 0) return HPNFFT_OK;
  constexpr int kWarps = 8;
  const int64_t blocks = (M + kPointsPerCta - 1) / kPointsPerCta;
  k_interpolate<M_><<<(unsigned)blocks, 32 * kWarps, 0, p->stream>>>(
      reinterpret_cast<const double2*>(p->grid), p->xs, p->perm, p->poly, reinterpret_cast<double2*>(f), M,
      (int)p->n[0], (int)p->n[1], (int)p->n[2], 3 - p->d, p->sigma, p->window);
  p->launches++;
  return check_launch(p, "interpolate");
}

}  // namespace

int interpolate(Plan* p, double* f) {
  switch (p->m) {
    case 1: return launch_interp<1>(p, f);
    case 2: return launch_interp<2>(p, f);
    case 3: return launch_interp<3>(p, f);
    case 4: return launch_interp<4>(p, f);
    case 5: return launch_interp<5>(p, f);
    case 6: return launch_interp<6>(p, f);
    case 7: return launch_interp<7>(p, f);
    case 8: return launch_interp<8>(p, f);
    case 9: return launch_interp<9>(p, f);
    case 10: return launch_interp<10>(p, f);
    case 11: return launch_interp<11>(p, f);
    case 12: return launch_interp<12>(p, f);
    case 13: return launch_interp<13>(p, f);
    case 14: return launch_interp<14>(p, f);
    case 15: return launch_interp<15>(p, f);
    default:
      set_error("m not supported by the interpolation kernel");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
