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

template <int M_>
__global__ void __launch_bounds__(256) k_interpolate(const double2* __restrict__ g, const double* __restrict__ xs,
                                                      const uint32_t* __restrict__ perm,
                                                      const double* __restrict__ poly_g, double2* __restrict__ f,
                                                      int64_t M, int n0, int n1, int n2) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  static_assert(3 * W <= 64, "two shuffle rounds of taps");
  __shared__ double poly[W * PD];
  for (int e = threadIdx.x; e < W * PD; e += blockDim.x) poly[e] = poly_g[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= M) return;
  const CellT a0 = cell_of(xs[3 * k], n0), a1 = cell_of(xs[3 * k + 1], n1), a2 = cell_of(xs[3 * k + 2], n2);
  // tap weights: value q = 32 * round + lane is tap q % W of dimension q / W
  auto tap = [&](int q) -> double {
    const int d = q / W, i = q - d * W;
    const double tt = d == 0 ? a0.t : (d == 1 ? a1.t : a2.t);
    return q < 3 * W ? tap_weight(poly, i, tt, M_) : 0.0;
  };
  const double tv0 = tap(lane), tv1 = tap(32 + lane);
  auto weight = [&](int q) -> double {   // warp-uniform q
    const double v0 = __shfl_sync(0xffffffffu, tv0, q & 31);
    const double v1 = __shfl_sync(0xffffffffu, tv1, q & 31);
    return q < 32 ? v0 : v1;
  };
  const int r = lane / W, i2 = lane - r * W;     // r in {0, 1} for the 2W active lanes
  const bool act = lane < 2 * W;
  const int l2 = (a2.c - M_ + 1 + (act ? i2 : 0)) & (n2 - 1);
  double sr = 0.0, si = 0.0;
#pragma unroll 2
  for (int i0 = 0; i0 < W; ++i0) {
    const double w0 = weight(i0);
    const int l0 = (a0.c - M_ + 1 + i0) & (n0 - 1);
    const double2* plane = g + (size_t)l0 * n1 * n2;
#pragma unroll
    for (int i1 = 0; i1 < W; i1 += 2) {
      const double w1a = weight(W + i1), w1b = weight(W + i1 + 1);   // all lanes shuffle
      const double w01 = w0 * (r == 0 ? w1a : w1b);
      const int l1 = (a1.c - M_ + 1 + i1 + r) & (n1 - 1);
      if (act) {
        const double2 v = __ldg(plane + (size_t)l1 * n2 + l2);
        sr = fma(w01, v.x, sr);
        si = fma(w01, v.y, si);
      }
    }
  }
  // (weight() shuffles: every lane calls it, the idle ones with a dummy index)
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

template <int M_>
int launch_interp(Plan* p, double* f) {
  const int64_t M = p->M;
  if (M == 0) return HPNFFT_OK;
  constexpr int kWarps = 8;
  const int64_t blocks = (M + kWarps - 1) / kWarps;
  k_interpolate<M_><<<(unsigned)blocks, 32 * kWarps, 0, p->stream>>>(
      reinterpret_cast<const double2*>(p->grid), p->xs, p->perm, p->poly, reinterpret_cast<double2*>(f), M,
      (int)p->n[0], (int)p->n[1], (int)p->n[2]);
  p->launches++;
  return check_launch(p, "interpolate");
}

}  // namespace

int interpolate(Plan* p, double* f) {
  switch (p->m) {
    case 2: return launch_interp<2>(p, f);
    case 3: return launch_interp<3>(p, f);
    case 4: return launch_interp<4>(p, f);
    case 5: return launch_interp<5>(p, f);
    case 6: return launch_interp<6>(p, f);
    case 7: return launch_interp<7>(p, f);
    case 8: return launch_interp<8>(p, f);
    default:
      set_error("m not supported by the interpolation kernel");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
