// spread_atomic.cu -- generic spreading kernel (A4 of SURVEY.md §8(a)), the paper's scheme:
// "each thread is responsible for one point ... AtomicAdd()" (§3), refined to one
// thread per (point, tap i0) so a point's (2m)^3 stencil is split over 2m threads.
//   g(l) += f_j * w0[i0] * w1[i1] * w2[i2]   over the 2m x 2m taps (i1, i2) of this thread,
// with native FP64 global atomics (RED.E.ADD.F64) into the zeroed grid.  Points are visited
// in sorted (bin) order for L2 locality.  Works for every supported grid (n_t >= 2m); it is
// the correctness baseline that the sweep kernel (spread_sweep.cu) is measured against.
#include "spread_common.cuh"

namespace hpnfft {

template <int M_>
__global__ void k_spread_atomic(const double* __restrict__ xs, const uint32_t* __restrict__ perm,
                                const double* __restrict__ f, int64_t M, int64_t n0, int64_t n1, int64_t n2,
                                const double* __restrict__ poly_g, double* __restrict__ grid, int lead,
                                double sigma, int window, int real) {
  constexpr int W = 2 * M_;
  __shared__ double poly[W * (kPolyDeg + 1)];
  for (int e = threadIdx.x; e < W * (kPolyDeg + 1); e += blockDim.x) poly[e] = poly_g[e];
  __syncthreads();
  // trivial leading dimensions of a d < 3 plan (lead = 3 - d): the single tap i = m - 1 (node
  // l = c = 0) of weight exactly 1
  const int W0 = lead >= 1 ? 1 : W;
  int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= M * W0) return;
  int64_t j = gid / W0;
  int i0 = lead >= 1 ? M_ - 1 : (int)(gid % W0);
  CellT a0 = cell_of(xs[3 * j], n0), a1 = cell_of(xs[3 * j + 1], n1), a2 = cell_of(xs[3 * j + 2], n2);
  uint32_t src = perm[j];
  double fr = f[2 * (int64_t)src], fi = f[2 * (int64_t)src + 1];
  double w0 = lead >= 1 ? 1.0 : tap_w<M_>(poly, i0, a0.t, sigma, window);
  double w1[W], w2[W];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    w1[i] = lead >= 2 ? (i == M_ - 1 ? 1.0 : 0.0) : tap_w<M_>(poly, i, a1.t, sigma, window);
    w2[i] = tap_w<M_>(poly, i, a2.t, sigma, window);
  }
  const int i1lo = lead >= 2 ? M_ - 1 : 0, i1hi = lead >= 2 ? M_ : W;
  int64_t l0 = (a0.c - M_ + 1 + i0) & (n0 - 1);
  double gr = fr * w0, gi = fi * w0;
#pragma unroll 1
  for (int i1 = i1lo; i1 < i1hi; ++i1) {
    int64_t l1 = (a1.c - M_ + 1 + i1) & (n1 - 1);
    double hr = gr * w1[i1], hi = gi * w1[i1];
    if (real) {   // real values onto the REAL grid [n0][n1][n2] (NEXT #2)
      double* row = grid + (l0 * n1 + l1) * n2;
#pragma unroll
      for (int i2 = 0; i2 < W; ++i2) atomicAdd(row + ((a2.c - M_ + 1 + i2) & (n2 - 1)), hr * w2[i2]);
      continue;
    }
    double* row = grid + 2 * ((l0 * n1 + l1) * n2);
#pragma unroll
    for (int i2 = 0; i2 < W; ++i2) {
      int64_t l2 = (a2.c - M_ + 1 + i2) & (n2 - 1);
      atomicAdd(row + 2 * l2, hr * w2[i2]);
      atomicAdd(row + 2 * l2 + 1, hi * w2[i2]);
    }
  }
}

template <int M_>
static int launch_atomic(Plan* p, const double* f) {
  const int lead = 3 - p->d;
  int64_t total = p->M * (lead >= 1 ? 1 : 2 * M_);
  if (total == 0) return HPNFFT_OK;
  k_spread_atomic<M_><<<(unsigned)((total + 255) / 256), 256, 0, p->stream>>>(
      p->xs, p->perm, f, p->M, p->n[0], p->n[1], p->n[2], p->poly, p->grid, lead, p->sigma, p->window,
      p->real_values ? 1 : 0);
  p->launches++;
  return check_launch(p, "spread_atomic");
}

int spread_atomic(Plan* p, const double* f) {
  size_t bytes = sizeof(double) * (p->real_values ? 1 : 2) * (size_t)(p->n[0] * p->n[1] * p->n[2]);
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->grid, 0, bytes, p->stream), "zero grid");
  switch (p->m) {
    case 1: return launch_atomic<1>(p, f);
    case 2: return launch_atomic<2>(p, f);
    case 3: return launch_atomic<3>(p, f);
    case 4: return launch_atomic<4>(p, f);
    case 5: return launch_atomic<5>(p, f);
    case 6: return launch_atomic<6>(p, f);
    case 7: return launch_atomic<7>(p, f);
    case 8: return launch_atomic<8>(p, f);
    case 9: return launch_atomic<9>(p, f);
    case 10: return launch_atomic<10>(p, f);
    case 11: return launch_atomic<11>(p, f);
    case 12: return launch_atomic<12>(p, f);
    case 13: return launch_atomic<13>(p, f);
    case 14: return launch_atomic<14>(p, f);
    case 15: return launch_atomic<15>(p, f);
    default:
      set_error("m not supported by the spread kernels");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
