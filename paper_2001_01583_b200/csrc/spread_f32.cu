// spread_f32.cu -- the spreading step of the FP32 plans (default: k_spread_red_f32 below; the box
// kernel described next is the measured alternative) ("lower-precision
// variants (FP32, m ~ 3), where spread turns HBM-bound").
//
// Same operation as the float64 path ("Spreading", PAPER.md:57 Fig. 1, :162 §3):
//     g(l) = sum_j f_j prod_t Phi(n_t x_jt - l_t),   l in I_n (periodic),
// in float: complex64 values onto a complex64 grid.  Design: a CTA owns a BOX of cells -- BZ planes (whole sort chunks) x BY
// rows x BX columns (whole 8-column sort bins) -- accumulates the taps of the box's points into the
// box + halo tile of nodes in shared memory (one warp per point, lanes over the (2m)^3 taps), and
// adds the tile to the zeroed grid with one vector float2 reduction per nonzero node.  The box's
// points are the contiguous ranges of the chunk-major bin sort (sort.cu), one per (chunk, row).
// (On sm_100a a float atomicAdd to shared memory compiles to a compare-and-swap loop,
// ATOMS.CAST.SPIN, like the float64 one; the lanes of a warp update distinct nodes, so retries
// come only from other warps' points on the same node.  The global reduction of the tile is the
// native vector REDG.E.ADD.F32x2.)
// Tap weights: the plan's window polynomials (tables.cu) divided by Phi(0), evaluated in float
// (the float deconvolution tables carry the factor Phi(0) per dimension, api.cu).
#include <stdlib.h>

#include "spread_common.cuh"

namespace hpnfft {

namespace {

constexpr int kBoxThreads = 256;
constexpr int kBoxWarps = kBoxThreads / 32;

__host__ __device__ constexpr int align16(int bytes) { return (bytes + 15) & ~15; }

template <int M_>
__global__ void __launch_bounds__(kBoxThreads) k_spread_box_f32(
    const double* __restrict__ xs, const uint32_t* __restrict__ perm, const float2* __restrict__ f,
    const uint32_t* __restrict__ start, const double* __restrict__ poly_g, const double* __restrict__ wpeak,
    float2* __restrict__ grid, int n0, int n1, int n2, int nb2, int lc, int s2, int BZ, int BY, int BX, int nbz,
    int nby, int nbx, int lead) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  extern __shared__ __align__(16) unsigned char sm[];
  float* poly = reinterpret_cast<float*>(sm);                                        // [W][PD]
  float* scratch = reinterpret_cast<float*>(sm + align16(W * PD * 4));               // [warps][3 W]
  float2* tile = reinterpret_cast<float2*>(sm + align16(W * PD * 4) + align16(kBoxWarps * 3 * W * 4));
  const int TZ = BZ + W - 1, TY = BY + W - 1, TX = BX + W - 1;
  const int tile_n = TZ * TY * TX;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double inv_peak = 1.0 / *wpeak;   // taps in units of Phi(0) (the float tables carry Phi(0))
  for (int e = tid; e < W * PD; e += blockDim.x) poly[e] = (float)(poly_g[e] * inv_peak);
  float* ws = scratch + warp * 3 * W;
  const int CH = 1 << lc;
  const int nranges = (BZ / CH) * BY;
  const int nboxes = nbz * nby * nbx;
  for (int box = blockIdx.x; box < nboxes; box += gridDim.x) {
    for (int e = tid; e < tile_n; e += blockDim.x) tile[e] = make_float2(0.f, 0.f);
    __syncthreads();
    const int bx = box % nbx, by = (box / nbx) % nby, bz = box / (nbx * nby);
    const int Z0 = bz * BZ, Y0 = by * BY, X0 = bx * BX;
    for (int r = warp; r < nranges; r += kBoxWarps) {
      const int ch = Z0 / CH + r / BY, row = Y0 + r % BY;
      const size_t rowbase = ((size_t)ch * n1 + row) * nb2;
      const uint32_t beg = __ldg(start + (rowbase + (X0 >> s2)));
      const uint32_t end = __ldg(start + (rowbase + ((X0 + BX - 1) >> s2) + 1));
      for (uint32_t j = beg; j < end; ++j) {   // one warp per point
        const CellT a0 = cell_of(xs[3 * (size_t)j], n0), a1 = cell_of(xs[3 * (size_t)j + 1], n1),
                    a2 = cell_of(xs[3 * (size_t)j + 2], n2);
        // tap weights: lane q < 3W -> dimension q / W, tap q % W (strict truncation: the last
        // tap is 0 on a node; a trivial dimension of a d < 3 plan has the single tap m - 1)
        for (int q = lane; q < 3 * W; q += 32) {
          const int dd = q / W, i = q - dd * W;
          const float tt = (float)(dd == 0 ? a0.t : (dd == 1 ? a1.t : a2.t));
          float v;
          if (dd < lead) {
            v = i == M_ - 1 ? 1.f : 0.f;
          } else {
            const float s = fmaf(2.f, tt, -1.f);
            const float* cf = poly + i * PD;
            v = cf[PD - 1];
#pragma unroll
            for (int k = PD - 2; k >= 0; --k) v = fmaf(v, s, cf[k]);
            if (i == W - 1 && tt == 0.f) v = 0.f;
          }
          ws[q] = v;
        }
        __syncwarp();
        const float2 fv = __ldg(f + __ldg(perm + j));
        const int lz = a0.c - Z0, ly = a1.c - Y0, lx = a2.c - X0;   // cell inside the box
        for (int q = lane; q < W * W * W; q += 32) {
          const int i0 = q / (W * W), rem = q - i0 * W * W, i1 = rem / W, i2 = rem - i1 * W;
          const float w = ws[i0] * ws[W + i1] * ws[2 * W + i2];
          if (w != 0.f) {
            float2* node = tile + ((lz + i0) * TY + (ly + i1)) * TX + (lx + i2);
            atomicAdd(&node->x, fv.x * w);
            atomicAdd(&node->y, fv.y * w);
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // tile -> grid: node (tz, ty, tx) is grid node (Z0 - m + 1 + tz, ...) mod n
    for (int e = tid; e < tile_n; e += blockDim.x) {
      const float2 v = tile[e];
      if (v.x != 0.f || v.y != 0.f) {
        const int tz = e / (TY * TX), rem = e - tz * TY * TX, ty = rem / TX, tx = rem - ty * TX;
        const int gz = (Z0 - M_ + 1 + tz) & (n0 - 1), gy = (Y0 - M_ + 1 + ty) & (n1 - 1),
                  gx = (X0 - M_ + 1 + tx) & (n2 - 1);
        atomicAdd(grid + ((size_t)gz * n1 + gy) * n2 + gx, v);   // one vector float2 reduction
      }
    }
    __syncthreads();
  }
}

// The default FP32 spread: one warp per sorted point, lanes over the (i1, i2) taps, every tap one
// vector float2 reduction (REDG.E.ADD.F32x2) straight into the zeroed grid (the sort keeps
// consecutive points' footprints in the same L2 lines).  Measured at config 4 (1e7 points,
// 512^3): m = 2 / 3 / 6 spread 3.4 / 5.5 / 32 ms against 24 / 131 ms for the shared-memory box
// kernel above (HPNFFT_F32_SPREAD=box), whose float shared atomics are CAS loops on sm_100a.
template <int M_>
__global__ void __launch_bounds__(256) k_spread_red_f32(const double* __restrict__ xs, const uint32_t* __restrict__ perm,
                                                         const float2* __restrict__ f, const double* __restrict__ poly_g,
                                                         const double* __restrict__ wpeak, float2* __restrict__ grid,
                                                         int64_t M, int n0, int n1, int n2, int lead) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  __shared__ float poly[W * PD];
  __shared__ float wsm[8][3 * W];
  const double inv_peak = 1.0 / *wpeak;
  for (int e = threadIdx.x; e < W * PD; e += blockDim.x) poly[e] = (float)(poly_g[e] * inv_peak);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* ws = wsm[warp];
  for (int64_t j = (int64_t)blockIdx.x * 8 + warp; j < M; j += (int64_t)gridDim.x * 8) {
    const CellT a0 = cell_of(xs[3 * j], n0), a1 = cell_of(xs[3 * j + 1], n1), a2 = cell_of(xs[3 * j + 2], n2);
    for (int q = lane; q < 3 * W; q += 32) {
      const int dd = q / W, i = q - dd * W;
      const float tt = (float)(dd == 0 ? a0.t : (dd == 1 ? a1.t : a2.t));
      float v;
      if (dd < lead) {
        v = i == M_ - 1 ? 1.f : 0.f;
      } else {
        const float s = fmaf(2.f, tt, -1.f);
        const float* cf = poly + i * PD;
        v = cf[PD - 1];
#pragma unroll
        for (int k = PD - 2; k >= 0; --k) v = fmaf(v, s, cf[k]);
        if (i == W - 1 && tt == 0.f) v = 0.f;
      }
      ws[q] = v;
    }
    __syncwarp();
    const float2 fv = __ldg(f + __ldg(perm + j));
    for (int q = lane; q < W * W; q += 32) {
      const int i1 = q / W, i2 = q - i1 * W;
      const float w12 = ws[W + i1] * ws[2 * W + i2];
      const int l1 = (a1.c - M_ + 1 + i1) & (n1 - 1), l2 = (a2.c - M_ + 1 + i2) & (n2 - 1);
#pragma unroll
      for (int i0 = 0; i0 < W; ++i0) {
        const float w = ws[i0] * w12;
        if (w != 0.f) {
          const int l0 = (a0.c - M_ + 1 + i0) & (n0 - 1);
          atomicAdd(grid + ((size_t)l0 * n1 + l1) * n2 + l2, make_float2(fv.x * w, fv.y * w));
        }
      }
    }
    __syncwarp();
  }
}

template <int M_>
int launch_red(Plan* p, const float* f) {
  const int64_t blocks64 = (p->M + 7) / 8;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  const int64_t blocks = blocks64 < cap ? blocks64 : cap;
  k_spread_red_f32<M_><<<(unsigned)blocks, 256, 0, p->stream>>>(p->xs, p->perm, reinterpret_cast<const float2*>(f),
                                                                   p->poly, p->wpeak, reinterpret_cast<float2*>(p->grid),
                                                                   p->M, (int)p->n[0], (int)p->n[1], (int)p->n[2],
                                                                   3 - p->d);
  p->launches++;
  return check_launch(p, "spread red f32");
}

template <int M_>
int launch_box(Plan* p, const float* f) {
  constexpr int W = 2 * M_;
  const int n0 = (int)p->n[0], n1 = (int)p->n[1], n2 = (int)p->n[2];
  int s2 = 0;
  while ((1 << (s2 + 1)) <= 8 && (1 << (s2 + 1)) <= n2) ++s2;
  const int lc = p->chunk_log, CH = 1 << lc;
  // box: whole chunks (8 planes, at least one chunk), rows and whole sort bins of columns
  int BZ = n0 < 8 ? n0 : 8;
  if (BZ < CH) BZ = CH;
  const int BY = n1 < (W <= 8 ? 16 : 8) ? n1 : (W <= 8 ? 16 : 8);
  const int BX = n2 < (W <= 8 ? 64 : 32) ? n2 : (W <= 8 ? 64 : 32);
  const int TZ = BZ + W - 1, TY = BY + W - 1, TX = BX + W - 1;
  const size_t smem = (size_t)align16(W * (kPolyDeg + 1) * 4) + align16(kBoxWarps * 3 * W * 4) +
                      sizeof(float2) * (size_t)TZ * TY * TX;
  if (smem > 227 * 1024) {
    set_error("FP32 box spread: tile does not fit in shared memory");
    return HPNFFT_E_UNSUPPORTED;
  }
  auto kern = k_spread_box_f32<M_>;
  HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(kern), smem), "box smem attr");
  const int nbz = n0 / BZ, nby = n1 / BY, nbx = n2 / BX;
  const int64_t nboxes = (int64_t)nbz * nby * nbx;
  const int per_sm = smem <= 113 * 1024 ? 2 : 1;
  const int64_t slots = (int64_t)device_sm_count() * per_sm;
  const int64_t blocks = nboxes < slots ? nboxes : slots;
  kern<<<(unsigned)blocks, kBoxThreads, smem, p->stream>>>(
      p->xs, p->perm, reinterpret_cast<const float2*>(f), p->bin_count, p->poly, p->wpeak,
      reinterpret_cast<float2*>(p->grid), n0,
      n1, n2, n2 >> s2, lc, s2, BZ, BY, BX, nbz, nby, nbx, 3 - p->d);
  p->launches++;
  return check_launch(p, "spread box f32");
}

}  // namespace

int spread_f32(Plan* p, const float* f) {
  const size_t bytes = sizeof(float) * 2 * (size_t)(p->n[0] * p->n[1] * p->n[2]);
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->grid, 0, bytes, p->stream), "zero grid");
  if (p->M == 0) return HPNFFT_OK;
  const char* e = getenv("HPNFFT_F32_SPREAD");   // "box": the shared-memory box kernel (measured slower)
  if (!(e && e[0] == 'b')) {
    switch (p->m) {
      case 1: return launch_red<1>(p, f);
      case 2: return launch_red<2>(p, f);
      case 3: return launch_red<3>(p, f);
      case 4: return launch_red<4>(p, f);
      case 5: return launch_red<5>(p, f);
      case 6: return launch_red<6>(p, f);
      case 7: return launch_red<7>(p, f);
      case 8: return launch_red<8>(p, f);
      default: break;
    }
  }
  switch (p->m) {
    case 1: return launch_box<1>(p, f);
    case 2: return launch_box<2>(p, f);
    case 3: return launch_box<3>(p, f);
    case 4: return launch_box<4>(p, f);
    case 5: return launch_box<5>(p, f);
    case 6: return launch_box<6>(p, f);
    case 7: return launch_box<7>(p, f);
    case 8: return launch_box<8>(p, f);
    default:
      set_error("FP32 plans: m must be in [1, 8]");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
