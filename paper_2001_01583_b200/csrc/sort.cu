// sort.cu -- A1 (keys) + A2 (bin sort) of SURVEY.md §8(a): `hpnfft_set_points`.
//
// Not in the paper (its CUNFFT spreads points in input order, one thread per point,
// PAPER.md:162-164); the B200 design sorts the points once so the spread kernel can sweep
// the grid with register/tensor-core resident windows.
//   u_t = n_t x_t (exact for power-of-two n_t), c_t = floor(u_t) mod n_t  (integer cell)
//   key = ((c0 >> lc) * n1 + c1) * nb2 + (c2 >> s2),
//   CH = 2^lc planes per chunk, nb2 = n2 >> s2, s2 = log2(min(8, n2))
// so the points of one plane chunk and one c1 row are contiguous across consecutive c2 bins:
// a sweep CTA fetches the records of its (chunk, row) with one bulk copy.  The cell plane inside
// the chunk (c0 mod CH) is not part of the key: the sweep applies a chunk's records in any order
// (round 1 kept it in the key, four times the bins to zero and scan: 0.46 ms at n = 1024^3).
// Counting sort: histogram with arrival ranks (atomicAdd) -> exclusive scan -> scatter.
// The order inside a bin is the atomic arrival order (not deterministic; Q21).
#include <stdlib.h>

#include "common.cuh"

namespace hpnfft {

// coordinate t of point j: x is [M][d] with the d given dimensions last; the 3 - d leading
// (trivial) dimensions of a d < 3 plan read 0
// (x is float for the FP32 plans: the conversion to double is exact)
template <typename T>
__device__ __forceinline__ double coord(const T* __restrict__ x, int64_t j, int d, int t) {
  const int lead = 3 - d;
  return t < lead ? 0.0 : (double)x[(int64_t)d * j + (t - lead)];
}

__global__ void k_range_init(int* err) {
  const int t = threadIdx.x;
  if (t == 0) err[0] = 0;                                 // range-error flag
  else err[t] = (t & 1) ? 0x7fffffff : -1;                // slot minima / maxima
}

// bin key of point j (A1): cells c_t = floor(n_t x_t) mod n_t, chunk-major key; out-of-range
// coordinates (or NaN) set *err = 1 and count as the origin; keys outside [k_lo, k_hi) (a
// grid-slab rank's foreign planes) set *err = 2 and take k_lo
template <typename T>
__device__ __forceinline__ uint32_t point_key(const T* __restrict__ x, int64_t j, int d, int64_t n0, int64_t n1,
                                              int64_t n2, int s2, int lc, uint32_t k_lo, uint32_t k_hi,
                                              int* __restrict__ err, double* xo) {
  double x0 = coord(x, j, d, 0), x1 = coord(x, j, d, 1), x2 = coord(x, j, d, 2);
  if (!(fabs(x0) <= 0.5 && fabs(x1) <= 0.5 && fabs(x2) <= 0.5)) {
    *err = 1;   // benign race: any writer sets 1
    x0 = x1 = x2 = 0.0;
  }
  if (xo) {
    xo[0] = x0;
    xo[1] = x1;
    xo[2] = x2;
  }
  int64_t c0 = (int64_t)floor(__dmul_rn((double)n0, x0)) & (n0 - 1);
  int64_t c1 = (int64_t)floor(__dmul_rn((double)n1, x1)) & (n1 - 1);
  int64_t c2 = (int64_t)floor(__dmul_rn((double)n2, x2)) & (n2 - 1);
  int64_t nb2 = n2 >> s2;
  uint32_t k = (uint32_t)(((c0 >> lc) * n1 + c1) * nb2 + (c2 >> s2));
  if (k < k_lo || k >= k_hi) {   // grid-slab plan: the point is outside this rank's planes
    *err = 2;
    k = k_lo;
  }
  return k;
}

template <typename T>
__global__ void k_keys(const T* __restrict__ x, int d, int64_t M, int64_t n0, int64_t n1, int64_t n2, int s2, int lc,
                       uint32_t k_lo, uint32_t k_hi, uint32_t* __restrict__ count, uint32_t* __restrict__ key,
                       uint32_t* __restrict__ rank, int* __restrict__ err) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  // occupied range of the x-ordered plane index c0x = (c0 + n0/2) mod n0 (monotone in x0):
  // warp min/max, one atomic per warp
  unsigned cx = 0xffffffffu, cxm = 0u;
  if (j < M) {
    const int64_t c0 = (int64_t)floor(__dmul_rn((double)n0, coord(x, j, d, 0))) & (n0 - 1);
    cx = cxm = (unsigned)((c0 + n0 / 2) & (n0 - 1));
  }
  // block min/max, then one atomic pair per block into one of kRangeSlots slot pairs
  __shared__ unsigned s_min[8], s_max[8];
  const unsigned wmin = __reduce_min_sync(0xffffffffu, cx), wmax = __reduce_max_sync(0xffffffffu, cxm);
  if ((threadIdx.x & 31) == 0) {
    s_min[threadIdx.x >> 5] = wmin;
    s_max[threadIdx.x >> 5] = wmax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned bmin = 0xffffffffu, bmax = 0u;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      bmin = min(bmin, s_min[w]);
      bmax = max(bmax, s_max[w]);
    }
    if (bmin != 0xffffffffu) {
      const int slot = (int)(blockIdx.x % kRangeSlots);
      atomicMin(err + 1 + 2 * slot, (int)bmin);
      atomicMax(err + 2 + 2 * slot, (int)bmax);
    }
  }
  if (j >= M) return;
  const uint32_t k = point_key(x, j, d, n0, n1, n2, s2, lc, k_lo, k_hi, err, nullptr);
  key[j] = k;
  rank[j] = atomicAdd(&count[k], 1u);
}

// ---- two-level sort for large M (HPNFFT_SORT2; default from 2^25 points) -------------------
// Level 1 partitions the points by plane chunk (the key's top bits, C <= 1024 buckets): every
// block owns one contiguous slice of the input, counts its chunks in shared memory (K1), a scan
// of the chunk-major [C][blocks] counts gives every (chunk, block) a contiguous output run, and
// the block re-reads its slice and moves (key, index, coordinates) into its runs (K2).  Level 2
// is the counting sort of above on the chunk-ordered points: its count atomics, rank and output
// writes then stay inside one chunk's slice of the bin table / output at a time (L2-resident)
// instead of spreading random atomics over the whole table and random 24-byte reads over the
// whole input (what made the single-level sort ~8 % of HBM at 1e9 points).
constexpr int kSortBlocks = 1024;
constexpr int kSortThreads = 256;
constexpr int kMaxChunks = 1024;

template <typename T>
__global__ void __launch_bounds__(kSortThreads) k_keys_coarse(const T* __restrict__ x, int d, int64_t M, int64_t n0,
                                                              int64_t n1, int64_t n2, int s2, int lc, int fine_bits,
                                                              int C, uint32_t k_lo, uint32_t k_hi,
                                                              uint32_t* __restrict__ key, uint32_t* __restrict__ histT,
                                                              int* __restrict__ err) {
  __shared__ uint32_t hist[kMaxChunks];
  __shared__ unsigned s_min, s_max;
  for (int c = threadIdx.x; c < C; c += blockDim.x) hist[c] = 0u;
  if (threadIdx.x == 0) {
    s_min = 0xffffffffu;
    s_max = 0u;
  }
  __syncthreads();
  const int64_t per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(M, lo + per);
  unsigned bmin = 0xffffffffu, bmax = 0u;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
    const int64_t c0 = (int64_t)floor(__dmul_rn((double)n0, coord(x, j, d, 0))) & (n0 - 1);
    const unsigned cx = (unsigned)((c0 + n0 / 2) & (n0 - 1));
    bmin = min(bmin, cx);
    bmax = max(bmax, cx);
    const uint32_t k = point_key(x, j, d, n0, n1, n2, s2, lc, k_lo, k_hi, err, nullptr);
    key[j] = k;
    atomicAdd(&hist[k >> fine_bits], 1u);
  }
  atomicMin(&s_min, bmin);
  atomicMax(&s_max, bmax);
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) histT[(size_t)c * gridDim.x + blockIdx.x] = hist[c];
  if (threadIdx.x == 0 && s_min != 0xffffffffu) {   // occupied planes (see k_keys)
    const int slot = (int)(blockIdx.x % kRangeSlots);
    atomicMin(err + 1 + 2 * slot, (int)s_min);
    atomicMax(err + 2 + 2 * slot, (int)s_max);
  }
}

// K2: the block's slice in tiles of kTile points, each tile counting-sorted by chunk in shared
// memory first, so that the runs of one chunk leave the block as contiguous (coalesced) writes
constexpr int kTile = 1024;   // static shared memory < 48 KB

template <typename T>
__global__ void __launch_bounds__(kSortThreads) k_coarse_scatter(const T* __restrict__ x, int d, int64_t M,
                                                                 const uint32_t* __restrict__ key, int fine_bits, int C,
                                                                 const uint32_t* __restrict__ offT,
                                                                 uint32_t* __restrict__ tkey, uint32_t* __restrict__ tidx,
                                                                 double* __restrict__ tx) {
  __shared__ uint32_t cursor[kMaxChunks];   // next global position of every chunk (this block)
  __shared__ uint32_t lstart[kMaxChunks];   // tile: first local slot of every chunk
  __shared__ uint32_t lfill[kMaxChunks];    // tile: slots used so far
  __shared__ uint32_t skey[kTile], sidx[kTile];
  __shared__ double sx[kTile * 3];
  __shared__ uint32_t wsum[kSortThreads / 32];
  for (int c = threadIdx.x; c < C; c += blockDim.x) cursor[c] = offT[(size_t)c * gridDim.x + blockIdx.x];
  const int64_t per = (M + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(M, lo + per);
  constexpr int PT = kTile / kSortThreads;   // points per thread per tile
  for (int64_t t0 = lo; t0 < hi; t0 += kTile) {
    const int cnt = (int)min((int64_t)kTile, hi - t0);
    for (int c = threadIdx.x; c < C; c += blockDim.x) lfill[c] = 0u;
    __syncthreads();
    uint32_t kk[PT], rk[PT];
#pragma unroll
    for (int q = 0; q < PT; ++q) {
      const int i = threadIdx.x + q * kSortThreads;
      kk[q] = i < cnt ? key[t0 + i] : 0xffffffffu;
      rk[q] = i < cnt ? atomicAdd(&lfill[kk[q] >> fine_bits], 1u) : 0u;
    }
    __syncthreads();
    // exclusive scan of the tile's chunk counts (C <= 1024, kSortThreads threads, <= 4 per thread)
    {
      constexpr int CPT = kMaxChunks / kSortThreads;
      uint32_t v[CPT], sum = 0;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = threadIdx.x * CPT + q;
        v[q] = c < C ? lfill[c] : 0u;
        sum += v[q];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= o) incl += y;
      }
      if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = incl;
      __syncthreads();
      uint32_t wbase = 0;
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wbase += wsum[w];
      uint32_t run = wbase + incl - sum;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = threadIdx.x * CPT + q;
        if (c < C) lstart[c] = run;
        run += v[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PT; ++q) {
      const int i = threadIdx.x + q * kSortThreads;
      if (i < cnt) {
        const uint32_t slot = lstart[kk[q] >> fine_bits] + rk[q];
        const int64_t j = t0 + i;
        skey[slot] = kk[q];
        sidx[slot] = (uint32_t)j;
        sx[3 * slot] = coord(x, j, d, 0);
        sx[3 * slot + 1] = coord(x, j, d, 1);
        sx[3 * slot + 2] = coord(x, j, d, 2);
      }
    }
    __syncthreads();
    // slot s (chunk c) -> global cursor[c] + (s - lstart[c]): consecutive threads, consecutive addresses
    for (int sl = threadIdx.x; sl < cnt; sl += blockDim.x) {
      const uint32_t c = skey[sl] >> fine_bits;
      const uint32_t pos = cursor[c] + (uint32_t)sl - lstart[c];
      tkey[pos] = skey[sl];
      tidx[pos] = sidx[sl];
      tx[3 * (size_t)pos] = sx[3 * sl];
      tx[3 * (size_t)pos + 1] = sx[3 * sl + 1];
      tx[3 * (size_t)pos + 2] = sx[3 * sl + 2];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) cursor[c] += lfill[c];
    __syncthreads();
  }
}

__global__ void k_fine_count(const uint32_t* __restrict__ tkey, int64_t M, uint32_t* __restrict__ count,
                             uint32_t* __restrict__ rank) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < M) rank[i] = atomicAdd(&count[tkey[i]], 1u);
}

__global__ void k_fine_scatter(const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ tidx,
                               const double* __restrict__ tx, const uint32_t* __restrict__ rank,
                               const uint32_t* __restrict__ start, int64_t M, uint32_t* __restrict__ perm,
                               double* __restrict__ xs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const uint32_t pos = start[tkey[i]] + rank[i];
  perm[pos] = tidx[i];
  xs[3 * (size_t)pos] = tx[3 * (size_t)i];
  xs[3 * (size_t)pos + 1] = tx[3 * (size_t)i + 1];
  xs[3 * (size_t)pos + 2] = tx[3 * (size_t)i + 2];
}

// ---- device-wide exclusive scan of uint32 (three-phase, recursive over block sums) ----
// HPNFFT_SCAN_VEC=1: 256-thread tiles, 32 contiguous elements per thread moved as 8 uint4 (one
// 8-warp block scan per 8192 elements); 0: 1024 threads x 8 scalar elements (round 1).
#ifndef HPNFFT_SCAN_VEC
#define HPNFFT_SCAN_VEC 1
#endif
#if HPNFFT_SCAN_VEC
constexpr int kScanThreads = 256;
constexpr int kScanPerThread = 32;
#else
constexpr int kScanThreads = 1024;
constexpr int kScanPerThread = 8;
#endif
constexpr int kScanTile = kScanThreads * kScanPerThread;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[32];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0u;
    uint32_t si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += t;
    }
    warp_sums[lane] = si - s;   // exclusive warp offsets
    if (lane == 31) *total = si;
  }
  __syncthreads();
  uint32_t r = warp_sums[wid] + incl - v;
  __syncthreads();
  return r;
}

// scans each tile of kScanTile elements in place (exclusive), writes tile totals to sums
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(uint32_t* __restrict__ a, int64_t n,
                                                             uint32_t* __restrict__ sums) {
  __shared__ uint32_t total;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanPerThread;
  uint32_t v[kScanPerThread];
  uint32_t s = 0;
#if HPNFFT_SCAN_VEC
  // a is 16-byte aligned at every tile boundary when the caller's base is (bin_count + k_lo is
  // not in general): vector path only for full, aligned thread slices
  const bool vec = base + kScanPerThread <= n && ((reinterpret_cast<uintptr_t>(a + base) & 15) == 0);
  if (vec) {
    const uint4* a4 = reinterpret_cast<const uint4*>(a + base);
#pragma unroll
    for (int q = 0; q < kScanPerThread / 4; ++q) {
      const uint4 t = a4[q];
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanPerThread; ++q) v[q] = (base + q < n) ? a[base + q] : 0u;
  }
#pragma unroll
  for (int q = 0; q < kScanPerThread; ++q) s += v[q];
  uint32_t off = block_exclusive_scan(s, &total);
  if (vec) {
    uint4* a4 = reinterpret_cast<uint4*>(a + base);
#pragma unroll
    for (int q = 0; q < kScanPerThread / 4; ++q) {
      uint4 t;
      t.x = off; off += v[4 * q];
      t.y = off; off += v[4 * q + 1];
      t.z = off; off += v[4 * q + 2];
      t.w = off; off += v[4 * q + 3];
      a4[q] = t;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kScanPerThread; ++q) {
      if (base + q < n) a[base + q] = off;
      off += v[q];
    }
  }
#else
#pragma unroll
  for (int q = 0; q < kScanPerThread; ++q) {
    v[q] = (base + q < n) ? a[base + q] : 0u;
    s += v[q];
  }
  uint32_t off = block_exclusive_scan(s, &total);
#pragma unroll
  for (int q = 0; q < kScanPerThread; ++q) {
    if (base + q < n) a[base + q] = off;
    off += v[q];
  }
#endif
  if (threadIdx.x == 0 && sums) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_add(uint32_t* __restrict__ a, int64_t n,
                                                           const uint32_t* __restrict__ sums) {
  const uint32_t add = sums[blockIdx.x];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
#if HPNFFT_SCAN_VEC
  const int64_t head = (int64_t)((16 - (reinterpret_cast<uintptr_t>(a + t0) & 15)) & 15) / 4;   // to alignment
  const int64_t tile_n = n - t0 < kScanTile ? n - t0 : kScanTile;
  if (head == 0 && tile_n == kScanTile) {
    uint4* a4 = reinterpret_cast<uint4*>(a + t0);
#pragma unroll
    for (int q = 0; q < kScanPerThread / 4; ++q) {
      uint4 t = a4[q * kScanThreads + threadIdx.x];
      t.x += add; t.y += add; t.z += add; t.w += add;
      a4[q * kScanThreads + threadIdx.x] = t;
    }
    return;
  }
#endif
  for (int64_t e = t0 + threadIdx.x; e < t0 + kScanTile && e < n; e += kScanThreads) a[e] += add;
}
static int64_t scan_tmp_need(int64_t n) {
  int64_t need = 0;
  while (n > kScanTile) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    need += tiles;
    n = tiles;
  }
  return need + 1;
}

static int scan_exclusive(Plan* p, uint32_t* a, int64_t n, uint32_t* tmp) {
  int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if (tiles <= 1) {
    k_scan_tiles<<<1, kScanThreads, 0, p->stream>>>(a, n, nullptr);
    p->launches++;
    return check_launch(p, "scan");
  }
  k_scan_tiles<<<(unsigned)tiles, kScanThreads, 0, p->stream>>>(a, n, tmp);
  p->launches++;
  int rc = scan_exclusive(p, tmp, tiles, tmp + tiles);
  if (rc) return rc;
  k_scan_add<<<(unsigned)tiles, kScanThreads, 0, p->stream>>>(a, n, tmp);
  p->launches++;
  return check_launch(p, "scan add");
}

// scatter only the 4-byte permutation (random writes), then gather the coordinates in sorted
// order (random 24-byte reads, coalesced writes): scattered partial-sector writes of the
// coordinates would cost a DRAM read-modify-write each.
__global__ void k_scatter(int64_t M, const uint32_t* __restrict__ key, const uint32_t* __restrict__ rank,
                          const uint32_t* __restrict__ start, uint32_t* __restrict__ perm) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= M) return;
  uint32_t pos = start[key[j]] + rank[j];
  perm[pos] = (uint32_t)j;
}

template <typename T>
__global__ void k_gather_x(const T* __restrict__ x, int d, int64_t M, const uint32_t* __restrict__ perm,
                           double* __restrict__ xs) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= M) return;
  const int64_t j = perm[k];
  const double a = coord(x, j, d, 0), b = coord(x, j, d, 1), c = coord(x, j, d, 2);
  xs[3 * k] = a;
  xs[3 * k + 1] = b;
  xs[3 * k + 2] = c;
}

int64_t scan_workspace_elems(int64_t nbins) { return scan_tmp_need(nbins + 1); }

// Key range [k_lo, k_hi) this plan's points may use: all bins, or for a grid-slab rank only the
// bins of its own cell planes (one contiguous key range thanks to the chunk-major order).  Only
// that range is zeroed and scanned per set_points; the bins outside stay 0 (zeroed at plan
// time), so every lookup outside reads an empty range.
void key_range(const Plan* p, uint32_t& k_lo, uint32_t& k_hi) {
  int s2 = 0;
  while ((1 << (s2 + 1)) <= 8 && (1ll << (s2 + 1)) <= p->n[2]) ++s2;
  k_lo = 0;
  k_hi = (uint32_t)p->nbins;
  if (p->dist_mode == HPNFFT_DIST_GRID_SLAB && p->nranks > 1) {
    const int64_t n0 = p->n[0], lc = p->chunk_log, per_chunk = p->n[1] * (p->n[2] >> s2);
    const int64_t c0a = ((p->slab_lo + n0 / 2) % n0);   // first memory plane of the slab
    k_lo = (uint32_t)((c0a >> lc) * per_chunk);
    k_hi = (uint32_t)(((c0a + p->slab_len) >> lc) * per_chunk);
  }
}

// two-level sort workspace (lazy): chunk-ordered keys, indices, coordinates, the [C][blocks]
// counts and their scan's block sums
static int sort2_workspace(Plan* p, int64_t hist_n) {
  if (p->sort2_buf && p->sort2_hist_n >= hist_n) return HPNFFT_OK;
  cudaFree(p->sort2_buf);
  p->sort2_buf = nullptr;
  const size_t M = (size_t)(p->M > 0 ? p->M : 1);
  const size_t scan_n = (size_t)scan_tmp_need(hist_n);
  const size_t bytes = M * (4 + 4 + 24) + sizeof(uint32_t) * ((size_t)hist_n + scan_n) + 256;
  if (cudaMalloc(&p->sort2_buf, bytes) != cudaSuccess) {
    cudaGetLastError();
    p->sort2_buf = nullptr;
    return HPNFFT_E_NOMEM;
  }
  p->sort2_hist_n = hist_n;
  return HPNFFT_OK;
}

template <typename T>
static int sort_points_t(Plan* p, const T* x) {
  const int64_t M = p->M;
  int s2 = 0;
  while ((1 << (s2 + 1)) <= 8 && (1ll << (s2 + 1)) <= p->n[2]) ++s2;
  uint32_t k_lo, k_hi;
  key_range(p, k_lo, k_hi);
  const int lc = p->chunk_log;
  const int64_t C = p->n[0] >> lc;   // plane chunks = level-1 buckets
  int fine_bits = 0;   // key bits below the chunk
  while ((int64_t(1) << fine_bits) < p->n[1] * (p->n[2] >> s2)) ++fine_bits;
  const char* e2 = getenv("HPNFFT_SORT2");
  bool two = M >= (int64_t(1) << 25);
  if (e2) two = e2[0] == '1';
  two = two && M > 0 && C <= kMaxChunks && (int64_t(1) << fine_bits) == p->n[1] * (p->n[2] >> s2);
  const int64_t hist_n = C * kSortBlocks + 1;
  if (two && sort2_workspace(p, hist_n) != HPNFFT_OK) two = false;   // out of memory: one level
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->bin_count + k_lo, 0, sizeof(uint32_t) * ((size_t)(k_hi - k_lo) + 1), p->stream),
                  "memset bins");
  k_range_init<<<1, 2 * kRangeSlots + 1, 0, p->stream>>>(p->err_flag);
  p->launches++;
  if (two) {
    uint32_t* tkey = reinterpret_cast<uint32_t*>(p->sort2_buf);
    uint32_t* tidx = tkey + M;
    double* tx = reinterpret_cast<double*>(tidx + M);   // 8 M bytes in: 8-byte aligned
    uint32_t* histT = reinterpret_cast<uint32_t*>(tx + 3 * M);
    uint32_t* scan_tmp = histT + hist_n;
    stage_begin(p, 0);
    HPNFFT_CUDA_TRY(p, cudaMemsetAsync(histT + hist_n - 1, 0, sizeof(uint32_t), p->stream), "memset hist tail");
    k_keys_coarse<<<kSortBlocks, kSortThreads, 0, p->stream>>>(x, p->d, M, p->n[0], p->n[1], p->n[2], s2, lc,
                                                                fine_bits, (int)C, k_lo, k_hi, p->key, histT,
                                                                p->err_flag);
    p->launches++;
    int rc = check_launch(p, "keys (level 1)");
    if (rc) return rc;
    rc = scan_exclusive(p, histT, hist_n, scan_tmp);
    if (rc) return rc;
    k_coarse_scatter<<<kSortBlocks, kSortThreads, 0, p->stream>>>(x, p->d, M, p->key, fine_bits, (int)C, histT, tkey,
                                                                   tidx, tx);
    k_fine_count<<<(unsigned)((M + 255) / 256), 256, 0, p->stream>>>(tkey, M, p->bin_count, p->rank);
    p->launches += 2;
    rc = check_launch(p, "level-1 scatter / level-2 count");
    if (rc) return rc;
    stage_end(p, 0);
    stage_begin(p, 1);
    rc = scan_exclusive(p, p->bin_count + k_lo, (int64_t)(k_hi - k_lo) + 1, reinterpret_cast<uint32_t*>(p->scan_tmp));
    if (rc) return rc;
    stage_end(p, 1);
    stage_begin(p, 2);
    k_fine_scatter<<<(unsigned)((M + 255) / 256), 256, 0, p->stream>>>(tkey, tidx, tx, p->rank, p->bin_count, M, p->perm,
                                                                      p->xs);
    p->launches++;
    rc = check_launch(p, "level-2 scatter");
    if (rc) return rc;
    stage_end(p, 2);
    return HPNFFT_OK;
  }
  stage_begin(p, 0);
  if (M > 0) {
    k_keys<<<(unsigned)((M + 255) / 256), 256, 0, p->stream>>>(x, p->d, M, p->n[0], p->n[1], p->n[2], s2, p->chunk_log,
                                                               k_lo, k_hi, p->bin_count,
                                                               p->key, p->rank, p->err_flag);
    p->launches++;
    int rc = check_launch(p, "keys");
    if (rc) return rc;
  }
  stage_end(p, 0);
  stage_begin(p, 1);
  int rc = scan_exclusive(p, p->bin_count + k_lo, (int64_t)(k_hi - k_lo) + 1, reinterpret_cast<uint32_t*>(p->scan_tmp));
  if (rc) return rc;
  stage_end(p, 1);
  stage_begin(p, 2);
  if (M > 0) {
    k_scatter<<<(unsigned)((M + 255) / 256), 256, 0, p->stream>>>(M, p->key, p->rank, p->bin_count, p->perm);
    k_gather_x<<<(unsigned)((M + 255) / 256), 256, 0, p->stream>>>(x, p->d, M, p->perm, p->xs);
    p->launches += 2;
    rc = check_launch(p, "scatter");
    if (rc) return rc;
  }
  stage_end(p, 2);
  return HPNFFT_OK;
}

int sort_points(Plan* p, const double* x) { return sort_points_t(p, x); }
int sort_points_f32(Plan* p, const float* x) { return sort_points_t(p, x); }

}  // namespace hpnfft
