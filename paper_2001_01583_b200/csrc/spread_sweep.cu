// spread_sweep.cu -- the B200 spreading path (A3 + A4 of SURVEY.md §8(a)).
//
// Computes the "Spreading" step of CUNFFT (Fig. 1; §3)
//     g(l) = sum_j f_j * prod_t Phi(n_t x_jt - l_t),   l in I_n (periodic),
// without atomics and (for a single point group) without a zero fill: every grid node is
// written exactly once.
//
// Two kernels:
//  k_point_records  sorted point -> record in HBM (A3): cell (c1, c2, c0), f_j and the 3 x 2m
//                   tap weights from the window polynomials, in the shared-memory layout below.
//  k_spread_sweep   (A4) a persistent CTA owns a P1 x P2 patch of grid columns (l1, l2) and a
//                   segment of node planes l0; it sweeps the plane chunks (CH = 4 planes of cells
//                   for m <= 6) of the segment.  Consumer warps own 4 x 4 column sub-patches and
//                   keep the 16 node planes around the current chunk in FP64 tensor-core
//                   accumulators (DMMA m8n8k4): per k-step of 4 records
//                       C[node][col] += w0[record][node] * (f w1 w2)[record][col],
//                   i.e. the 2 (2m)^3 FMAs of a point run as rank-4 updates on the tensor core.
//                   A chunk's cells touch CH + 2m - 1 <= 16 node planes, so the records of a
//                   chunk can be applied in any order; after the chunk, the CH node planes no
//                   later chunk touches are stored (once, coalesced) and their rows zeroed.
// Record supply: sort.cu orders the points by (plane chunk, c1 row, c2 bin, c0), so the records a
// CTA needs for one chunk are one contiguous HBM range per candidate row (P1 + 2m - 1 rows).  A
// single producer warp looks the ranges up in the bin table and moves them into an NS-stage
// shared-memory ring with TMA bulk copies (cp.async.bulk, mbarrier transaction counts).
// When the records of all M points do not fit in the workspace, the sorted points are processed
// in groups ("the mass data have to be divided into several groups"): the grid is
// zeroed once and every group's sweep accumulates.
#include <stdio.h>
#include <stdlib.h>

#include "spread_common.cuh"

namespace hpnfft {

namespace {

#ifndef HPNFFT_SWEEP_WR
#define HPNFFT_SWEEP_WR 4
#endif
constexpr int kWR = HPNFFT_SWEEP_WR;   // warp sub-patch of the DMMA consumer: kWR rows (l1) x 4 cols (l2)
constexpr int kWC = 4;
constexpr int kBinW = 8;
// CTA patch shapes instantiated by the dispatch (run_sweep): the default (D) and the measurement
// variants; kWR = 2 (measurement builds) has 2x the sub-patches per patch, so its patches shrink
#if HPNFFT_SWEEP_WR == 4
#define HPNFFT_P_D1 8
#define HPNFFT_P_D2 32
#define HPNFFT_P_A1 12
#define HPNFFT_P_A2 32
#define HPNFFT_P_B1 16
#define HPNFFT_P_B2 16
#else
#define HPNFFT_P_D1 8
#define HPNFFT_P_D2 16
#define HPNFFT_P_A1 4
#define HPNFFT_P_A2 32
#define HPNFFT_P_B1 8
#define HPNFFT_P_B2 8
#endif        // c2 bin width of the sort keys (sort.cu)
#ifndef HPNFFT_SWEEP_NTSKIP
#define HPNFFT_SWEEP_NTSKIP 0   // skip n-tiles no record of a k-step reaches (measured: DESIGN.md)
#endif
#ifndef HPNFFT_SWEEP_PROFILE
#define HPNFFT_SWEEP_PROFILE 0  // measurement builds only: clock64 phase counters (HPNFFT_SWEEP_PROF=1)
#endif
constexpr bool kProf = HPNFFT_SWEEP_PROFILE != 0;
#ifndef HPNFFT_SWEEP_LEANFLUSH
#define HPNFFT_SWEEP_LEANFLUSH 1   // single-row-per-lane flush of short blocks (0: the generic loop)
#endif
#ifndef HPNFFT_SWEEP_DEBUG
#define HPNFFT_SWEEP_DEBUG 0    // measurement builds only: 1 = skip the MMAs, 2 = skip apply
#endif

// record layout in doubles (HBM and shared memory), no padding:
//   [0] c1|c2 (int2)  [1] c0|perm (int2: cell plane, original point index)  [2..3] f
//   [4 .. 4+W) w0   [4+W .. 4+2W) w1   [4+2W .. 4+3W) w2
// Operand lookups past a field (the DMMA A operand indexes w0 modulo 16 rows; w1/w2 indices
// outside the footprint) read the stage's zero record instead (tap_addr).
#ifndef HPNFFT_REC_PAD
#define HPNFFT_REC_PAD 3   // 3 = w0 zero-padded to 16 and w1/w2 + one zero (measured fastest)
#endif
template <int W>
struct Rec {
  static constexpr bool kPad0 = (HPNFFT_REC_PAD & 1) != 0, kPad12 = (HPNFFT_REC_PAD & 2) != 0;
  static constexpr int kW0 = 4;
  static constexpr int kW1 = 4 + (kPad0 ? 16 : W);
  static constexpr int kW2 = kW1 + W + (kPad12 ? 1 : 0);
  static constexpr int kEnd = kW2 + W + (kPad12 ? 1 : 0);
  static constexpr int kDoubles = (kEnd + 1) / 2 * 2;   // even -> 16-byte multiple
};

// shared-memory address of entry i of the record field starting at `off` (doubles), or of the
// zero record when i is outside the field (i >= W, incl. negative i wrapped to unsigned)
template <int W>
__device__ __forceinline__ uint32_t tap_addr(uint32_t rec_addr, int off, unsigned i, uint32_t zaddr) {
  return i < (unsigned)W ? rec_addr + 8u * ((unsigned)off + i) : zaddr;
}
// w0 lookup (cyclic row index i in [0, 16)) and w1 / w2 lookups, padded or via tap_addr
template <int W>
__device__ __forceinline__ uint32_t w0_addr(uint32_t ra, unsigned i, uint32_t zaddr) {
  if constexpr (Rec<W>::kPad0) return ra + 8u * (Rec<W>::kW0 + i);
  else return tap_addr<W>(ra, Rec<W>::kW0, i, zaddr);
}
template <int W>
__device__ __forceinline__ uint32_t w12_addr(uint32_t ra, int off, unsigned i, uint32_t zaddr) {
  if constexpr (Rec<W>::kPad12) return ra + 8u * ((unsigned)off + min(i, (unsigned)W));
  else return tap_addr<W>(ra, off, i, zaddr);
}

// plane chunk (cells per chunk) for a window half-width m: CH + 2m - 1 <= 16
template <int M_>
struct Chunk {
  static constexpr int CH = M_ <= 6 ? 4 : (M_ == 7 ? 2 : 1);
  static constexpr int LOG = M_ <= 6 ? 2 : (M_ == 7 ? 1 : 0);
  static_assert(CH + 2 * M_ - 1 <= 16, "chunk must fit the 16-row cyclic accumulator");
};

// Ring stages and list warps per sweep mode (measured): the list warp is the
// bottleneck of the one-chunk adjoint sweep with one list warp (consumers idle waiting for lists),
// so the dense adjoint and the inverse gather run three (one per ring stage), the merged-chunk
// (sparse) adjoint four stages with two.
#ifndef HPNFFT_SWEEP_NS
#define HPNFFT_SWEEP_NS 3
#endif
#ifndef HPNFFT_SWEEP_LISTW
#define HPNFFT_SWEEP_LISTW 3
#endif
#ifndef HPNFFT_SWEEP_NS_SPARSE
#define HPNFFT_SWEEP_NS_SPARSE 4
#endif
#ifndef HPNFFT_SWEEP_LISTW_SPARSE
#define HPNFFT_SWEEP_LISTW_SPARSE 2
#endif
#ifndef HPNFFT_SWEEP_NS_INV
#define HPNFFT_SWEEP_NS_INV 3
#endif
#ifndef HPNFFT_SWEEP_LISTW_INV
#define HPNFFT_SWEEP_LISTW_INV 3
#endif
enum SweepMode { kDense = 0, kSparse = 1, kInverse = 2 };
__host__ __device__ constexpr int sweep_mode(bool inv, bool merge) { return inv ? kInverse : (merge ? kSparse : kDense); }

template <int P1, int P2, int M_, int MODE = kDense>
struct SweepCfg {
  static constexpr int W = 2 * M_;                         // taps per dimension
  static constexpr int NL = (P1 / kWR) * (P2 / kWC);       // 4 x 4 sub-patches (= record lists)
#ifndef HPNFFT_SWEEP_SUB
#define HPNFFT_SWEEP_SUB 1
#endif
  static constexpr int SUB = HPNFFT_SWEEP_SUB;             // sub-patches per consumer warp
  static_assert(NL % SUB == 0, "whole sub-patches per warp");
  static constexpr int NW = NL / SUB;                      // consumer warps
  static constexpr int NS = MODE == kSparse ? HPNFFT_SWEEP_NS_SPARSE
                           : MODE == kInverse ? HPNFFT_SWEEP_NS_INV : HPNFFT_SWEEP_NS;   // ring stages
  // list warps: warp i owns ring stages i, i + kListWarps, ... (so that it waits on every phase of
  // its stages' barriers in order; a parity wait must never skip a phase)
  static constexpr int kListWarps = MODE == kSparse ? HPNFFT_SWEEP_LISTW_SPARSE
                                    : MODE == kInverse ? HPNFFT_SWEEP_LISTW_INV : HPNFFT_SWEEP_LISTW;
  static_assert(NS % kListWarps == 0, "a list warp owns whole ring stages");
  static constexpr int kThreads = (NW + 1 + kListWarps) * 32;   // + copy warp + list warps
  static constexpr int kRows = P1 + W - 1;                 // candidate c1 rows
  static constexpr int kCtasPerSm = NL <= 8 ? 2 : 1;        // small patches: 2 resident CTAs
  // the whole register file for the resident warps (multiple of 8 per thread, <= 255)
  // (registers are granted to warps in groups of 4)
  static constexpr int kMaxRegs0 = (65536 / ((NW + 1 + kListWarps + 3) / 4 * 4 * 32 * kCtasPerSm)) / 8 * 8;
  static constexpr int kMaxRegs = kMaxRegs0 > 248 ? 248 : kMaxRegs0;
  static_assert(kRows <= 32, "one producer lane per candidate row");
};

struct SweepParams {
  const double* rec;       // point records of the group (record r = sorted point g0 + r)
  const uint32_t* start;   // bin_start [nbins + 1]
  double* grid;            // [n0][n1][n2] complex
  const int* chunks;       // [2] plane chunks spanned by the group (multi-group pass only)
  uint32_t g0, g1;         // sorted point range of this group
  int accumulate;          // 1: grid += window (multi-group), 0: grid = window
  int n0, n1, n2;
  int nb2;                 // n2 / 8
  int seg;                 // S: node planes per segment (multiple of CH)
  int nseg;                // segments covering the occupied node planes
  int plane_lo, plane_len; // occupied node planes, aligned to CH (circular interval)
  int cap;                 // record capacity of one shared-memory ring stage
  int* tile_counter;       // dynamic tile scheduler (zeroed before the launch)
  unsigned long long* prof;   // optional clock64 phase counters (HPNFFT_SWEEP_PROF=1), else null
  double* fout;            // inverse direction: f [M][2] in original point order (atomically summed)
  const int* order;        // tile processing order (largest record count first), or null
};

}  // namespace

// ------------------------------------------------------------------------------------------
// A3: point records, one thread per sorted point (128 points per CTA): the 3 x 2m Horner chains
// of a tap share the tap's coefficients (a broadcast shared-memory load per step); the records
// are staged in shared memory and written to HBM with coalesced 16-byte stores.
constexpr int kRecPts = 128;
#ifndef HPNFFT_REC_CHUNKS
#define HPNFFT_REC_CHUNKS 4   // runs of kRecPts points per CTA (measured: 1 / 4 -> 1.12 / 1.02 ms at config 4)
#endif
#ifndef HPNFFT_REC_UNROLL
#define HPNFFT_REC_UNROLL 2   // taps evaluated together (independent Horner chains: 3 per tap)
#endif
constexpr int kRecUnroll = HPNFFT_REC_UNROLL;

template <int M_>
__global__ void __launch_bounds__(kRecPts) k_point_records(const double* __restrict__ xs, const uint32_t* __restrict__ perm,
                                                            const double* __restrict__ f, const double* __restrict__ poly_g,
                                                            double* __restrict__ rec, uint32_t g0, uint32_t count,
                                                            int64_t n0, int64_t n1, int64_t n2) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  using R = Rec<W>;
  constexpr int RD = R::kDoubles;
  __shared__ double poly[W * PD];
  extern __shared__ __align__(16) double stage[];   // [kRecPts][RD]
  for (int e = threadIdx.x; e < W * PD; e += blockDim.x) poly[e] = poly_g[e];
  // a CTA builds HPNFFT_REC_CHUNKS consecutive runs of kRecPts points (the table load amortised)
  for (uint32_t kb = blockIdx.x * kRecPts * HPNFFT_REC_CHUNKS; kb < count && kb < (blockIdx.x + 1) * kRecPts * HPNFFT_REC_CHUNKS;
       kb += kRecPts) {
  const uint32_t k = kb + threadIdx.x;
  double2 fv = make_double2(0.0, 0.0);
  double x0 = 0.0, x1 = 0.0, x2 = 0.0;
  if (k < count) {
    const size_t src = (size_t)g0 + k;
    if (f) fv = __ldg(reinterpret_cast<const double2*>(f) + __ldg(perm + src));   // null: inverse
    x0 = __ldg(xs + 3 * src);
    x1 = __ldg(xs + 3 * src + 1);
    x2 = __ldg(xs + 3 * src + 2);
  }
  __syncthreads();
  double* out = stage + threadIdx.x * RD;
  const CellT a0 = cell_of(x0, n0), a1 = cell_of(x1, n1), a2 = cell_of(x2, n2);
  const double s0 = fma(2.0, a0.t, -1.0), s1 = fma(2.0, a1.t, -1.0), s2 = fma(2.0, a2.t, -1.0);
#pragma unroll kRecUnroll
  for (int i = 0; i < W; ++i) {
    const double* cf = poly + i * PD;
    double v0 = cf[PD - 1], v1 = v0, v2 = v0;
#pragma unroll
    for (int j = PD - 2; j >= 0; --j) {
      const double c = cf[j];
      v0 = fma(v0, s0, c);
      v1 = fma(v1, s1, c);
      v2 = fma(v2, s2, c);
    }
    if (i == W - 1) {   // strict truncation |u - l| < m (Q4)
      if (a0.t == 0.0) v0 = 0.0;
      if (a1.t == 0.0) v1 = 0.0;
      if (a2.t == 0.0) v2 = 0.0;
    }
    out[R::kW0 + i] = v0;
    out[R::kW1 + i] = v1;
    out[R::kW2 + i] = v2;
  }
  if constexpr (R::kPad0) {
#pragma unroll
    for (int i = W; i < 16; ++i) out[R::kW0 + i] = 0.0;
  }
  if constexpr (R::kPad12) {
    out[R::kW1 + W] = 0.0;
    out[R::kW2 + W] = 0.0;
  }
  reinterpret_cast<int4*>(out)[0] = make_int4(a1.c, a2.c, a0.c, (int)(k < count ? perm[(size_t)g0 + k] : 0u));
  reinterpret_cast<double2*>(out)[1] = fv;
  __syncthreads();
  const uint32_t npts = min((uint32_t)kRecPts, count - kb);
  const int nchunk = (int)npts * (RD / 2);
  const double2* sp = reinterpret_cast<const double2*>(stage);
  double2* gp = reinterpret_cast<double2*>(rec + (size_t)kb * RD);
  for (int c = threadIdx.x; c < nchunk; c += blockDim.x) gp[c] = sp[c];
  }
}

// plane chunks spanned by sorted points [g0, g1): binary search of the bin table (multi-group).
// Only bins [k_lo, k_hi] are non-decreasing: a grid-slab rank zeroes and scans its own key range
// (sort.cu key_range) and every bin outside reads 0, so the search is confined to that range.
__global__ void k_group_chunks(const uint32_t* __restrict__ start, int64_t k_lo, int64_t k_hi, uint32_t g0,
                               uint32_t g1, int64_t bins_per_chunk, int* chunks) {
  const int which = threadIdx.x;   // 0: first point, 1: last point
  if (which > 1) return;
  const uint32_t target = which == 0 ? g0 : g1 - 1;
  int64_t lo = k_lo, hi = k_hi - 1;   // largest bin in [k_lo, k_hi) with start[bin] <= target
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (start[mid] <= target) lo = mid;
    else hi = mid - 1;
  }
  chunks[which] = (int)(lo / bins_per_chunk);
}

// ------------------------------------------------------------------------------------------
// shared-memory and barrier helpers
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
// try_wait with a suspend-time hint so waiting warps sleep instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ok = 0;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
#if HPNFFT_CHECKED
  const long long t0 = clock64();
#endif
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000)
        : "memory");
#if HPNFFT_CHECKED
    HPNFFT_DCHECK(clock64() - t0 < (1ll << 35));   // ~17 s at 2 GHz: a lost arrival (deadlock)
#endif
  }
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_copy_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(smem)),
      "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
// 4-byte asynchronous global -> shared copies (the producer's bin-bound prefetch ring)
__device__ __forceinline__ void cp_async4(uint32_t* smem, const uint32_t* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
// D = A (16x4, row) x B (4x8, col) + D on the FP64 tensor core.  Lane (g = lane/4, t = lane%4):
// a0 = A[g][t], a1 = A[g+8][t], b = B[t][g], c = {D[g][2t], D[g][2t+1], D[g+8][2t], D[g+8][2t+1]}
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b));
}

// A batch holds the records of one chunk or, at low point density, of up to kMaxSeg chunks
// (segments; records in chunk order), so that sparse inputs do not pay one pipeline round trip
// per chunk of a handful of records.
#ifndef HPNFFT_MAX_SEG
#define HPNFFT_MAX_SEG 16
#endif
constexpr int kMaxSeg = HPNFFT_MAX_SEG;
struct BatchHdr {
  int B;      // records in the batch; -1 terminates
  int tile;   // tile id
  int chunk;  // chunk index within the tile of the first segment (step = chunk * CH + (c0 mod CH))
  int end;    // 1: end of tile (flush the rest), 2: tile skipped in this group pass
  int nseg;   // segments: records [seg_end[j-1], seg_end[j]) belong to chunk `chunk + seg_dch[j]`
  int16_t seg_end[kMaxSeg];
  uint8_t seg_dch[kMaxSeg];
};
// list capacity: every list of a multi-segment batch is padded to whole k-steps per segment
__host__ __device__ constexpr int list_cap(int cap, bool merge) { return merge ? cap + 3 * kMaxSeg : cap; }

__host__ __device__ __forceinline__ int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// chunks whose bin bounds the producer has in flight (cp.async ring): at low point density most
// chunks are empty and the producer would otherwise wait one global-load latency per chunk
constexpr int kBinPrefetch = 8;

template <int P1, int P2, int M_, int MODE>
__host__ __device__ constexpr size_t sweep_smem_bytes_of(int cap, bool merge) {
  using C = SweepCfg<P1, P2, M_, MODE>;
  return sizeof(double) * ((size_t)C::NS * cap * Rec<2 * M_>::kDoubles + Rec<2 * M_>::kDoubles) +
         (sizeof(uint64_t) * 3 + sizeof(BatchHdr)) * C::NS + sizeof(uint32_t) * (size_t)C::NS * C::NL * (list_cap(cap, merge) + 1) +
         sizeof(uint32_t) * kBinPrefetch * 32 * 4 + 32;
}

// ------------------------------------------------------------------------------------------
// A4: the warp-specialised persistent sweep (see the file header).
// REAL (the ENUF charges): real values f_j = q_j onto a REAL grid
// [n0][n1][n2] (doubles; the R2C z pass reads it as n2/2 complex per line): an n-tile is then 8
// real columns = 2 rows x 4 columns of the 4 x 4 sub-patch, half the DMMAs of the complex sweep.
template <int P1, int P2, int M_, bool INV, bool MERGE, bool REAL = false>
__global__ void __launch_bounds__(SweepCfg<P1, P2, M_, sweep_mode(INV, MERGE)>::kThreads)
    __maxnreg__((SweepCfg<P1, P2, M_, sweep_mode(INV, MERGE)>::kMaxRegs)) k_spread_sweep(SweepParams prm) {
  using C = SweepCfg<P1, P2, M_, sweep_mode(INV, MERGE)>;
  using R = Rec<2 * M_>;
  constexpr int W = C::W, NW = C::NW, NS = C::NS, NL = C::NL, SUB = C::SUB;
  constexpr int RD = R::kDoubles;
  constexpr int CH = Chunk<M_>::CH;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int cap = prm.cap;
  double* s_rec = reinterpret_cast<double*>(smem_raw);                            // [NS][cap][RD]
  double* s_zero = s_rec + (size_t)NS * cap * RD;                                 // [RD] zeros
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_zero + RD);                    // [NS] lists ready
  uint64_t* s_empty = s_full + NS;                                                // [NS] stage free
  uint64_t* s_landed = s_empty + NS;                                              // [NS] records landed
  BatchHdr* s_hdr = reinterpret_cast<BatchHdr*>(s_landed + NS);                   // [NS]
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_hdr + NS);                      // [NS][NL]
  // multi-chunk batches (MERGE, chosen for sparse inputs): adjoint consumers with one sub-patch
  // per warp only (the inverse consumer loads its grid window per chunk, two interleaved
  // sub-patches share one flush front)
  constexpr bool kMerge = MERGE && !INV && SUB == 1;
  const int capL = list_cap(cap, kMerge);
  uint32_t* s_list = s_cnt + NS * NL;                                             // [NS][NL][capL]
  uint32_t* s_pf = reinterpret_cast<uint32_t*>(                                   // [kBinPrefetch][32][4]
      (reinterpret_cast<uintptr_t>(s_list + (size_t)NS * NL * capL) + 15) & ~(uintptr_t)15);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = prm.n0, n1 = prm.n1, n2 = prm.n2;
  const int nchunks0 = n0 / CH;   // plane chunks around the circle
  const int npc = n2 / P2, npr = (n1 + P1 - 1) / P1;
  (void)C::kRows;
  const int ntiles = npc * npr * prm.nseg;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_landed[i], 1);
      mbar_init(&s_empty[i], NW);
    }
  }
  for (int i = tid; i < RD; i += blockDim.x) s_zero[i] = 0.0;
  __syncthreads();

  // tile t = (segment, patch row, patch col); node planes [L0, L0 + S); chunks a_lo .. a_lo + nch - 1
  // (absolute chunk index, may be negative: taken mod n0 / CH) hold every cell that reaches them.
  auto tile_geom = [&](int t, int& R0, int& C0, int& L0, int& S, int& a_lo, int& nch) {
    const int pc = t % npc;
    const int rest = t / npc;
    const int pr = rest % npr;
    const int segi = rest / npr;
    R0 = pr * P1;
    C0 = pc * P2;
    L0 = prm.plane_lo + segi * prm.seg;
    S = min(prm.seg, prm.plane_len - segi * prm.seg);
    a_lo = floor_div(L0 - M_, CH);
    nch = floor_div(L0 + S + M_ - 2, CH) - a_lo + 1;
  };

  if (warp == NW) {
    // =============================== producer warp ===============================
    int stage = 0;
    uint32_t phase = 0;
    auto next_stage = [&]() {
      if (++stage == NS) {
        stage = 0;
        phase ^= 1u;
      }
    };
    for (;;) {
      int t = 0;
      if (lane == 0) t = atomicAdd(prm.tile_counter, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= ntiles) break;
      if (prm.order) t = __ldg(prm.order + t);   // heaviest tiles first (clustered inputs)
      int R0, C0, L0, S, a_lo, nch;
      tile_geom(t, R0, C0, L0, S, a_lo, nch);
      bool skip = false;
      if (prm.accumulate) {   // multi-group pass: the group's chunks miss the tile
        const int clo = prm.chunks[0], chi = prm.chunks[1];
        bool hit = false;
        for (int sft = -nchunks0; sft <= nchunks0; sft += nchunks0)
          hit |= !(a_lo + nch - 1 + sft < clo || a_lo + sft > chi);
        skip = !hit;
      }
      if (!skip) {
        // this lane's candidate row and its c2 bin runs (at most 2 when the bins wrap around n2)
        const int r = lane;
        const int c1 = (R0 - M_ + r) & (n1 - 1);
        const int b2lo = floor_div(C0 - M_, kBinW);
        const int b2hi = (C0 + P2 + M_ - 2) / kBinW;
        int ra0 = b2lo, rb0 = b2hi, ra1 = 0, rb1 = -1;   // bin runs [ra, rb]
        if (b2lo < 0) {
          ra0 = 0;
          ra1 = b2lo + prm.nb2;
          rb1 = prm.nb2 - 1;
        } else if (b2hi >= prm.nb2) {
          rb0 = prm.nb2 - 1;
          ra1 = 0;
          rb1 = b2hi - prm.nb2;
        }
        // bin bounds of chunk ci (lo0, hi0, lo1, hi1 of this lane's row) -> ring slot ci mod PF
        auto prefetch = [&](int ci) {
          uint32_t* d = s_pf + ((ci % kBinPrefetch) * 32 + lane) * 4;
          if (ci < nch && r < C::kRows) {
            int a = a_lo + ci;   // chunk index mod nchunks0 (no integer division on the producer's path)
            while (a < 0) a += nchunks0;
            while (a >= nchunks0) a -= nchunks0;
            const size_t rowbase = ((size_t)a * n1 + c1) * prm.nb2;
            cp_async4(d + 0, prm.start + (rowbase + ra0));
            cp_async4(d + 1, prm.start + (rowbase + rb0 + 1));
            if (rb1 >= ra1) {
              cp_async4(d + 2, prm.start + (rowbase + ra1));
              cp_async4(d + 3, prm.start + (rowbase + rb1 + 1));
            } else {
              d[2] = d[3] = 0u;
            }
          } else {
            d[0] = d[1] = d[2] = d[3] = 0u;
          }
          cp_async_commit();
        };
#pragma unroll 1
        for (int u = 0; u < kBinPrefetch; ++u) prefetch(u);
        // the open batch: oB records of onseg segments so far, first chunk och0
        bool open = false;
        int oB = 0, onseg = 0, och0 = 0;
        auto close_batch = [&]() {
          if (!open) return;
          if (lane == 0) {
            BatchHdr& h = s_hdr[stage];
            h.B = oB;
            h.tile = t;
            h.chunk = och0;
            h.end = 0;
            h.nseg = onseg;
            mbar_arrive(&s_landed[stage]);
          }
          open = false;
          next_stage();
        };
        for (int ci = 0; ci < nch; ++ci) {
          const unsigned long long p0 = kProf ? clock64() : 0ull;
          uint32_t beg0 = 0, len0 = 0, beg1 = 0, len1 = 0;
          cp_async_wait<kBinPrefetch - 1>();   // chunk ci's group has landed (one group per chunk)
          {
            const uint4 v = *reinterpret_cast<const uint4*>(s_pf + ((ci % kBinPrefetch) * 32 + lane) * 4);
            const uint32_t lo0 = v.x, hi0 = v.y, lo1 = v.z, hi1 = v.w;
            // clip to the group, make group-relative
            const uint32_t l0c = max(lo0, prm.g0), h0c = min(hi0, prm.g1);
            const uint32_t l1c = max(lo1, prm.g0), h1c = min(hi1, prm.g1);
            beg0 = l0c - prm.g0;
            len0 = h0c > l0c ? h0c - l0c : 0u;
            beg1 = l1c - prm.g0;
            len1 = h1c > l1c ? h1c - l1c : 0u;
          }
          prefetch(ci + kBinPrefetch);   // (after this slot's values are in registers)
          // chunk offsets: exclusive warp scan of the lane totals
          const uint32_t cnt = len0 + len1;
          uint32_t incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
          }
          const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
          const uint32_t off0 = incl - cnt, off1 = off0 + len0;
          if (kProf && lane == 0) atomicAdd(prm.prof + 4, clock64() - p0);
          if (total == 0) continue;
          if (open && (oB + (int)total > cap || onseg == kMaxSeg || ci - och0 > 127)) close_batch();
          for (uint32_t b0 = 0; b0 < total;) {
            const unsigned long long p1 = kProf ? clock64() : 0ull;
            if (!open) {
              mbar_wait(&s_empty[stage], phase ^ 1u);
              open = true;
              oB = 0;
              onseg = 0;
              och0 = ci;
            }
            const unsigned long long p2 = kProf ? clock64() : 0ull;
            const uint32_t b1 = min(total, b0 + (uint32_t)(cap - oB));
            const int take = (int)(b1 - b0);
            HPNFFT_DCHECK(take > 0 && oB + take <= cap && onseg < kMaxSeg);
            if (lane == 0) mbar_expect_tx(&s_landed[stage], (uint32_t)take * (uint32_t)(RD * sizeof(double)));
            __syncwarp();
            double* dst = s_rec + ((size_t)stage * cap + oB) * RD;
            // the part of each run inside [b0, b1) -> consecutive ring slots, one bulk copy
            auto issue = [&](uint32_t off, uint32_t beg, uint32_t len) {
              if (len == 0 || off >= b1 || off + len <= b0) return;
              const uint32_t k0 = off < b0 ? b0 - off : 0u;
              const uint32_t k1 = min(len, b1 - off);
              HPNFFT_DCHECK(beg + k1 <= prm.g1 - prm.g0);                    // inside the group's records
              HPNFFT_DCHECK((uint32_t)oB + (off + k1 - b0) <= (uint32_t)cap);   // inside the stage
              bulk_copy_g2s(dst + (size_t)(off + k0 - b0) * RD, prm.rec + (size_t)(beg + k0) * RD,
                            (k1 - k0) * (uint32_t)(RD * sizeof(double)), &s_landed[stage]);
            };
            issue(off0, beg0, len0);
            issue(off1, beg1, len1);
            oB += take;
            if (lane == 0) {
              s_hdr[stage].seg_end[onseg] = (int16_t)oB;
              s_hdr[stage].seg_dch[onseg] = (uint8_t)(ci - och0);
            }
            ++onseg;
            b0 = b1;
            if (kProf && lane == 0) {
              atomicAdd(prm.prof + 5, p2 - p1);
              atomicAdd(prm.prof + 6, clock64() - p2);
            }
            if (!kMerge || oB == cap) close_batch();
          }
        }
        close_batch();
      }
      // end-of-tile marker (consumers flush every remaining node of the tile unless it is skipped)
      mbar_wait(&s_empty[stage], phase ^ 1u);
      if (lane == 0) {
        s_hdr[stage].B = 0;
        s_hdr[stage].tile = t;
        s_hdr[stage].chunk = skip ? 0 : nch;
        s_hdr[stage].end = skip ? 2 : 1;
        s_hdr[stage].nseg = 0;
        mbar_arrive(&s_landed[stage]);
      }
      next_stage();
    }
    // one terminal marker per list warp (the consumers stop at the first)
    for (int i = 0; i < C::kListWarps; ++i) {
      mbar_wait(&s_empty[stage], phase ^ 1u);
      if (lane == 0) {
        s_hdr[stage].B = -1;
        s_hdr[stage].tile = -1;
        s_hdr[stage].chunk = 0;
        s_hdr[stage].end = 0;
        s_hdr[stage].nseg = 0;
        mbar_arrive(&s_landed[stage]);
      }
      next_stage();
    }
    return;
  }

  if (warp > NW) {
    // ============================ list warps ============================
    // Once a stage's records have landed, sort them into one list per consumer warp: the records
    // whose 2m x 2m column footprint meets the warp's 4 x 4 sub-patch, entry = record | (c0 mod
    // CH) << 9 | d1 << 18 | d2 << 23 with d1 = (warp row) - (c1 - m + 1) + 3 < 2m + 3 and
    // d2 = (warp col) - (c2 - m + 1) + 3 < 2m + 3.  (Each consumer warp scanning the whole batch
    // itself would keep the FP64 tensor pipe idle while all of them do it at the same time.)
    // List warp i takes batches i, i + kListWarps, ... of the ring (= stages it owns).
    constexpr int NWC = P2 / kWC;   // consumer warps per sub-patch row
    for (uint32_t seq = (uint32_t)(warp - NW - 1);; seq += C::kListWarps) {
      const int stage = (int)(seq % NS);
      const uint32_t phase = (seq / NS) & 1u;
      const unsigned long long l0c = kProf ? clock64() : 0ull;
      mbar_wait(&s_landed[stage], phase);
      const unsigned long long l1c = kProf ? clock64() : 0ull;
      const BatchHdr hdr = s_hdr[stage];
      HPNFFT_DCHECK(hdr.B <= cap && (hdr.B < 0 || hdr.tile >= 0) && (!kMerge || hdr.nseg <= kMaxSeg));
      int cnt[NL];   // list lengths (0 for tile-end markers)
#pragma unroll
      for (int w = 0; w < NL; ++w) cnt[w] = 0;
      if (hdr.B > 0) {
        int R0, C0, L0, S_, a_lo, nch;
        tile_geom(hdr.tile, R0, C0, L0, S_, a_lo, nch);
        const double* recs = s_rec + (size_t)stage * cap * RD;
        uint32_t* lists = s_list + (size_t)stage * NL * capL;
        // entry = record | (c0 mod CH) << 9 | segment chunk offset << 11 | d1 << 18 | d2 << 23
        // (single-chunk batches: one segment [0, B), offset 0)
        const int nseg = kMerge ? hdr.nseg : 1;
        for (int j = 0; j < nseg; ++j) {
          const int sb = (kMerge && j) ? (int)s_hdr[stage].seg_end[j - 1] : 0;
          const int se = kMerge ? (int)s_hdr[stage].seg_end[j] : hdr.B;
          const uint32_t dch = kMerge ? (uint32_t)s_hdr[stage].seg_dch[j] << 11 : 0u;
          for (int base = sb; base < se; base += 32) {
            const int e = base + lane;
            int dr = -1000, dc = -1000;   // footprint origin relative to the patch origin
            uint32_t ebase = 0;
            if (e < se) {
              const int4 cc = *reinterpret_cast<const int4*>(recs + (size_t)e * RD);
              dr = ((cc.x - M_ + 1 - R0 + W) & (n1 - 1)) - W;
              dc = ((cc.y - M_ + 1 - C0 + W) & (n2 - 1)) - W;
              ebase = (uint32_t)e | ((uint32_t)(cc.z & (CH - 1)) << 9) | dch;
            }
#pragma unroll
            for (int wr = 0; wr < P1 / kWR; ++wr) {
              const uint32_t d1 = (uint32_t)(kWR * wr - dr + (kWR - 1));
              const bool relr = d1 < (uint32_t)(W + kWR - 1);
#pragma unroll
              for (int wc = 0; wc < NWC; ++wc) {
                const uint32_t d2 = (uint32_t)(kWC * wc - dc + (kWC - 1));
                const bool rel = relr && d2 < (uint32_t)(W + kWC - 1);
                const unsigned bal = __ballot_sync(0xffffffffu, rel);
                const int w = wr * NWC + wc;
                if (rel) {
                  HPNFFT_DCHECK(cnt[w] + __popc(bal & ((1u << lane) - 1)) < capL && e < cap);
                  lists[(size_t)w * capL + cnt[w] + __popc(bal & ((1u << lane) - 1))] = ebase | (d1 << 18) | (d2 << 23);
                }
                cnt[w] += __popc(bal);
              }
            }
          }
          if (kMerge && nseg > 1) {
            // pad every list to whole k-steps (4 entries) with null records (index 0x1ff: the
            // all-zero record) of this segment's chunk, so that no k-step spans two chunks
#pragma unroll
            for (int w = 0; w < NL; ++w) {
              const int pad = (-cnt[w]) & 3;
              if (lane < pad) lists[(size_t)w * capL + cnt[w] + lane] = 0x1ffu | dch;
              cnt[w] += pad;
            }
          }
        }
      }
#pragma unroll
      for (int w = 0; w < NL; ++w)
        if (lane == w % 32) s_cnt[stage * NL + w] = (uint32_t)cnt[w];
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_full[stage]);
      if (kProf && lane == 0) {
        atomicAdd(prm.prof + 9, l1c - l0c);
        atomicAdd(prm.prof + 10, clock64() - l1c);
      }
      if (hdr.B < 0) break;
    }
    return;
  }

  if constexpr (INV) {
    // ======================= consumer warps, inverse direction (gather) =======================
    // Interpolating step of the inverse CUNFFT: f_j = sum_l g(l) w0 w1 w2.  A warp
    // holds the grid values of its 4 x 4 column sub-patch for the 16 cyclic node rows around the
    // current chunk as the A operand of DMMA m16n8k4 (A[node][col], rows g and g + 8, column t
    // of slice s = sub-patch row s), loaded once per node.  Per k-step of 8 records (N = record):
    //   H[node][record] = sum_{s, t} G[node][(s, t)] * (w1[i1(s)] w2[i2(t)])[record]   (4 DMMA, re and im)
    //   partial_j = sum_node w0_j[node] H[node][j]   (lane products + shuffle reduction)
    // and the partials of a point from the warps (and CTAs) its footprint spans are summed with
    // global atomics (native f64 RED in L2).  Nodes outside the tile's segment read as 0, so
    // every (point, node) pair is gathered exactly once, mirroring the adjoint's flush.
    static_assert(C::SUB == 1, "inverse consumer: one sub-patch per warp");
    constexpr int NT = kWR * kWC / 4;   // slices (sub-patch rows), 4 columns each
    const int wr_off = (warp / (P2 / kWC)) * kWR;
    const int wc_off = (warp % (P2 / kWC)) * kWC;
    const int g = lane >> 2, t = lane & 3;
    int cur_tile = -1;
    int first = 0, off = 0, S = 0, wr0 = 0, wc0 = 0;
    double gre[NT][2], gim[NT][2];
    int ld = 0;                         // relative nodes < ld are loaded
    const size_t plane = (size_t)n1 * n2;
    // load relative nodes [ld, upto] into their cyclic rows (node & 15): in blocks of <= 16
    // nodes, each lane fetches the (at most two) nodes of its rows g and g + 8 with all their
    // global loads in flight before any register is written
    auto load_nodes = [&](int upto) {
      while (ld <= upto) {
        const int nb = min(16, upto - ld + 1);
        const int row0 = ld & 15;
        double2 v[2][NT];
        bool has[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ds = (g + 8 * h - row0) & 15;   // offset of this lane's row h in the block
          has[h] = ds < nb;
          const int node = ld + ds;
          const int rel = node - off;                // node - L0
          const bool in = has[h] && rel >= 0 && rel < S;
          const int l0 = (first + node) & (n0 - 1);
          const double2* base = reinterpret_cast<const double2*>(prm.grid) + (size_t)l0 * plane +
                                (size_t)wr0 * n2 + (wc0 + t);
#pragma unroll
          for (int sl = 0; sl < NT; ++sl)
            v[h][sl] = (in && wr0 + sl < n1) ? __ldg(base + (size_t)sl * n2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (has[h]) {
#pragma unroll
            for (int sl = 0; sl < NT; ++sl) {
              gre[sl][h] = v[h][sl].x;
              gim[sl][h] = v[h][sl].y;
            }
          }
        }
        ld += nb;
      }
    };
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t zaddr = (uint32_t)__cvta_generic_to_shared(s_zero);
    for (;;) {
      mbar_wait(&s_full[stage], phase);
      const BatchHdr hdr = s_hdr[stage];
      if (hdr.B < 0) break;
      if (hdr.tile != cur_tile) {
        cur_tile = hdr.tile;
        int R0, C0, L0, a_lo, nch;
        tile_geom(cur_tile, R0, C0, L0, S, a_lo, nch);
        first = a_lo * CH;
        off = L0 - first;
        wr0 = R0 + wr_off;
        wc0 = C0 + wc_off;
        ld = -M_ + 1;
#pragma unroll
        for (int sl = 0; sl < NT; ++sl) gre[sl][0] = gre[sl][1] = gim[sl][0] = gim[sl][1] = 0.0;
      }
      const int step0 = hdr.chunk * CH;
      if (hdr.B > 0) load_nodes(step0 + CH - 1 + M_);   // the chunk's cells reach these nodes
      const double* recs = s_rec + (size_t)stage * cap * RD;
      const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(recs);
      const int nlist = (int)s_cnt[stage * NL + warp];
      const uint32_t* my = s_list + ((size_t)stage * NL + warp) * capL;
      for (int k = 0; k < nlist; k += 8) {
        // B: lane (g, t) = record k + g, column t of every slice
        const bool act = k + g < nlist;
        const uint32_t en = act ? my[k + g] : 0u;
        const uint32_t ra = act ? rbase + (en & 0x1ffu) * (uint32_t)(RD * sizeof(double)) : zaddr;
        const int d1 = (int)((en >> 18) & 31u), d2 = (int)((en >> 23) & 31u);
        const double w2v = lds_f64(w12_addr<W>(ra, R::kW2, (unsigned)(d2 - (kWC - 1) + t), zaddr));
        double hre[4] = {0.0, 0.0, 0.0, 0.0}, him[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int sl = 0; sl < NT; ++sl) {
          const double b =
              w2v * lds_f64(w12_addr<W>(ra, R::kW1, (unsigned)(d1 - (kWR - 1) + sl), zaddr));
          dmma16(hre, gre[sl][0], gre[sl][1], b);
          dmma16(him, gim[sl][0], gim[sl][1], b);
        }
        // lane holds H[g][2t], H[g][2t+1], H[g+8][2t], H[g+8][2t+1] (re and im)
        double pr[2], pi[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = 2 * t + q;      // record of this column pair
          const uint32_t enr = __shfl_sync(0xffffffffu, en, 4 * r);
          const bool actr = k + r < nlist;
          const uint32_t rar = actr ? rbase + (enr & 0x1ffu) * (uint32_t)(RD * sizeof(double)) : zaddr;
          const int sh = step0 + (int)((enr >> 9) & (uint32_t)(CH - 1)) - M_ + 1;
          const double wa = lds_f64(w0_addr<W>(rar, (unsigned)((g - sh) & 15), zaddr));
          const double wb = lds_f64(w0_addr<W>(rar, (unsigned)((8 + g - sh) & 15), zaddr));
          pr[q] = wa * hre[q] + wb * hre[2 + q];
          pi[q] = wa * him[q] + wb * him[2 + q];
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {   // sum over g (lanes with the same t)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            pr[q] += __shfl_xor_sync(0xffffffffu, pr[q], o);
            pi[q] += __shfl_xor_sync(0xffffffffu, pi[q], o);
          }
        }
        if (g == 0) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int r = 2 * t + q;
            if (k + r < nlist) {
              const uint32_t enr = my[k + r];
              const int pj = reinterpret_cast<const int*>(recs + (size_t)(enr & 0x1ffu) * RD)[3];
              atomicAdd(prm.fout + 2 * (size_t)pj, pr[q]);
              atomicAdd(prm.fout + 2 * (size_t)pj + 1, pi[q]);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[stage]);
      if (++stage == NS) {
        stage = 0;
        phase ^= 1u;
      }
    }
    return;
  }

  // =============================== consumer warps ===============================
  // A warp owns a 4 x 4 sub-patch of columns; its accumulator is the 16 x 32 real matrix
  // C[node row][2 x complex column] held as 4 DMMA m16n8k4 C-fragments.  Node rows are cyclic
  // (row = relative node mod 16), so the sliding window needs no data movement: a finished node
  // row is stored and zeroed.  Four records per k-step:
  //   C += A (16 x 4: w0 of each record placed at its cell's cyclic offset)
  //      x B (4 x 32: f w1[i1] w2[i2] of each record for every column, 0 outside its footprint)
  // consumer warp `warp` owns sub-patches warp * SUB .. warp * SUB + SUB - 1 (each 4 x 4 columns)
  int wr_off[SUB], wc_off[SUB];
#pragma unroll
  for (int u = 0; u < SUB; ++u) {
    const int spid = warp * SUB + u;
    wr_off[u] = (spid / (P2 / kWC)) * kWR;
    wc_off[u] = (spid % (P2 / kWC)) * kWC;
  }
  const int g = lane >> 2, t = lane & 3;
  static_assert(!(REAL && INV), "the real sweep is a spread");
  // n-tiles of 8 real columns: complex = 4 complex columns (row nt, cols 0..3, re/im); REAL = 8
  // real columns (rows 2 nt, 2 nt + 1, cols 0..3)
  constexpr int NT = REAL ? kWR * kWC / 8 : kWR * kWC / 4;
  const int part = REAL ? 0 : (g & 1);    // B: real (0) or imaginary (1) part of the column
  const int bc0 = REAL ? (g & 3) : (g >> 1);   // B: sub-patch column of B's column g
  const int br0 = REAL ? (g >> 2) : 0;    // B: row of B's column g within the n-tile (REAL)
  // C: the complex column (row nt, col t) | REAL: the real columns 2t, 2t + 1 = (row 2 nt + t/2,
  // cols 2 (t & 1), + 1) -- either way one 16-byte store per accumulator row
  const int cr0 = REAL ? (t >> 1) : 0, cc0 = REAL ? 2 * (t & 1) : t;
  int cur_tile = -1;
  int first = 0, off = 0, S = 0, nsteps = 0;
  int wr0[SUB], wc0[SUB];
  double acc[SUB][NT][4];                 // m16n8k4 C-fragment per n-tile: rows g (0, 1), g + 8 (2, 3)
#pragma unroll
  for (int u = 0; u < SUB; ++u) {
    wr0[u] = wc0[u] = 0;
#pragma unroll
    for (int a = 0; a < NT; ++a) acc[u][a][0] = acc[u][a][1] = acc[u][a][2] = acc[u][a][3] = 0.0;
  }
  int cur = 0;                            // steps (cells first + s) < cur are flushed

  // Flush steps [cur, upto): after step sp (cell first + sp) node first + sp - m + 1 is final
  // (accumulator row (sp - m + 1) mod 16).  In blocks of at most 16 steps, each lane stores its
  // rows g and g + 8 if they belong to a step of the block: nodes inside the tile's planes
  // [L0, L0 + S) (node - L0 = sp - m + 1 - off) go to the grid, then the row is zeroed.
  const size_t plane = (size_t)n1 * n2;
  // row (within the sub-patch) and grid address of this lane's C columns of n-tile nt, plane l0
  auto node_row = [&](int nt) { return REAL ? 2 * nt + cr0 : nt; };
  auto node_dst = [&](int u, int l0, int nt) -> double2* {
    if constexpr (REAL)
      return reinterpret_cast<double2*>(prm.grid + (size_t)l0 * plane + (size_t)(wr0[u] + node_row(nt)) * n2 +
                                        (wc0[u] + cc0));
    else
      return reinterpret_cast<double2*>(prm.grid) + (size_t)l0 * plane + (size_t)(wr0[u] + nt) * n2 + (wc0[u] + cc0);
  };
  auto advance = [&](int upto) {
#if HPNFFT_SWEEP_DEBUG == 3
    cur = upto > cur ? upto : cur;   // measurement only: no flush
    return;
#endif
    while (cur < upto) {
      const int nb = min(16, upto - cur);
      const int row0 = (cur - M_ + 1) & 15;
#if HPNFFT_SWEEP_LEANFLUSH
      if (nb <= 8) {
        // a block of <= 8 steps (the per-chunk flush: CH steps) holds at most one of this lane's
        // rows g, g + 8: one address computation, values picked by select
        const int d0 = (g - row0) & 15, d1 = (g + 8 - row0) & 15;
        const bool a0 = d0 < nb, a1 = d1 < nb;
        if (a0 || a1) {
          const int sp = cur + (a0 ? d0 : d1);
          const int rel = sp - M_ + 1 - off;
          const int l0 = (first + sp - M_ + 1) & (n0 - 1);
          const bool in_seg = rel >= 0 && rel < S;
#pragma unroll
          for (int u = 0; u < SUB; ++u) HPNFFT_DCHECK(!in_seg || (wc0[u] + cc0 < n2 && wr0[u] >= 0 && l0 >= 0));
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const double vx = a0 ? acc[u][nt][0] : acc[u][nt][2];
              const double vy = a0 ? acc[u][nt][1] : acc[u][nt][3];
              if (in_seg && wr0[u] + node_row(nt) < n1) {
                double2* dst = node_dst(u, l0, nt);
                if (prm.accumulate) {
                  double2 o = *dst;
                  o.x += vx;
                  o.y += vy;
                  *dst = o;
                } else {
                  *dst = make_double2(vx, vy);
                }
              }
              if (a0) {
                acc[u][nt][0] = acc[u][nt][1] = 0.0;
              } else {
                acc[u][nt][2] = acc[u][nt][3] = 0.0;
              }
            }
          }
        }
        cur += nb;
        continue;
      }
#endif
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ds = (g + 8 * h - row0) & 15;     // step offset of this lane's row in the block
        if (ds < nb) {
          const int sp = cur + ds;
          const int rel = sp - M_ + 1 - off;
          const int l0 = (first + sp - M_ + 1) & (n0 - 1);
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {   // the lane's C columns of n-tile nt
              if (rel >= 0 && rel < S && wr0[u] + node_row(nt) < n1) {
                double2* dst = node_dst(u, l0, nt);
                if (prm.accumulate) {
                  double2 o = *dst;
                  o.x += acc[u][nt][2 * h];
                  o.y += acc[u][nt][2 * h + 1];
                  *dst = o;
                } else {
                  *dst = make_double2(acc[u][nt][2 * h], acc[u][nt][2 * h + 1]);
                }
              }
              acc[u][nt][2 * h] = acc[u][nt][2 * h + 1] = 0.0;
            }
          }
        }
      }
      cur += nb;
    }
  };

  int stage = 0;
  uint32_t phase = 0;
  unsigned long long tw = 0, tl = 0, tf = 0, tA = 0;
  const uint32_t zaddr = (uint32_t)__cvta_generic_to_shared(s_zero);
  for (;;) {
    const unsigned long long q0 = kProf ? clock64() : 0ull;
    mbar_wait(&s_full[stage], phase);
    const unsigned long long q1 = kProf ? clock64() : 0ull;
    const BatchHdr hdr = s_hdr[stage];
    if (hdr.B < 0) break;
    if (hdr.tile != cur_tile) {
      cur_tile = hdr.tile;
      int R0, C0, L0, a_lo, nch;
      tile_geom(cur_tile, R0, C0, L0, S, a_lo, nch);
      first = a_lo * CH;
      off = L0 - first;
      nsteps = nch * CH;
      cur = 0;
#pragma unroll
      for (int u = 0; u < SUB; ++u) {
        wr0[u] = R0 + wr_off[u];
        wc0[u] = C0 + wc_off[u];
#pragma unroll
        for (int a = 0; a < NT; ++a) acc[u][a][0] = acc[u][a][1] = acc[u][a][2] = acc[u][a][3] = 0.0;
      }
    }
    const int step0 = hdr.chunk * CH;
    const double* recs = s_rec + (size_t)stage * cap * RD;
    // ---- this warp's lists (built by the list warp) ----
    int nl[SUB];
    const uint32_t* ml[SUB];
#pragma unroll
    for (int u = 0; u < SUB; ++u) {
      nl[u] = (int)s_cnt[stage * NL + warp * SUB + u];
      ml[u] = s_list + ((size_t)stage * NL + warp * SUB + u) * capL;
    }
    int nlist = nl[0];
    const uint32_t* my = ml[0];
#pragma unroll
    for (int u = 0; u < SUB; ++u) HPNFFT_DCHECK(nl[u] >= 0 && nl[u] <= capL);
    const unsigned long long q2 = kProf ? clock64() : 0ull;
#if HPNFFT_SWEEP_DEBUG == 2
    nlist = 0;   // measurement only: skip apply
#pragma unroll
    for (int u = 0; u < SUB; ++u) nl[u] = 0;
#endif
    // ---- k-steps of 4 records (any order inside the chunk); lanes past the list end read the
    //      all-zero record ----
    const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(recs);
    // operands of one k-step (lane: record k + t), loaded as a group so that two k-steps' shared
    // memory loads are in flight before their DMMAs issue
    // Sub-patch rows (n-tiles) outside every footprint of the k-step are skipped
    // (HPNFFT_SWEEP_NTSKIP): lists are in batch order = candidate-row order, so the 4 records of
    // a k-step mostly share d1.
    // kc: the k-step's chunk offset within a multi-chunk batch (entries of a k-step share it;
    // lane 0 always holds a live entry); null entries (0x1ff, list padding) read the zero record
    auto fetch_l = [&](const uint32_t* lst, int n, int k, double& a0, double& a1, double& fp, double& w2v,
                       double (&w1v)[NT], int& ntlo, int& nthi, int& kc) {
      const bool act = k + t < n;
      const uint32_t en = act ? lst[k + t] : 0u;
      const bool live = act && (!kMerge || (en & 0x1ffu) != 0x1ffu);
      HPNFFT_DCHECK(!live || (int)(en & 0x1ffu) < hdr.B);
      const uint32_t ra = live ? rbase + (en & 0x1ffu) * (uint32_t)(RD * sizeof(double)) : zaddr;
      kc = kMerge ? (int)__shfl_sync(0xffffffffu, (en >> 11) & 127u, 0) : 0;
      const int sh = step0 + kc * CH + (int)((en >> 9) & (uint32_t)(CH - 1)) - M_ + 1;
      const int d1 = (int)((en >> 18) & 31u), d2 = (int)((en >> 23) & 31u);
      // A fragments: rows 8 mt + g hold node (row - (st - m + 1)) mod 16 of this record
      a0 = lds_f64(w0_addr<W>(ra, (unsigned)((g - sh) & 15), zaddr));
      a1 = lds_f64(w0_addr<W>(ra, (unsigned)((8 + g - sh) & 15), zaddr));
      // B fragments: complex column q = 4 nt + g/2 = (row nt, col g/2) of the 4 x 4 sub-patch,
      // part g & 1; value f_part w1[i1(nt)] w2[i2(g/2)] (indices past the footprint hit zero pads)
      fp = lds_f64(ra + 8u * (uint32_t)(2 + part));
      w2v = lds_f64(w12_addr<W>(ra, R::kW2, (unsigned)(d2 - (kWC - 1) + bc0), zaddr));
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        w1v[nt] = lds_f64(w12_addr<W>(ra, R::kW1, (unsigned)(d1 - (kWR - 1) + (REAL ? 2 * nt + br0 : nt)), zaddr));
#if HPNFFT_SWEEP_NTSKIP
      if constexpr (!REAL) {
        const int lo = act ? max(0, (kWR - 1) - d1) : NT, hi = act ? min(NT - 1, W + kWR - 2 - d1) : -1;
        ntlo = (int)__reduce_min_sync(0xffffffffu, (unsigned)lo);
        nthi = __reduce_max_sync(0xffffffffu, hi + 1) - 1;
      } else {
        ntlo = 0;
        nthi = NT - 1;
      }
#else
      ntlo = 0;
      nthi = NT - 1;
#endif
    };
    auto fetch = [&](int k, double& a0, double& a1, double& fp, double& w2v, double (&w1v)[NT], int& ntlo,
                     int& nthi, int& kc) { fetch_l(my, nlist, k, a0, a1, fp, w2v, w1v, ntlo, nthi, kc); };
    auto apply_u = [&](double (&ac)[NT][4], double a0, double a1, double fp, double w2v, const double (&w1v)[NT],
                       int ntlo, int nthi) {
      const double fw2 = fp * w2v;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if (nt < ntlo || nt > nthi) continue;   // warp-uniform
        const double b = fw2 * w1v[nt];
#if HPNFFT_SWEEP_DEBUG == 1
        ac[nt][0] += a0 * b + a1;   // measurement only: keep the operands alive, skip the MMAs
#else
        dmma16(ac[nt], a0, a1, b);
#endif
      }
    };
    auto apply = [&](double a0, double a1, double fp, double w2v, const double (&w1v)[NT], int ntlo, int nthi) {
      apply_u(acc[0], a0, a1, fp, w2v, w1v, ntlo, nthi);
    };
    if constexpr (SUB == 1) {
      // the first k-step's operand loads are issued before the flush of the earlier chunks, whose
      // accumulator reads wait for this warp's in-flight DMMAs
      double p0, p1, pf, p2v, p1v[NT];
      int plo = 0, phi = NT - 1, pkc = 0;
      if (nlist > 0) fetch(0, p0, p1, pf, p2v, p1v, plo, phi, pkc);
      advance(step0 + pkc * CH);            // earlier chunks are complete
      int ckc = pkc;                        // chunk (offset) the accumulator window is at
      auto to_chunk = [&](int kc) {         // a multi-chunk batch moves on: flush the chunks before
        if (kMerge && kc != ckc) {
          advance(step0 + kc * CH);
          ckc = kc;
        }
      };
      int k = 0;
      if (nlist > 0) {
        if (nlist > 4) {
          double b0, b1, gp, g2v, g1v[NT];
          int blo, bhi, bkc;
          fetch(4, b0, b1, gp, g2v, g1v, blo, bhi, bkc);
          apply(p0, p1, pf, p2v, p1v, plo, phi);
          to_chunk(bkc);
          apply(b0, b1, gp, g2v, g1v, blo, bhi);
          k = 8;
        } else {
          apply(p0, p1, pf, p2v, p1v, plo, phi);
          k = 4;
        }
      }
      for (; k + 4 < nlist; k += 8) {   // two k-steps per iteration
        double a0, a1, fp, w2v, w1v[NT], b0, b1, gp, g2v, g1v[NT];
        int alo, ahi, blo, bhi, akc, bkc;
        fetch(k, a0, a1, fp, w2v, w1v, alo, ahi, akc);
        fetch(k + 4, b0, b1, gp, g2v, g1v, blo, bhi, bkc);
        to_chunk(akc);
        apply(a0, a1, fp, w2v, w1v, alo, ahi);
        to_chunk(bkc);
        apply(b0, b1, gp, g2v, g1v, blo, bhi);
      }
      if (k < nlist) {
        double a0, a1, fp, w2v, w1v[NT];
        int alo, ahi, akc;
        fetch(k, a0, a1, fp, w2v, w1v, alo, ahi, akc);
        to_chunk(akc);
        apply(a0, a1, fp, w2v, w1v, alo, ahi);
      }
    } else {
      // two sub-patches: their k-steps (independent accumulators) are interleaved
      double p0, p1, pf, p2v, p1v[NT], b0, b1, gp, g2v, g1v[NT];
      int plo = 0, phi = NT - 1, blo = 0, bhi = NT - 1;
      int kc_unused = 0;   // single-chunk batches (no merging with two sub-patches per warp)
      if (nl[0] > 0) fetch_l(ml[0], nl[0], 0, p0, p1, pf, p2v, p1v, plo, phi, kc_unused);
      if (nl[1] > 0) fetch_l(ml[1], nl[1], 0, b0, b1, gp, g2v, g1v, blo, bhi, kc_unused);
      advance(step0);                     // earlier chunks are complete
      int ka = 0, kb = 0;
      while (ka < nl[0] || kb < nl[1]) {
        const bool da = ka < nl[0], db = kb < nl[1];
        if (da) apply_u(acc[0], p0, p1, pf, p2v, p1v, plo, phi);
        if (db) apply_u(acc[1], b0, b1, gp, g2v, g1v, blo, bhi);
        ka += 4;
        kb += 4;
        if (ka < nl[0]) fetch_l(ml[0], nl[0], ka, p0, p1, pf, p2v, p1v, plo, phi, kc_unused);
        if (kb < nl[1]) fetch_l(ml[1], nl[1], kb, b0, b1, gp, g2v, g1v, blo, bhi, kc_unused);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[stage]);
    const unsigned long long q3 = kProf ? clock64() : 0ull;
    if (hdr.end == 1) advance(nsteps);   // tile finished: flush the remaining nodes
    if (hdr.end == 2) cur = nsteps;      // tile skipped in a multi-group pass: nothing to write
    if (kProf) {
      tw += q1 - q0;
      tl += q2 - q1;
      tf += q3 - q2;
      tA += clock64() - q3;
    }
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
#if HPNFFT_SWEEP_DEBUG == 3
  {  // keep the accumulators alive
    double z = 0.0;
#pragma unroll
    for (int u = 0; u < SUB; ++u)
#pragma unroll
      for (int a = 0; a < NT; ++a) z += acc[u][a][0] + acc[u][a][1] + acc[u][a][2] + acc[u][a][3];
    if (z == 1234.5678) prm.grid[0] = z;
  }
#endif
  if (kProf && lane == 0) {
    atomicAdd(prm.prof + 0, tw);
    atomicAdd(prm.prof + 1, tl);
    atomicAdd(prm.prof + 2, tf);
    atomicAdd(prm.prof + 3, tA);
    atomicAdd(prm.prof + 7, 1ull);
  }
}

namespace {

// CTA patch variant (consumer warps = patch / 4 x 4, + copy and list warps): 0 = 8 x 32 (16, the
// default), 1 = 12 x 32 (24), 2 = 16 x 16 (16), 3 = 8 x 16 (8, two CTAs per SM), 4 = 12 x 16 (12,
// 128 registers); HPNFFT_SWEEP_PATCH = "8x32" | "12x32" | "16x16" | "8x16" | "12x16".
int sweep_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HPNFFT_SWEEP_PATCH");
    if (e && e[0] == '1' && e[1] == '2' && e[3] == '3') v = 1;
    else if (e && e[0] == '1' && e[1] == '6') v = 2;
    else if (e && e[0] == '8' && e[2] == '1') v = 3;
    else if (e && e[0] == '1' && e[1] == '2' && e[3] == '1') v = 4;
    else v = 0;
  }
  return v;
}

// ---------------------------------------------------------------------------------------------
// Tile order for the persistent sweep: clustered inputs make a few tiles (the patches under a
// cluster core) carry a large share of the records; taken in index order, one of them can start
// late and leave every other SM idle (a tail of up to one heavy tile).  One warp per tile counts
// the records the producer will copy (the same rows, bin runs and group clipping), then one CTA
// sorts the tiles by count, largest first (longest-processing-time-first), unless the counts are
// nearly uniform (max <= 2 x mean: index order, which keeps neighbouring tiles together).
constexpr int kMaxOrderTiles = 16384;

template <int P1, int P2, int M_>
__global__ void __launch_bounds__(256) k_tile_counts(SweepParams prm, int ntiles, unsigned long long* keys) {
  using C = SweepCfg<P1, P2, M_>;
  constexpr int CH = Chunk<M_>::CH;
  const int lane = threadIdx.x & 31;
  const int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  if (t >= ntiles) return;
  const int n1 = prm.n1, n2 = prm.n2, nchunks0 = prm.n0 / CH;
  const int npc = n2 / P2, npr = (n1 + P1 - 1) / P1;
  const int pc = t % npc, rest = t / npc, pr = rest % npr, segi = rest / npr;
  const int R0 = pr * P1, C0 = pc * P2;
  const int L0 = prm.plane_lo + segi * prm.seg;
  const int S = min(prm.seg, prm.plane_len - segi * prm.seg);
  const int a_lo = floor_div(L0 - M_, CH);
  const int nch = floor_div(L0 + S + M_ - 2, CH) - a_lo + 1;
  // an estimate is enough to rank the tiles: the records of the patch's own rows and c2 bins
  // (no footprint halo) in every other chunk -- ~5x fewer bin lookups than the producer makes
  // lanes = 8 rows x 4 chunk phases (all 32 lanes busy, ~9 independent lookups each)
  const int row = lane & 7, phase = lane >> 3;
  const int c1 = (R0 + row) & (n1 - 1);
  const int b2lo = C0 / kBinW, b2hi = (C0 + P2 - 1) / kBinW;
  int ra0 = b2lo, rb0 = b2hi, ra1 = 0, rb1 = -1;
  if (b2lo < 0) {
    ra0 = 0;
    ra1 = b2lo + prm.nb2;
    rb1 = prm.nb2 - 1;
  } else if (b2hi >= prm.nb2) {
    rb0 = prm.nb2 - 1;
    ra1 = 0;
    rb1 = b2hi - prm.nb2;
  }
  uint32_t cnt = 0;
  (void)sizeof(C);
  if (row < P1) {
#pragma unroll 4
    for (int ci = 2 * phase; ci < nch; ci += 8) {
      int a = a_lo + ci;
      while (a < 0) a += nchunks0;
      while (a >= nchunks0) a -= nchunks0;
      const size_t rowbase = ((size_t)a * n1 + c1) * prm.nb2;
      auto run = [&](int ra, int rb) {
        if (rb < ra) return;
        const uint32_t lo = max(__ldg(prm.start + (rowbase + ra)), prm.g0);
        const uint32_t hi = min(__ldg(prm.start + (rowbase + rb + 1)), prm.g1);
        cnt += hi > lo ? hi - lo : 0u;
      };
      run(ra0, rb0);
      run(ra1, rb1);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) keys[t] = ((unsigned long long)cnt << 32) | (unsigned long long)(t + 1);
}

// one CTA: bitonic sort of the (count, tile + 1) keys, descending; padding keys are 0 (last)
__global__ void __launch_bounds__(1024) k_tile_order(const unsigned long long* __restrict__ keys_in, int ntiles,
                                                     int* __restrict__ order) {
  extern __shared__ unsigned long long sk[];
  __shared__ unsigned long long s_max, s_sum;
  int P = 1;
  while (P < ntiles) P <<= 1;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_sum = 0;
  }
  __syncthreads();
  unsigned long long mx = 0, sm = 0;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const unsigned long long k = i < ntiles ? keys_in[i] : 0ull;
    sk[i] = k;
    mx = max(mx, k >> 32);
    sm += k >> 32;
  }
  atomicMax(&s_max, mx);
  atomicAdd(&s_sum, sm);
  __syncthreads();
  if (s_max * (unsigned long long)ntiles <= 2ull * s_sum) {   // nearly uniform: index order
    for (int i = threadIdx.x; i < ntiles; i += blockDim.x) order[i] = i;
    return;
  }
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = sk[i], b = sk[l];
          const bool desc = (i & k) == 0;   // descending overall
          if (desc ? (a < b) : (a > b)) {
            sk[i] = b;
            sk[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < ntiles; i += blockDim.x) order[i] = (int)(sk[i] & 0xffffffffull) - 1;
}

// Node planes per tile segment (HPNFFT_SWEEP_SEG, default 256; a multiple of the chunk).  Shorter
// segments split a patch's planes over more tiles (each with its 2m - 1 halo planes again): more
// total work, but a heavy patch (clustered points) no longer bounds the persistent grid's makespan.
template <int CH>
int sweep_max_seg() {
  const char* e = getenv("HPNFFT_SWEEP_SEG");
  int s = e ? atoi(e) : 256;
  if (s < 4 * CH) s = 4 * CH;
  return s / CH * CH;
}

// Tile order for the next sweep of group [g0, g1), computed on the plan's side stream so that
// it overlaps the records kernel (it only needs the bin table of set_points).  HPNFFT_SWEEP_LPT=0
// keeps index order.  Same plane range / segment geometry as launch_sweep_group.
template <int P1, int P2, int M_>
int prepare_tile_order(Plan* p, uint32_t g0, uint32_t g1) {
  constexpr int CH = Chunk<M_>::CH;
  p->sched_pending = false;
  const char* lpt_env = getenv("HPNFFT_SWEEP_LPT");   // read per call (tests switch it in-process)
  const bool lpt_off = lpt_env && lpt_env[0] == '0';
  if (lpt_off) return HPNFFT_OK;
  SweepParams prm{};
  prm.start = p->bin_count;
  prm.g0 = g0;
  prm.g1 = g1;
  prm.n0 = (int)p->n[0];
  prm.n1 = (int)p->n[1];
  prm.n2 = (int)p->n[2];
  prm.nb2 = (int)(p->n[2] / kBinW);
  const int64_t n0 = p->n[0];
  const int64_t lo_al = p->plane_lo & ~(int64_t)(CH - 1);
  int64_t len_al = p->plane_len + (p->plane_lo - lo_al);
  len_al = (len_al + CH - 1) & ~(int64_t)(CH - 1);
  if (len_al > n0) len_al = n0;
  prm.plane_lo = (int)lo_al;
  prm.plane_len = (int)len_al;
  prm.seg = (int)(len_al < sweep_max_seg<CH>() ? len_al : sweep_max_seg<CH>());
  prm.nseg = (int)((len_al + prm.seg - 1) / prm.seg);
  const int64_t tiles = ((p->n[1] + P1 - 1) / P1) * (p->n[2] / P2) * prm.nseg;
  if (tiles <= 1 || tiles > kMaxOrderTiles) return HPNFFT_OK;
  if (!p->tile_sched &&
      cudaMalloc(&p->tile_sched, (sizeof(unsigned long long) + sizeof(int)) * kMaxOrderTiles) != cudaSuccess) {
    cudaGetLastError();
    p->tile_sched = nullptr;
    return HPNFFT_OK;   // index order
  }
  if (!p->side) {
    if (cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->side_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->side_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return HPNFFT_OK;
    }
  }
  unsigned long long* keys = static_cast<unsigned long long*>(p->tile_sched);
  int* order = reinterpret_cast<int*>(keys + kMaxOrderTiles);
  HPNFFT_CUDA_TRY(p, cudaEventRecord(p->side_fork, p->stream), "fork tile order");
  HPNFFT_CUDA_TRY(p, cudaStreamWaitEvent(p->side, p->side_fork, 0), "fork tile order");
  k_tile_counts<P1, P2, M_><<<(unsigned)((tiles * 32 + 255) / 256), 256, 0, p->side>>>(prm, (int)tiles, keys);
  int pad = 1;
  while (pad < tiles) pad <<= 1;
  const size_t osmem = sizeof(unsigned long long) * (size_t)pad;
  HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(k_tile_order), (int)osmem),
                  "tile order smem attr");
  k_tile_order<<<1, 1024, osmem, p->side>>>(keys, (int)tiles, order);
  p->launches += 2;
  const int rc = check_launch(p, "tile order");
  if (rc) return rc;
  HPNFFT_CUDA_TRY(p, cudaEventRecord(p->side_join, p->side), "join tile order");
  p->sched_order = order;
  p->sched_pending = true;
  return HPNFFT_OK;
}

template <int P1, int P2, int M_, bool INV = false, bool REAL = false>
int launch_sweep_group(Plan* p, uint32_t g0, uint32_t g1, const int* chunks, bool accumulate, double* fout = nullptr) {
  using C = SweepCfg<P1, P2, M_>;
  constexpr int CH = Chunk<M_>::CH;
  const size_t smem_max = C::kCtasPerSm == 1 ? (size_t)(227 * 1024) : (size_t)(113 * 1024);
  // multi-chunk batches when a (tile, chunk) holds few records on average (sparse REAL points:
  // one pipeline round trip per chunk would dominate); HPNFFT_SWEEP_MERGE=0/1 forces the choice
  constexpr int W = 2 * M_;
  // (points per cell of the planes this plan spreads: a grid-slab rank's slab, occupied planes)
  const double planes = (double)(p->plane_len > 0 ? p->plane_len : p->n[0]);
  const double dens = (double)p->M / (planes * (double)p->n[1] * (double)p->n[2]);
  const double per_chunk = dens * (P1 + W - 1) * (P2 + W - 1) * CH;
  // measured (tools/merge_threshold.py, tools/enuf_bench.py): with one list warp per stage the
  // one-chunk kernel wins for complex values at every density down to ~1 record per (tile,
  // chunk); the merged kernel still wins for the REAL sweep of the ENUF charges (half the DMMA
  // work per record, so the per-chunk round trip dominates)
  bool merge = !INV && C::SUB == 1 && REAL && per_chunk < 64.0;
  if (const char* e = getenv("HPNFFT_SWEEP_MERGE")) merge = !INV && C::SUB == 1 && e[0] == '1';
  int cap = 32;
  static const int cap_max = [] {   // HPNFFT_SWEEP_CAP: smaller ring stages (measurement)
    const char* e = getenv("HPNFFT_SWEEP_CAP");
    return e ? atoi(e) : 480;
  }();
  constexpr int kModeA = INV ? kInverse : kDense;   // the non-merged instantiation's mode
  auto smem_of = [&](int c) {
    return merge ? sweep_smem_bytes_of<P1, P2, M_, kSparse>(c, true) : sweep_smem_bytes_of<P1, P2, M_, kModeA>(c, false);
  };
  while (cap + 32 <= 511 && cap + 32 <= cap_max && smem_of(cap + 32) <= smem_max) cap += 32;
  const size_t smem = smem_of(cap);
  SweepParams prm;
  prm.rec = p->rec;
  prm.start = p->bin_count;
  prm.grid = p->grid;
  prm.chunks = chunks;
  prm.g0 = g0;
  prm.g1 = g1;
  prm.accumulate = accumulate ? 1 : 0;
  prm.n0 = (int)p->n[0];
  prm.n1 = (int)p->n[1];
  prm.n2 = (int)p->n[2];
  prm.nb2 = (int)(p->n[2] / kBinW);
  // occupied node planes aligned to whole chunks
  const int64_t n0 = p->n[0];
  const int64_t lo_al = p->plane_lo & ~(int64_t)(CH - 1);
  int64_t len_al = p->plane_len + (p->plane_lo - lo_al);
  len_al = (len_al + CH - 1) & ~(int64_t)(CH - 1);
  if (len_al > n0) len_al = n0;
  prm.plane_lo = (int)lo_al;
  prm.plane_len = (int)len_al;
  prm.seg = (int)(len_al < sweep_max_seg<CH>() ? len_al : sweep_max_seg<CH>());
  prm.nseg = (int)((len_al + prm.seg - 1) / prm.seg);
  prm.cap = cap;
  prm.tile_counter = p->tile_counter;
  prm.fout = fout;
  static const bool prof_on = getenv("HPNFFT_SWEEP_PROF") != nullptr;
  unsigned long long* prof = nullptr;
  if (prof_on) {
    cudaMalloc(&prof, 16 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), p->stream);
  }
  prm.prof = prof;
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->tile_counter, 0, sizeof(int), p->stream), "tile counter");
  auto kern = k_spread_sweep<P1, P2, M_, INV, false, REAL>;
  if constexpr (!INV) {
    if (merge) kern = k_spread_sweep<P1, P2, M_, false, true, REAL>;
  }
  HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(kern), (int)smem),
                  "sweep smem attr");
  const int64_t tiles = ((p->n[1] + P1 - 1) / P1) * (p->n[2] / P2) * prm.nseg;
  prm.order = nullptr;
  if (p->sched_pending) {   // the tile order was computed on the side stream (prepare_tile_order)
    HPNFFT_CUDA_TRY(p, cudaStreamWaitEvent(p->stream, p->side_join, 0), "join tile order");
    prm.order = p->sched_order;
    p->sched_pending = false;
  }
  const int sms = device_sm_count();
  const int64_t slots = (int64_t)sms * C::kCtasPerSm;
  const int64_t blocks = tiles < slots ? tiles : slots;
  const int threads = merge ? SweepCfg<P1, P2, M_, kSparse>::kThreads : SweepCfg<P1, P2, M_, kModeA>::kThreads;
  kern<<<(unsigned)blocks, threads, smem, p->stream>>>(prm);
  p->launches++;
  if (prof) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, p->stream);
    cudaStreamSynchronize(p->stream);
    double nw = (double)h[7];
    fprintf(stderr,
            "[sweep prof] cap=%d consumer warps=%.0f  per warp Mcycles: wait_full %.2f  lists %.2f  apply %.2f  "
            "advance %.2f | producer (lane 0 sums, Mcycles): lookups %.2f  wait_empty %.2f  issue %.2f | list warp: "
            "wait_landed %.2f  build %.2f\n",
            cap, nw, h[0] / nw / 1e6, h[1] / nw / 1e6, h[2] / nw / 1e6, h[3] / nw / 1e6, h[4] / blocks / 1e6,
            h[5] / blocks / 1e6, h[6] / blocks / 1e6, h[9] / blocks / 1e6, h[10] / blocks / 1e6);
    cudaFree(prof);
  }
  return check_launch(p, "spread_sweep");
}

template <int M_>
int run_sweep(Plan* p, const double* f) {
  const uint32_t M = (uint32_t)p->M;
  const uint32_t G = (uint32_t)p->rec_group;
  const bool multi = M > G;
  const bool real = p->real_values;   // real f (ENUF charges): the REAL sweep onto a real grid
  if (multi) {
    const size_t bytes = sizeof(double) * (real ? 1 : 2) * (size_t)(p->n[0] * p->n[1] * p->n[2]);
    HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->grid, 0, bytes, p->stream), "zero grid");
  }
  uint32_t g0 = 0;
  do {
    const uint32_t g1 = (M - g0) < G ? M : g0 + G;
    const uint32_t cnt = g1 - g0;
    {
      const int v = real ? 0 : sweep_variant();
      const int rco = v == 4 ? prepare_tile_order<12, 16, M_>(p, g0, g1)
                    : v == 3 ? prepare_tile_order<8, 16, M_>(p, g0, g1)
                    : v == 1 ? prepare_tile_order<HPNFFT_P_A1, HPNFFT_P_A2, M_>(p, g0, g1)
                    : v == 2 ? prepare_tile_order<HPNFFT_P_B1, HPNFFT_P_B2, M_>(p, g0, g1)
                             : prepare_tile_order<HPNFFT_P_D1, HPNFFT_P_D2, M_>(p, g0, g1);
      if (rco) return rco;
    }
    if (cnt > 0) {
      stage_begin(p, 7);
      const size_t rsmem = sizeof(double) * kRecPts * Rec<2 * M_>::kDoubles;
      HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(k_point_records<M_>), (int)rsmem),
                      "records smem attr");
      k_point_records<M_><<<(cnt + kRecPts * HPNFFT_REC_CHUNKS - 1) / (kRecPts * HPNFFT_REC_CHUNKS), kRecPts, rsmem,
                            p->stream>>>(
          p->xs, p->perm, f, p->poly, p->rec, g0, cnt, p->n[0], p->n[1], p->n[2]);
      p->launches++;
      int rc = check_launch(p, "point records");
      stage_end(p, 7);
      if (rc) return rc;
    }
    if (multi) {
      const int64_t bins_per_chunk = (p->n[2] / kBinW) * p->n[1];
      uint32_t k_lo, k_hi;
      key_range(p, k_lo, k_hi);
      k_group_chunks<<<1, 32, 0, p->stream>>>(p->bin_count, k_lo, k_hi, g0, g1, bins_per_chunk, p->group_rows);
      p->launches++;
    }
    int rc;
    if (real) {
      rc = launch_sweep_group<HPNFFT_P_D1, HPNFFT_P_D2, M_, false, true>(p, g0, g1, p->group_rows, multi);
    } else {
      const int var = sweep_variant();
      rc = var == 4 ? launch_sweep_group<12, 16, M_>(p, g0, g1, p->group_rows, multi)
         : var == 3 ? launch_sweep_group<8, 16, M_>(p, g0, g1, p->group_rows, multi)
         : var == 1 ? launch_sweep_group<HPNFFT_P_A1, HPNFFT_P_A2, M_>(p, g0, g1, p->group_rows, multi)
         : var == 2 ? launch_sweep_group<HPNFFT_P_B1, HPNFFT_P_B2, M_>(p, g0, g1, p->group_rows, multi)
                    : launch_sweep_group<HPNFFT_P_D1, HPNFFT_P_D2, M_>(p, g0, g1, p->group_rows, multi);
    }
    if (rc) return rc;
    g0 = g1;
  } while (g0 < M);
  return HPNFFT_OK;
}

// inverse direction: records (no f) + the gather sweep, f summed atomically in original order
template <int M_>
int run_interp_sweep(Plan* p, double* fout) {
  const uint32_t M = (uint32_t)p->M;
  const uint32_t G = (uint32_t)p->rec_group;
  const bool multi = M > G;
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(fout, 0, sizeof(double) * 2 * (size_t)M, p->stream), "zero f");
  uint32_t g0 = 0;
  do {
    const uint32_t g1 = (M - g0) < G ? M : g0 + G;
    const uint32_t cnt = g1 - g0;
    {
      const int rco = prepare_tile_order<HPNFFT_P_D1, HPNFFT_P_D2, M_>(p, g0, g1);
      if (rco) return rco;
    }
    if (cnt > 0) {
      const size_t rsmem = sizeof(double) * kRecPts * Rec<2 * M_>::kDoubles;
      HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(k_point_records<M_>),
                                              (int)rsmem),
                      "records smem attr");
      k_point_records<M_><<<(cnt + kRecPts * HPNFFT_REC_CHUNKS - 1) / (kRecPts * HPNFFT_REC_CHUNKS), kRecPts, rsmem,
                            p->stream>>>(
          p->xs, p->perm, nullptr, p->poly, p->rec, g0, cnt, p->n[0], p->n[1], p->n[2]);
      p->launches++;
      int rc = check_launch(p, "point records");
      if (rc) return rc;
    }
    if (multi) {
      const int64_t bins_per_chunk = (p->n[2] / kBinW) * p->n[1];
      uint32_t k_lo, k_hi;
      key_range(p, k_lo, k_hi);
      k_group_chunks<<<1, 32, 0, p->stream>>>(p->bin_count, k_lo, k_hi, g0, g1, bins_per_chunk, p->group_rows);
      p->launches++;
    }
    const int rc = launch_sweep_group<HPNFFT_P_D1, HPNFFT_P_D2, M_, true>(p, g0, g1, p->group_rows, multi, fout);
    if (rc) return rc;
    g0 = g1;
  } while (g0 < M);
  return HPNFFT_OK;
}

}  // namespace

size_t record_bytes(int m) {
  switch (m) {
    case 1: return sizeof(double) * Rec<2>::kDoubles;
    case 2: return sizeof(double) * Rec<4>::kDoubles;
    case 3: return sizeof(double) * Rec<6>::kDoubles;
    case 4: return sizeof(double) * Rec<8>::kDoubles;
    case 5: return sizeof(double) * Rec<10>::kDoubles;
    case 6: return sizeof(double) * Rec<12>::kDoubles;
    case 7: return sizeof(double) * Rec<14>::kDoubles;
    default: return sizeof(double) * Rec<16>::kDoubles;
  }
}

bool sweep_supported(const Plan* p) {
  if (p->m > kMaxSweepM) return false;   // m = 9..15: the generic atomic spread / warp gather
  if (p->precision != HPNFFT_PRECISION_F64) return false;   // FP32 plans: spread_f32.cu
  const int W = 2 * p->m;
  const int P1 = 16, P2 = 32;   // largest extent of any patch variant
  if (p->n[2] < P2 || p->n[1] < P1) return false;
  if (p->n[1] < P1 + W) return false;                         // candidate rows must be distinct
  const int bins = (P2 + W - 1 + kBinW - 1) / kBinW + 1;      // candidate c2 bins must be distinct
  if (p->n[2] / kBinW < bins) return false;
  if (p->n[0] < 16 || p->n[0] < 2 * W) return false;
  if (p->rec == nullptr || p->rec_group == 0) return false;
  return true;
}

int interp_sweep(Plan* p, double* f) {
  switch (p->m) {
    case 1: return run_interp_sweep<1>(p, f);
    case 2: return run_interp_sweep<2>(p, f);
    case 3: return run_interp_sweep<3>(p, f);
    case 4: return run_interp_sweep<4>(p, f);
    case 5: return run_interp_sweep<5>(p, f);
    case 6: return run_interp_sweep<6>(p, f);
    case 7: return run_interp_sweep<7>(p, f);
    case 8: return run_interp_sweep<8>(p, f);
    default:
      set_error("m not supported by the sweep kernel");
      return HPNFFT_E_UNSUPPORTED;
  }
}

int spread_sweep(Plan* p, const double* f) {
  switch (p->m) {
    case 1: return run_sweep<1>(p, f);
    case 2: return run_sweep<2>(p, f);
    case 3: return run_sweep<3>(p, f);
    case 4: return run_sweep<4>(p, f);
    case 5: return run_sweep<5>(p, f);
    case 6: return run_sweep<6>(p, f);
    case 7: return run_sweep<7>(p, f);
    case 8: return run_sweep<8>(p, f);
    default:
      set_error("m not supported by the sweep kernel");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
