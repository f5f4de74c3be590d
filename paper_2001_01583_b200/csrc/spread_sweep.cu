// spread_sweep.cu -- the B200 spreading path (A3 + A4 of SURVEY.md §8(a)).
//
// Computes the "Spreading" step of CUNFFT (Fig. 1; §3)
//     g(l) = sum_j f_j * prod_t Phi(n_t x_jt - l_t),   l in I_n (periodic),
// without atomics and (for a single point group) without a zero fill: every grid node is
// written exactly once.
//
// Two kernels:
//  k_point_records  one thread per sorted point: cell (c1, c2), f_j, and the 3 x 2m tap weights
//                   from the window polynomials -> a 16-byte aligned record in HBM (A3).
//  k_spread_sweep   a CTA owns a P1 x P2 patch of grid columns (l1, l2) and a segment of S planes
//                   along l0.  Each lane owns ONE column and keeps a sliding window of the 2m nodes
//                   l0 = cur-m+1 .. cur+m of that column in registers.  The CTA sweeps cur over the
//                   planes; every point whose cell c0 equals cur adds f w1[i1] w2[i2] w0[i] to the
//                   2m window registers (static register indices), i.e. the 2(2m)^3 FMAs of a
//                   point become 2m FMA pairs on each lane of its footprint.  After plane cur, node
//                   cur-m+1 is final and stored once (a warp covers 4 rows x 8 consecutive l2:
//                   coalesced 128-byte rows), then the window shifts by one plane.
// The points of plane cur come from the bin table of sort.cu: bins are (c1 row, 8 consecutive
// c2, c0 plane) with c0 fastest, so for each (row, c2-bin) pencil around the patch the points of
// plane cur are one contiguous range of sorted records.  Per batch of planes the CTA copies those
// records to shared memory; each warp compacts the records whose 2m x 2m footprint touches its
// 4 x 8 sub-patch into its own plane-ordered list and applies them.
// When the records of all M points do not fit in the workspace, the sorted points are processed
// in groups ("the mass data have to be divided into several groups"): the grid is
// zeroed once and every group's sweep accumulates (CTAs whose rows miss the group exit early).
#include <stdio.h>
#include <stdlib.h>

#include "spread_common.cuh"

namespace hpnfft {

namespace {

#ifdef HPNFFT_SWEEP_DFMA
constexpr int kWR = 4;          // warp sub-patch: 4 rows (l1) x 8 cols (l2) = 32 lanes
constexpr int kWC = 8;
#else
constexpr int kWR = 4;          // warp sub-patch of the DMMA consumer: 4 rows (l1) x 4 cols (l2)
constexpr int kWC = 4;
#endif
constexpr int kBinW = 8;        // c2 bin width of the sort keys (sort.cu)
#ifndef HPNFFT_SWEEP_NS
#define HPNFFT_SWEEP_NS 3
#endif
#ifndef HPNFFT_SWEEP_CHUNK
#define HPNFFT_SWEEP_CHUNK 8
#endif
constexpr int kChunk = HPNFFT_SWEEP_CHUNK;   // planes whose pencil ranges are looked up together

// record layout in doubles: [0] c1|c2 (int2)  [1] pad  [2..3] f  [4..4+W) w0
//                           [4+W .. 5+2W) w1 (+ zero pad)  [5+2W .. 6+3W) w2 (+ zero pad)
template <int W>
struct Rec {
  static constexpr int kW0 = 4;
  static constexpr int kW1 = 4 + W;
  static constexpr int kW2 = 5 + 2 * W;
  static constexpr int kDoubles = 6 + 3 * W;      // even -> 16-byte multiple
  static constexpr int kChunks16 = kDoubles / 2;
};

template <int P1, int P2, int M_>
struct SweepCfg {
  static constexpr int W = 2 * M_;                       // taps per dimension
  static constexpr int kWarps = (P1 / kWR) * (P2 / kWC);
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kRows = P1 + W - 1;                // candidate c1 rows
  static constexpr int kBins = (P2 + W - 1 + kBinW - 1) / kBinW + 1;   // candidate c2 bins (upper bound)
  static constexpr int kPencils = kRows * kBins;
  static constexpr int kEntries = kChunk * kPencils;      // (plane, pencil) ranges per chunk
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

struct SweepParams {
  const double* rec;       // point records of the group (record r = sorted point g0 + r)
  const uint32_t* start;   // bin_start [nbins + 1]
  double* grid;            // [n0][n1][n2] complex
  const int* rows;         // [2] c1 rows spanned by the group (multi-group pass only)
  uint32_t g0, g1;         // sorted point range of this group
  int accumulate;          // 1: grid += window (multi-group), 0: grid = window
  int n0, n1, n2;
  int nb2;                 // n2 / 8
  int seg;                 // S: planes per segment
  int nseg;                // segments covering the occupied planes
  int plane_lo, plane_len; // occupied l0 planes (circular interval)
  int cap;                 // record capacity of one shared-memory batch buffer
  int* tile_counter;       // dynamic tile scheduler (zeroed before the launch)
  unsigned long long* prof;   // optional clock64 phase counters (HPNFFT_SWEEP_PROF=1), else null
  int debug;               // measurement only (HPNFFT_SWEEP_DEBUG): 1 = skip the MMAs, 2 = skip apply
};

}  // namespace

// ------------------------------------------------------------------------------------------
// A3: point records.  A CTA of 256 threads handles PB = 256 / 2m consecutive sorted points:
// thread (k, i) evaluates tap i of point k in the three dimensions (coefficients of tap i in
// registers, 3 independent Horner chains) into a shared-memory staging copy of the records, which
// is then written to HBM with coalesced 16-byte stores (the records of a CTA are contiguous).
template <int M_>
__global__ void __launch_bounds__(256) k_point_records(const double* __restrict__ xs, const uint32_t* __restrict__ perm,
                                                        const double* __restrict__ f, const double* __restrict__ poly_g,
                                                        double* __restrict__ rec, uint32_t g0, uint32_t count,
                                                        int64_t n0, int64_t n1, int64_t n2) {
  constexpr int W = 2 * M_;
  constexpr int PD = kPolyDeg + 1;
  constexpr int PB = 256 / W;
  using R = Rec<W>;
  __shared__ double poly[W * PD];
  __shared__ __align__(16) double stage[PB * R::kDoubles];
  for (int e = threadIdx.x; e < W * PD; e += blockDim.x) poly[e] = poly_g[e];
  __syncthreads();
  const uint32_t kb = blockIdx.x * PB;                 // first point of this CTA (group-relative)
  const int kl = threadIdx.x / W, i = threadIdx.x - kl * W;
  const uint32_t k = kb + kl;
  if (kl < PB && k < count) {
    const size_t src = (size_t)g0 + k;
    double* out = stage + kl * R::kDoubles;
    // issue the dependent gather f[perm[src]] first so its latency overlaps the Horner chains
    double2 fv = make_double2(0.0, 0.0);
    if (i == 0) fv = __ldg(reinterpret_cast<const double2*>(f) + __ldg(perm + src));
    const CellT a0 = cell_of(__ldg(xs + 3 * src), n0);
    const CellT a1 = cell_of(__ldg(xs + 3 * src + 1), n1);
    const CellT a2 = cell_of(__ldg(xs + 3 * src + 2), n2);
    double cf[PD];
#pragma unroll
    for (int j = 0; j < PD; ++j) cf[j] = poly[i * PD + j];
    const double s0 = fma(2.0, a0.t, -1.0), s1 = fma(2.0, a1.t, -1.0), s2 = fma(2.0, a2.t, -1.0);
    double v0 = cf[PD - 1], v1 = cf[PD - 1], v2 = cf[PD - 1];
#pragma unroll
    for (int j = PD - 2; j >= 0; --j) {
      v0 = fma(v0, s0, cf[j]);
      v1 = fma(v1, s1, cf[j]);
      v2 = fma(v2, s2, cf[j]);
    }
    if (i == W - 1) {   // strict truncation |u - l| < m (Q4)
      if (a0.t == 0.0) v0 = 0.0;
      if (a1.t == 0.0) v1 = 0.0;
      if (a2.t == 0.0) v2 = 0.0;
    }
    out[R::kW0 + i] = v0;
    out[R::kW1 + i] = v1;
    out[R::kW2 + i] = v2;
    if (i == 0) {
      reinterpret_cast<int4*>(out)[0] = make_int4(a1.c, a2.c, 0, 0);
      reinterpret_cast<double2*>(out)[1] = fv;
      out[R::kW1 + W] = 0.0;
      out[R::kW2 + W] = 0.0;
    }
  }
  __syncthreads();
  const uint32_t npts = min((uint32_t)PB, count - kb);
  const int nchunk = (int)npts * R::kChunks16;
  const double2* sp = reinterpret_cast<const double2*>(stage);
  double2* gp = reinterpret_cast<double2*>(rec + (size_t)kb * R::kDoubles);
  for (int c = threadIdx.x; c < nchunk; c += blockDim.x) gp[c] = sp[c];
}

// c1 rows spanned by sorted points [g0, g1): binary search of the bin table (multi-group only).
__global__ void k_group_rows(const uint32_t* __restrict__ start, int64_t nbins, uint32_t g0, uint32_t g1,
                             int64_t bins_per_row, int* rows) {
  const int which = threadIdx.x;   // 0: first point, 1: last point
  if (which > 1) return;
  const uint32_t target = which == 0 ? g0 : g1 - 1;
  int64_t lo = 0, hi = nbins - 1;   // largest bin with start[bin] <= target
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) / 2;
    if (start[mid] <= target) lo = mid;
    else hi = mid - 1;
  }
  rows[which] = (int)(lo / bins_per_row);
}

// ------------------------------------------------------------------------------------------
// Warp-specialised persistent sweep.  NW consumer warps own the 4 x 8 sub-patches of the CTA's
// P1 x P2 patch; NP producer warps fetch tiles (patch x segment) from a global counter, look up
// the (plane, pencil) ranges and stage batches of records into an NS-stage shared-memory ring with
// cp.async.  Stages are handed over with mbarriers (full: producer threads arrive; empty: one
// arrival per consumer warp), so consumer warps never wait for each other or for global memory.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
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
  while (!ok) {
    __nanosleep(64);
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000)
        : "memory");
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
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void producer_bar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

struct BatchHdr {
  int B;      // records in the batch; -1 terminates
  int tile;   // tile id
  int end;    // 1: last batch of the tile (flush), 2: tile skipped in this group pass
  int pad;
};

template <int P1, int P2, int M_>
struct SweepLayout {
  static constexpr int NW = (P1 / kWR) * (P2 / kWC);   // consumer warps
  static constexpr int NP = 4;                          // producer warps
  static constexpr int NS = HPNFFT_SWEEP_NS;            // ring stages
  static constexpr int kThreads = (NW + NP) * 32;
};

template <int P1, int P2, int M_>
__global__ void __launch_bounds__(SweepLayout<P1, P2, M_>::kThreads, 1) k_spread_sweep(SweepParams prm) {
  using C = SweepCfg<P1, P2, M_>;
  using L = SweepLayout<P1, P2, M_>;
  using R = Rec<2 * M_>;
  constexpr int W = C::W;
  constexpr int NW = L::NW, NS = L::NS;
  constexpr int NPT = L::NP * 32;        // producer threads
  constexpr int NE = C::kEntries;
  constexpr int RD = R::kDoubles;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int cap = prm.cap;
  double* s_rec = reinterpret_cast<double*>(smem_raw);                            // [NS][cap][RD]
  uint64_t* s_full = reinterpret_cast<uint64_t*>(s_rec + (size_t)NS * cap * RD);  // [NS]
  uint64_t* s_empty = s_full + NS;                                                // [NS]
  BatchHdr* s_hdr = reinterpret_cast<BatchHdr*>(s_empty + NS);                    // [NS]
  uint16_t* s_step = reinterpret_cast<uint16_t*>(s_hdr + NS);                     // [NS][cap]
  uint32_t* s_list = reinterpret_cast<uint32_t*>(s_step + NS * cap + (NS * cap & 1));   // [NW][cap]
  uint32_t* s_idx = s_list + (size_t)NW * cap;                                    // [cap]  producer
  uint32_t* s_beg = s_idx + cap;                                                  // [NE]   producer
  uint32_t* s_off = s_beg + NE;                                                   // [NE]   producer
  uint32_t* s_misc = s_off + NE;                                                  // [16]   producer

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = prm.n0, n1 = prm.n1, n2 = prm.n2;
  const int npc = n2 / P2, npr = (n1 + P1 - 1) / P1;
  const int ntiles = npc * npr * prm.nseg;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], NW);
    }
  }
  __syncthreads();

  auto tile_geom = [&](int t, int& R0, int& C0, int& L0) {
    const int pc = t % npc;
    const int rest = t / npc;
    const int pr = rest % npr;
    const int segi = rest / npr;
    R0 = pr * P1;
    C0 = pc * P2;
    L0 = prm.plane_lo + segi * prm.seg;
  };
  // planes cur = L0 - m .. L0 + S' + m - 2 of a tile, S' = its segment length
  auto tile_steps = [&](int t) -> int {
    const int segi = (t / npc) / npr;
    return min(prm.seg, prm.plane_len - segi * prm.seg) + W - 1;
  };
  auto tile_skip = [&](int R0) -> bool {   // multi-group pass: rows of the tile miss the group
    if (!prm.accumulate) return false;
    const int row_lo = prm.rows[0], row_hi = prm.rows[1];
    const int lo = R0 - M_, hi = R0 + P1 + M_ - 2;
    bool hit = false;
    for (int sft = -n1; sft <= n1; sft += n1) hit |= !(hi + sft < row_lo || lo + sft > row_hi);
    return !hit;
  };

  if (warp >= NW) {
    // =============================== producer warps ===============================
    const int pt = tid - NW * 32;   // 0 .. NPT-1
    const int pw = pt >> 5;
    int stage = 0;
    uint32_t phase = 0;
    auto next_stage = [&]() {
      if (++stage == NS) {
        stage = 0;
        phase ^= 1u;
      }
    };
    for (;;) {
      if (pt == 0) s_misc[8] = (uint32_t)atomicAdd(prm.tile_counter, 1);
      producer_bar(NPT);
      const int t = (int)s_misc[8];
      producer_bar(NPT);
      if (t >= ntiles) break;
      int R0, C0, L0;
      tile_geom(t, R0, C0, L0);
      const int first = L0 - M_;
      const int nsteps = tile_steps(t);
      const bool skip = tile_skip(R0);
      if (!skip) {
        const int b2lo = (C0 - M_ >= 0) ? (C0 - M_) / kBinW : -((M_ - C0 + kBinW - 1) / kBinW);
        const int b2hi = (C0 + P2 + M_ - 2) / kBinW;
        const int nq = b2hi - b2lo + 1;
        const int np_used = C::kRows * nq;
        for (int ch0 = 0; ch0 < nsteps; ch0 += kChunk) {
          const int nch = min(kChunk, nsteps - ch0);
          const int ne = nch * np_used;
          const int per = (ne + NPT - 1) / NPT;
          const unsigned long long p0 = prm.prof ? clock64() : 0ull;
          // (plane, pencil) ranges clipped to the group, pencil-major: thread -> pencil, all planes
          // of the chunk (independent loads, consecutive bins); stored plane-major for the scan
          for (int pp = pt; pp < np_used; pp += NPT) {
            const int r = pp / nq, q = pp - r * nq;
            const int c1 = (R0 - M_ + r) & (n1 - 1);
            int b2 = (b2lo + q) % prm.nb2;
            if (b2 < 0) b2 += prm.nb2;
            const size_t pbase = ((size_t)c1 * prm.nb2 + b2) * n0;
            uint32_t lo[kChunk], hi[kChunk];
#pragma unroll
            for (int sidx = 0; sidx < kChunk; ++sidx) {
              if (sidx < nch) {
                const size_t bin = pbase + ((first + ch0 + sidx) & (n0 - 1));
                lo[sidx] = __ldg(prm.start + bin);
                hi[sidx] = __ldg(prm.start + bin + 1);
              }
            }
#pragma unroll
            for (int sidx = 0; sidx < kChunk; ++sidx) {
              if (sidx < nch) {
                const uint32_t l = max(lo[sidx], prm.g0), h = min(hi[sidx], prm.g1);
                s_beg[sidx * np_used + pp] = l - prm.g0;
                s_off[sidx * np_used + pp] = h > l ? h - l : 0u;
              }
            }
          }
          producer_bar(NPT);
          // exclusive scan in (plane-major, pencil-minor) order; thread owns entries [pt*per, +per)
          uint32_t local = 0;
          for (int k = 0; k < per; ++k) {
            const int e = pt * per + k;
            if (e < ne) local += s_off[e];
          }
          const uint32_t incl = warp_incl_scan(local, lane);
          if (lane == 31) s_misc[pw] = incl;
          producer_bar(NPT);
          uint32_t wbase = 0, total = 0;
#pragma unroll
          for (int w = 0; w < L::NP; ++w) {
            const uint32_t v = s_misc[w];
            wbase += (w < pw) ? v : 0u;
            total += v;
          }
          uint32_t run = wbase + incl - local;
          for (int k = 0; k < per; ++k) {
            const int e = pt * per + k;
            if (e >= ne) break;
            const uint32_t c = s_off[e];
            s_off[e] = run;
            run += c;
          }
          producer_bar(NPT);
          if (prm.prof && pt == 0) atomicAdd(prm.prof + 4, clock64() - p0);
          for (uint32_t b0 = 0; b0 < total; b0 += (uint32_t)cap) {
            const uint32_t b1 = min(total, b0 + (uint32_t)cap);
            const int B = (int)(b1 - b0);
            const unsigned long long p1 = prm.prof ? clock64() : 0ull;
            mbar_wait(&s_empty[stage], phase ^ 1u);
            const unsigned long long p2 = prm.prof ? clock64() : 0ull;
            if (pt == 0) mbar_expect_tx(&s_full[stage], (uint32_t)B * (uint32_t)(RD * sizeof(double)));
            producer_bar(NPT);
            // one TMA bulk copy per (plane, pencil) range: its records are contiguous in HBM and
            // land in consecutive batch slots
            uint16_t* stp = s_step + stage * cap;
            double* dst = s_rec + (size_t)stage * cap * RD;
            for (int k = 0; k < per; ++k) {
              const int e = pt * per + k;
              if (e >= ne) break;
              const uint32_t off = s_off[e];
              const uint32_t cnt = (e + 1 < ne ? s_off[e + 1] : total) - off;
              if (cnt == 0 || off >= b1 || off + cnt <= b0) continue;
              const uint32_t beg = s_beg[e];
              const uint32_t k0 = off < b0 ? b0 - off : 0u;
              const uint32_t k1 = min(cnt, b1 - off);
              const uint16_t step = (uint16_t)(ch0 + e / np_used);
              for (uint32_t kk = k0; kk < k1; ++kk) stp[off + kk - b0] = step;
              bulk_copy_g2s(dst + (size_t)(off + k0 - b0) * RD, prm.rec + (size_t)(beg + k0) * RD,
                            (k1 - k0) * (uint32_t)(RD * sizeof(double)), &s_full[stage]);
            }
            producer_bar(NPT);   // all copies issued and plane ids written
            if (prm.prof && pt == 0) {
              atomicAdd(prm.prof + 5, p2 - p1);
              atomicAdd(prm.prof + 6, clock64() - p2);
            }
            if (pt == 0) {
              s_hdr[stage] = BatchHdr{B, t, 0, 0};
              mbar_arrive(&s_full[stage]);
            }
            next_stage();
          }
        }
      }
      // end-of-tile marker (consumers flush every node of the tile unless it is skipped)
      mbar_wait(&s_empty[stage], phase ^ 1u);
      if (pt == 0) {
        s_hdr[stage] = BatchHdr{0, t, skip ? 2 : 1, 0};
        mbar_arrive(&s_full[stage]);
      }
      next_stage();
    }
    mbar_wait(&s_empty[stage], phase ^ 1u);
    if (pt == 0) {
      s_hdr[stage] = BatchHdr{-1, -1, 0, 0};
      mbar_arrive(&s_full[stage]);
    }
    return;
  }

  // =============================== consumer warps ===============================
#ifndef HPNFFT_SWEEP_DFMA
  // FP64 tensor-core consumer (DMMA m8n8k4).  A warp owns a 4 x 4 sub-patch of columns; its
  // accumulator is the 16 x 32 real matrix C[node row][2 x complex column] held as 2 x 4 DMMA
  // C-fragments.  Node rows are cyclic (row = l0-node mod 16), so the 2m-node sliding window needs
  // no data movement: a finished node row is stored and zeroed.  Four records per k-step:
  //   C += A (16 x 4: w0 of each record placed at its plane's cyclic offset)
  //      x B (4 x 64: f w1[i1] w2[i2] of each record for every column, 0 outside its footprint)
  // i.e. 8 DMMA (2048 FMA) per k-step instead of 4 x 24 DFMA per lane; records of up to
  // 16 - 2m + 1 consecutive planes share a k-step.
  static_assert(2 * M_ <= 16, "cyclic 16-row window");
  const int wr_off = (warp / (P2 / kWC)) * kWR;
  const int wc_off = (warp % (P2 / kWC)) * kWC;
  const int g = lane >> 2, t = lane & 3;
  constexpr int NT = kWR * kWC / 4;       // n-tiles of 8 real columns (4 complex)
  const int part = g & 1;                 // B: real (0) or imaginary (1) part of the column
  const int bc0 = g >> 1;                 // B: column c of complex column q = 4 nt + g/2 (row nt)
  int cur_tile = -1;
  int first = 0, wr0 = 0, wc0 = 0, nsteps = 0;
  double cfr[2][NT][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) cfr[a][b][0] = cfr[a][b][1] = 0.0;
  int cur = 0;                            // planes < cur are flushed
  const size_t plane = (size_t)n1 * n2;

  auto flush_plane = [&](int sp) {        // plane sp (relative) done: node sp - m + 1 is final
    const int rho = (sp - M_ + 1) & 15;
    const bool mine = g == (rho & 7);
    const bool write = sp >= W - 1;
    const int l0 = (first + sp - M_ + 1) & (n0 - 1);
    double2* base = reinterpret_cast<double2*>(prm.grid) + (size_t)l0 * plane;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double v0, v1;
      if (rho < 8) { v0 = cfr[0][nt][0]; v1 = cfr[0][nt][1]; }
      else { v0 = cfr[1][nt][0]; v1 = cfr[1][nt][1]; }
      const int q = 4 * nt + t;           // complex column of this lane's pair (re, im)
      const int l1 = wr0 + q / kWC, l2 = wc0 + q % kWC;
      if (mine && write && l1 < n1) {
        double2* dst = base + (size_t)l1 * n2 + l2;
        if (prm.accumulate) {
          double2 o = *dst;
          o.x += v0;
          o.y += v1;
          *dst = o;
        } else {
          *dst = make_double2(v0, v1);
        }
      }
      if (mine) {
        if (rho < 8) { cfr[0][nt][0] = 0.0; cfr[0][nt][1] = 0.0; }
        else { cfr[1][nt][0] = 0.0; cfr[1][nt][1] = 0.0; }
      }
    }
  };
  auto advance = [&](int upto) {
    while (cur < upto) {
      flush_plane(cur);
      ++cur;
    }
  };

  int stage = 0;
  uint32_t phase = 0;
  unsigned long long tw = 0, tl = 0, tf = 0, tA = 0;
  for (;;) {
    const unsigned long long c0 = prm.prof ? clock64() : 0ull;
    mbar_wait(&s_full[stage], phase);
    const unsigned long long c1 = prm.prof ? clock64() : 0ull;
    const BatchHdr hdr = s_hdr[stage];
    if (hdr.B < 0) break;
    if (hdr.tile != cur_tile) {
      cur_tile = hdr.tile;
      int R0, C0, L0;
      tile_geom(cur_tile, R0, C0, L0);
      first = L0 - M_;
      nsteps = tile_steps(cur_tile);
      wr0 = R0 + wr_off;
      wc0 = C0 + wc_off;
      cur = 0;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) cfr[a][b][0] = cfr[a][b][1] = 0.0;
    }
    const int B = hdr.B;
    const double* recs = s_rec + (size_t)stage * cap * RD;
    const uint16_t* stp = s_step + stage * cap;
    // ---- plane-ordered list: entry = record | plane << 9 | d1 << 18 | d2 << 23 with
    //      d1 = wr0 - (c1-m+1) + 3 < 2m + 3, d2 = wc0 - (c2-m+1) + 7 < 2m + 7 ----
    int nlist = 0;
    uint32_t* my = s_list + (size_t)warp * cap;
    for (int base = 0; base < B; base += 32) {
      const int e = base + lane;
      bool rel = false;
      uint32_t entry = 0;
      if (e < B) {
        const int2 cc = *reinterpret_cast<const int2*>(recs + (size_t)e * RD);
        const uint32_t d1 = (uint32_t)((wr0 - (cc.x - M_ + 1) + (kWR - 1)) & (n1 - 1));
        const uint32_t d2 = (uint32_t)((wc0 - (cc.y - M_ + 1) + (kWC - 1)) & (n2 - 1));
        rel = (d1 < (uint32_t)(W + kWR - 1)) && (d2 < (uint32_t)(W + kWC - 1));
        entry = (uint32_t)e | ((uint32_t)stp[e] << 9) | (d1 << 18) | (d2 << 23);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) my[nlist + __popc(bal & ((1u << lane) - 1))] = entry;
      nlist += __popc(bal);
    }
    __syncwarp();
    const unsigned long long c2 = prm.prof ? clock64() : 0ull;
    // ---- k-steps of up to 4 records spanning at most 16 - 2m + 1 planes ----
    for (int k = 0; k < (prm.debug == 2 ? 0 : nlist);) {
      const uint32_t e0 = my[k];
      const int st0 = (int)((e0 >> 9) & 0x1ffu);
      const uint32_t en = (k + t < nlist) ? my[k + t] : 0xffffffffu;
      const int st = (int)((en >> 9) & 0x1ffu);
      const bool ok = (k + t < nlist) && (st - st0 <= 16 - W);
      const unsigned okm = __ballot_sync(0xffffffffu, ok) & 0xfu;   // lanes 0..3 decide
      const int cnt = __popc(okm);                                  // prefix by plane order
      advance(st0);
      // this lane's record: k + t (lanes with t >= cnt contribute zeros)
      const bool act = t < cnt;
      const double* r = recs + (size_t)(act ? (en & 0x1ffu) : 0u) * RD;
      const int d1 = (int)((en >> 18) & 31u), d2 = (int)((en >> 23) & 31u);
      // A fragments: rows 8 mt + g hold node (row - (st - m + 1)) mod 16 of this record
      double afr[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int i = (8 * mt + g - (st - M_ + 1)) & 15;
        afr[mt] = (act && i < W) ? r[R::kW0 + i] : 0.0;
      }
      // B fragments: complex column q = 4 nt + g/2 = (row nt, col g/2) of the 4 x 4 sub-patch,
      // part g & 1; value f_part w1[i1(nt)] w2[i2(g/2)]
      const double fp = act ? r[2 + part] : 0.0;
      const unsigned i2 = min((unsigned)(d2 - (kWC - 1) + bc0), (unsigned)W);
      const double fw2 = fp * r[R::kW2 + i2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const unsigned i1 = min((unsigned)(d1 - (kWR - 1) + nt), (unsigned)W);
        const double bfr = fw2 * r[R::kW1 + i1];
        if (prm.debug == 1) {   // measurement only: keep the operands alive, skip the MMAs
          cfr[0][nt][0] += afr[0] * bfr;
          continue;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
              : "+d"(cfr[mt][nt][0]), "+d"(cfr[mt][nt][1])
              : "d"(afr[mt]), "d"(bfr));
        }
      }
      k += cnt;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[stage]);
    const unsigned long long c3 = prm.prof ? clock64() : 0ull;
    if (hdr.end == 1) advance(nsteps);   // tile finished: flush the remaining nodes
    if (hdr.end == 2) cur = nsteps;      // tile skipped in a multi-group pass: nothing to write
    if (prm.prof) {
      tw += c1 - c0;
      tl += c2 - c1;
      tf += c3 - c2;
      tA += clock64() - c3;
    }
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
#else
  const int wr_off = (warp / (P2 / kWC)) * kWR;
  const int wc_off = (warp % (P2 / kWC)) * kWC;
  int cur_tile = -1;
  int first = 0, wr0 = 0, wc0 = 0, lo1 = 0, lo2 = 0, nsteps = 0;
  bool valid = true;
  double2* gcol = nullptr;
  const size_t plane = (size_t)n1 * n2;
  double2 acc[W];
#pragma unroll
  for (int i = 0; i < W; ++i) acc[i] = make_double2(0.0, 0.0);
  int cur = 0;

  auto advance = [&](int upto) {
    while (cur < upto) {
      if (cur >= W - 1 && valid) {
        const int l0 = (first + cur - M_ + 1) & (n0 - 1);
        double2* dst = gcol + (size_t)l0 * plane;
        if (prm.accumulate) {
          double2 o = *dst;
          o.x += acc[0].x;
          o.y += acc[0].y;
          *dst = o;
        } else {
          *dst = acc[0];
        }
      }
#pragma unroll
      for (int i = 0; i < W - 1; ++i) acc[i] = acc[i + 1];
      acc[W - 1] = make_double2(0.0, 0.0);
      ++cur;
    }
  };

  int stage = 0;
  uint32_t phase = 0;
  unsigned long long tw = 0, tl = 0, tf = 0, tA = 0;
  for (;;) {
    const unsigned long long c0 = prm.prof ? clock64() : 0ull;
    mbar_wait(&s_full[stage], phase);
    const unsigned long long c1 = prm.prof ? clock64() : 0ull;
    const BatchHdr hdr = s_hdr[stage];
    if (hdr.B < 0) break;
    if (hdr.tile != cur_tile) {
      cur_tile = hdr.tile;
      int R0, C0, L0;
      tile_geom(cur_tile, R0, C0, L0);
      first = L0 - M_;
      nsteps = tile_steps(cur_tile);
      wr0 = R0 + wr_off;
      wc0 = C0 + wc_off;
      const int l1 = wr0 + lane / kWC;
      const int l2 = wc0 + lane % kWC;
      valid = l1 < n1;   // ghost rows of the last row tile when P1 does not divide n1
      lo1 = l1 + M_ - 1;
      lo2 = l2 + M_ - 1;
      gcol = reinterpret_cast<double2*>(prm.grid) + (size_t)(l1 & (n1 - 1)) * n2 + l2;
      cur = 0;
#pragma unroll
      for (int i = 0; i < W; ++i) acc[i] = make_double2(0.0, 0.0);
    }
    const int B = hdr.B;
    const double* recs = s_rec + (size_t)stage * cap * RD;
    const uint16_t* stp = s_step + stage * cap;
    // ---- this warp's plane-ordered list of records touching its 4 x 8 sub-patch ----
    int nlist = 0;
    uint32_t* my = s_list + (size_t)warp * cap;
    for (int base = 0; base < B; base += 32) {
      const int e = base + lane;
      bool rel = false;
      if (e < B) {
        const int2 cc = *reinterpret_cast<const int2*>(recs + (size_t)e * RD);
        const int d1 = (wr0 - (cc.x - M_ + 1) + (kWR - 1)) & (n1 - 1);
        const int d2 = (wc0 - (cc.y - M_ + 1) + (kWC - 1)) & (n2 - 1);
        rel = (d1 < W + kWR - 1) && (d2 < W + kWC - 1);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, rel);
      if (rel) my[nlist + __popc(bal & ((1u << lane) - 1))] = (uint32_t)e | ((uint32_t)stp[e] << 16);
      nlist += __popc(bal);
    }
    __syncwarp();
    const unsigned long long c2 = prm.prof ? clock64() : 0ull;
    // ---- apply the records plane by plane (pairs of records share one pass over w0) ----
    if (nlist > 0) {
      auto coef = [&](int e, double& cr, double& ci) {
        const double* r = recs + (size_t)e * RD;
        const int2 cc = *reinterpret_cast<const int2*>(r);
        const unsigned i1 = min((unsigned)((lo1 - cc.x) & (n1 - 1)), (unsigned)W);
        const unsigned i2 = min((unsigned)((lo2 - cc.y) & (n2 - 1)), (unsigned)W);
        const double2 fv = *reinterpret_cast<const double2*>(r + 2);
        const double w12 = r[R::kW1 + i1] * r[R::kW2 + i2];
        cr = fv.x * w12;
        ci = fv.y * w12;
      };
      int k = 0;
      uint32_t ent = my[0];
      while (k < nlist) {
        const int st = (int)(ent >> 16);
        advance(st);
        for (;;) {
          const int ea = (int)(ent & 0xffffu);
          ++k;
          ent = (k < nlist) ? my[k] : 0xffffffffu;
          const bool pair = (int)(ent >> 16) == st && k < nlist;
          const int eb = pair ? (int)(ent & 0xffffu) : ea;
          if (pair) {
            ++k;
            ent = (k < nlist) ? my[k] : 0xffffffffu;
          }
          double ar, ai, br, bi;
          coef(ea, ar, ai);
          coef(eb, br, bi);
          if (!pair) {
            br = 0.0;
            bi = 0.0;
          }
          const double* wa = recs + (size_t)ea * RD + R::kW0;
          const double* wb = recs + (size_t)eb * RD + R::kW0;
#pragma unroll
          for (int i = 0; i < W; i += 2) {
            const double2 xa = *reinterpret_cast<const double2*>(wa + i);
            const double2 xb = *reinterpret_cast<const double2*>(wb + i);
            acc[i].x = fma(br, xb.x, fma(ar, xa.x, acc[i].x));
            acc[i].y = fma(bi, xb.x, fma(ai, xa.x, acc[i].y));
            acc[i + 1].x = fma(br, xb.y, fma(ar, xa.y, acc[i + 1].x));
            acc[i + 1].y = fma(bi, xb.y, fma(ai, xa.y, acc[i + 1].y));
          }
          if (!((int)(ent >> 16) == st && k < nlist)) break;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_empty[stage]);
    const unsigned long long c3 = prm.prof ? clock64() : 0ull;
    if (hdr.end == 1) advance(nsteps);   // tile finished: flush the remaining nodes
    if (hdr.end == 2) cur = nsteps;      // tile skipped in a multi-group pass: nothing to write
    if (prm.prof) {
      tw += c1 - c0;
      tl += c2 - c1;
      tf += c3 - c2;
      tA += clock64() - c3;
    }
    if (++stage == NS) {
      stage = 0;
      phase ^= 1u;
    }
  }
#endif
  if (prm.prof && lane == 0) {
    atomicAdd(prm.prof + 0, tw);
    atomicAdd(prm.prof + 1, tl);
    atomicAdd(prm.prof + 2, tf);
    atomicAdd(prm.prof + 3, tA);
    atomicAdd(prm.prof + 7, 1ull);
  }
}

namespace {

template <int P1, int P2, int M_>
size_t sweep_smem_bytes(int cap) {
  using C = SweepCfg<P1, P2, M_>;
  using L = SweepLayout<P1, P2, M_>;
  size_t b = 0;
  b += sizeof(double) * (size_t)L::NS * cap * Rec<2 * M_>::kDoubles;
  b += (sizeof(uint64_t) * 2 + sizeof(BatchHdr)) * L::NS;
  b += sizeof(uint16_t) * (L::NS * cap + 1);
  b += sizeof(uint32_t) * ((size_t)L::NW * cap);
  b += sizeof(uint32_t) * cap;
  b += sizeof(uint32_t) * (2 * C::kEntries + 16);
  return b + 64;
}

// CTA patch variant: 0 = 12 x 32 (12 consumer + 4 producer warps), 1 = 8 x 32 (8 + 4 warps).
// CTA patch variant: 0 = 12 x 32, 1 = 8 x 32, 2 = 16 x 32 columns (consumer warps = patch / warp
// sub-patch), each with 4 producer warps; HPNFFT_SWEEP_PATCH = "12x32" | "8x32" | "16x32".
int sweep_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HPNFFT_SWEEP_PATCH");
    if (e && e[0] == '8') v = 1;
    else if (e && e[0] == '1' && e[1] == '6') v = 2;
    else if (e && e[0] == '1' && e[1] == '2') v = 0;
    else v = 0;
  }
  return v;
}

template <int P1, int P2, int M_>
int launch_sweep_group(Plan* p, uint32_t g0, uint32_t g1, const int* rows, bool accumulate) {
  using L = SweepLayout<P1, P2, M_>;
  const size_t smem_max = (size_t)(226 * 1024);
  int cap = 64;
  while (sweep_smem_bytes<P1, P2, M_>(cap + 64) <= smem_max) cap += 64;
  const size_t smem = sweep_smem_bytes<P1, P2, M_>(cap);
  SweepParams prm;
  prm.rec = p->rec;
  prm.start = p->bin_count;
  prm.grid = p->grid;
  prm.rows = rows;
  prm.g0 = g0;
  prm.g1 = g1;
  prm.accumulate = accumulate ? 1 : 0;
  prm.n0 = (int)p->n[0];
  prm.n1 = (int)p->n[1];
  prm.n2 = (int)p->n[2];
  prm.nb2 = (int)(p->n[2] / kBinW);
  prm.plane_lo = (int)p->plane_lo;
  prm.plane_len = (int)p->plane_len;
  prm.seg = (int)(p->plane_len < 256 ? p->plane_len : 256);
  prm.nseg = (int)((p->plane_len + prm.seg - 1) / prm.seg);
  prm.cap = cap;
  prm.tile_counter = p->tile_counter;
  static const bool prof_on = getenv("HPNFFT_SWEEP_PROF") != nullptr;
  unsigned long long* prof = nullptr;
  if (prof_on) {
    cudaMalloc(&prof, 8 * sizeof(unsigned long long));
    cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), p->stream);
  }
  prm.prof = prof;
  static const int dbg = getenv("HPNFFT_SWEEP_DEBUG") ? atoi(getenv("HPNFFT_SWEEP_DEBUG")) : 0;
  prm.debug = dbg;
  HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->tile_counter, 0, sizeof(int), p->stream), "tile counter");
  auto kern = k_spread_sweep<P1, P2, M_>;
  HPNFFT_CUDA_TRY(p, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                  "sweep smem attr");
  const int64_t tiles = ((p->n[1] + P1 - 1) / P1) * (p->n[2] / P2) * prm.nseg;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t blocks = tiles < (int64_t)sms ? tiles : (int64_t)sms;
  kern<<<(unsigned)blocks, L::kThreads, smem, p->stream>>>(prm);
  p->launches++;
  if (prof) {
    unsigned long long h[8];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, p->stream);
    cudaStreamSynchronize(p->stream);
    double nw = (double)h[7];
    fprintf(stderr,
            "[sweep prof] cap=%d consumer warps=%.0f  per warp Mcycles: wait_full %.2f  lists %.2f  apply %.2f  "
            "advance %.2f | producer (thread 0 sums, Mcycles): lookups+scan %.2f  wait_empty %.2f  copy %.2f\n",
            cap, nw, h[0] / nw / 1e6, h[1] / nw / 1e6, h[2] / nw / 1e6, h[3] / nw / 1e6, h[4] / blocks / 1e6,
            h[5] / blocks / 1e6, h[6] / blocks / 1e6);
    cudaFree(prof);
  }
  return check_launch(p, "spread_sweep");
}

template <int M_>
int run_sweep(Plan* p, const double* f) {
  const uint32_t M = (uint32_t)p->M;
  const uint32_t G = (uint32_t)p->rec_group;
  const bool multi = M > G;
  if (multi) {
    const size_t bytes = sizeof(double) * 2 * (size_t)(p->n[0] * p->n[1] * p->n[2]);
    HPNFFT_CUDA_TRY(p, cudaMemsetAsync(p->grid, 0, bytes, p->stream), "zero grid");
  }
  uint32_t g0 = 0;
  do {
    const uint32_t g1 = (M - g0) < G ? M : g0 + G;
    const uint32_t cnt = g1 - g0;
    if (cnt > 0) {
      stage_begin(p, 7);
      constexpr int PB = 256 / (2 * M_);
      k_point_records<M_><<<(unsigned)((cnt + PB - 1) / PB), 256, 0, p->stream>>>(
          p->xs, p->perm, f, p->poly, p->rec, g0, cnt, p->n[0], p->n[1], p->n[2]);
      p->launches++;
      int rc = check_launch(p, "point records");
      stage_end(p, 7);
      if (rc) return rc;
    }
    if (multi) {
      k_group_rows<<<1, 32, 0, p->stream>>>(p->bin_count, p->nbins, g0, g1, (p->n[2] / kBinW) * p->n[0],
                                            p->group_rows);
      p->launches++;
    }
    const int var = sweep_variant();
    int rc;
#ifdef HPNFFT_SWEEP_DFMA
    rc = var == 1 ? launch_sweep_group<8, 32, M_>(p, g0, g1, p->group_rows, multi)
       : var == 2 ? launch_sweep_group<16, 32, M_>(p, g0, g1, p->group_rows, multi)
                  : launch_sweep_group<12, 32, M_>(p, g0, g1, p->group_rows, multi);
#else
    // 4 x 4 warp sub-patches: 12 x 32 = 24 consumer warps, 8 x 32 = 16 (+ 4 producer warps)
    rc = var == 1 ? launch_sweep_group<8, 32, M_>(p, g0, g1, p->group_rows, multi)
                  : launch_sweep_group<12, 32, M_>(p, g0, g1, p->group_rows, multi);
#endif
    if (rc) return rc;
    g0 = g1;
  } while (g0 < M);
  return HPNFFT_OK;
}

}  // namespace

size_t record_bytes(int m) { return sizeof(double) * (6 + 3 * 2 * m); }

bool sweep_supported(const Plan* p) {
  const int W = 2 * p->m;
  const int P1 = 12, P2 = 32;   // largest patch of any variant
  if (p->n[2] < P2 || p->n[1] < P1) return false;
  if (p->n[1] < P1 + W - 1) return false;                     // candidate rows must be distinct
  const int bins = (P2 + W - 1 + kBinW - 1) / kBinW + 1;      // candidate c2 bins must be distinct
  if (p->n[2] / kBinW < bins) return false;
  if (p->n[0] < W) return false;
  if (p->n[0] + W > 65535) return false;
  if (p->rec == nullptr || p->rec_group == 0) return false;
  return true;
}

int spread_sweep(Plan* p, const double* f) {
  switch (p->m) {
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
