// spread_sweep.cu -- the B200 spreading kernel (A3 + A4 of SURVEY.md §8(a)).
//
// Computes the "Spreading" step of CUNFFT (Fig. 1; §3)
//     g(l) = sum_j f_j * prod_t Phi(n_t x_jt - l_t),   l in I_n (periodic),
// without atomics and without a zero fill: every grid node is written exactly once.
//
// Design: a CTA owns a P1 x P2 patch of grid columns (l1, l2) and a segment
// of S planes along l0.  Each lane owns ONE column and keeps a sliding window of the 2m nodes
// l0 = cur-m+1 .. cur+m of that column in registers.  The CTA sweeps cur over the planes; all
// points whose cell c0 equals cur contribute to exactly the 2m window registers (static register
// indices, no dynamic addressing), so the 2(2m)^3 FMAs of a point become 2m FMA pairs per active
// lane.  After the points of plane cur are applied, node cur-m+1 is final and is stored once
// (coalesced: a warp covers 4 rows x 8 consecutive l2), then the window shifts by one plane.
// The points of plane cur are found through the bin table of sort.cu: bins are (c1 row, 8
// consecutive c2, c0 plane) with c0 fastest, so for each (row, c2-bin) "pencil" around the patch
// the points of plane cur are one contiguous range.  Per batch of planes the CTA stages the
// candidate points in shared memory: cell, t, f and the 3 x 2m tap weights (computed once per
// CTA from the window polynomials), and each warp compacts the records whose 2m x 2m footprint
// touches its 4 x 8 sub-patch into its own ordered list.
#include "spread_common.cuh"

namespace hpnfft {

namespace {

constexpr int kWR = 4;          // warp sub-patch: 4 rows (l1) x 8 cols (l2) = 32 lanes
constexpr int kWC = 8;
constexpr int kBinW = 8;        // c2 bin width of the sort keys (sort.cu)
constexpr int kChunk = 8;       // planes whose pencil ranges are looked up together

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
  const double* xs;        // sorted coordinates [M][3]
  const uint32_t* perm;    // sorted -> original
  const double* f;         // values, original order [M][2]
  const uint32_t* start;   // bin_start [nbins + 1]
  const double* poly;      // [2m][kPolyDeg+1]
  double* grid;            // [n0][n1][n2] complex
  int n0, n1, n2;
  int nb2;                 // n2 / 8
  int seg;                 // S: planes per segment
  int nseg;                // n0 / S
  int cap;                 // record capacity of the shared-memory batch
};

}  // namespace

template <int P1, int P2, int M_>
__global__ void __launch_bounds__(SweepCfg<P1, P2, M_>::kThreads, 1) k_spread_sweep(SweepParams prm) {
  using C = SweepCfg<P1, P2, M_>;
  constexpr int W = C::W;
  constexpr int NT = C::kThreads;
  constexpr int NP = C::kPencils;
  constexpr int NE = C::kEntries;
  constexpr int NW = C::kWarps;
  constexpr int PD = kPolyDeg + 1;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  // ---- shared-memory carve-up ----
  double* s_poly = reinterpret_cast<double*>(smem_raw);                 // [W][PD]
  double* s_w = s_poly + W * PD;                                        // [cap][3][W] weights
  double2* s_f = reinterpret_cast<double2*>(s_w + (size_t)prm.cap * 3 * W);   // [cap]
  double* s_t = reinterpret_cast<double*>(s_f + prm.cap);               // [cap][3]
  int* s_c = reinterpret_cast<int*>(s_t + (size_t)prm.cap * 3);         // [cap][2] (c1, c2)
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_c + (size_t)prm.cap * 2);   // [cap] sorted point index
  uint16_t* s_step = reinterpret_cast<uint16_t*>(s_idx + prm.cap);      // [cap] plane (relative)
  uint16_t* s_list = s_step + prm.cap;                                  // [NW][cap] per-warp lists
  uint32_t* s_beg = reinterpret_cast<uint32_t*>(s_list + (size_t)NW * prm.cap + ((NW * prm.cap) & 1));
  uint32_t* s_off = s_beg + NE;                                         // exclusive offsets
  uint32_t* s_misc = s_off + NE;                                        // [32] scan scratch + totals

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = prm.n0, n1 = prm.n1, n2 = prm.n2;

  // CTA -> (patch row block, patch col block, segment)
  const int npc = n2 / P2;
  const int npr = n1 / P1;
  int b = blockIdx.x;
  const int segi = b % prm.nseg;
  b /= prm.nseg;
  const int pc = b % npc;
  const int pr = b / npc;
  (void)npr;
  const int R0 = pr * P1, C0 = pc * P2;
  const int L0 = segi * prm.seg;
  const int nsteps = prm.seg + W - 1;            // planes cur = L0 - m .. L0 + S + m - 2
  const int first = L0 - M_;

  // this lane's column
  const int wr0 = R0 + (warp / (P2 / kWC)) * kWR;
  const int wc0 = C0 + (warp % (P2 / kWC)) * kWC;
  const int l1 = wr0 + lane / kWC;
  const int l2 = wc0 + lane % kWC;

  // candidate pencils: rows c1 = R0 - m + r (r < kRows), bins b2 = b2lo + q (q < nq)
  const int b2lo = (C0 - M_ >= 0) ? (C0 - M_) / kBinW : -((M_ - C0 + kBinW - 1) / kBinW);
  const int b2hi = (C0 + P2 + M_ - 2) / kBinW;
  const int nq = b2hi - b2lo + 1;
  const int np_used = C::kRows * nq;

  for (int e = tid; e < W * PD; e += NT) s_poly[e] = prm.poly[e];

  double2 acc[W];
#pragma unroll
  for (int i = 0; i < W; ++i) acc[i] = make_double2(0.0, 0.0);
  int cur = 0;   // relative plane of the window (warp-uniform)

  // flush node of plane `cur` (relative) and shift the window by one plane
  auto advance = [&](int upto) {
    while (cur < upto) {
      if (cur >= W - 1) {
        int l0 = (first + cur - M_ + 1) & (n0 - 1);
        reinterpret_cast<double2*>(prm.grid)[((size_t)l0 * n1 + l1) * n2 + l2] = acc[0];
      }
#pragma unroll
      for (int i = 0; i < W - 1; ++i) acc[i] = acc[i + 1];
      acc[W - 1] = make_double2(0.0, 0.0);
      ++cur;
    }
  };

  for (int ch0 = 0; ch0 < nsteps; ch0 += kChunk) {
    const int nch = min(kChunk, nsteps - ch0);
    // ---- A: (plane, pencil) ranges of this chunk ----
    __syncthreads();
    for (int e = tid; e < kChunk * np_used; e += NT) {
      int s = e / np_used, p = e % np_used;
      uint32_t beg = 0, cnt = 0;
      if (s < nch) {
        int r = p / nq, q = p % nq;
        int c1 = (R0 - M_ + r) & (n1 - 1);
        int b2 = (b2lo + q) % prm.nb2;
        if (b2 < 0) b2 += prm.nb2;
        int c0 = (first + ch0 + s) & (n0 - 1);
        size_t bin = ((size_t)c1 * prm.nb2 + b2) * n0 + c0;
        beg = __ldg(prm.start + bin);
        cnt = __ldg(prm.start + bin + 1) - beg;
      }
      s_beg[e] = beg;
      s_off[e] = cnt;
    }
    __syncthreads();
    // exclusive scan of the counts in (plane-major, pencil-minor) order
    {
      const int ne = kChunk * np_used;
      const int per = (ne + NT - 1) / NT;
      uint32_t local = 0;
      for (int k = 0; k < per; ++k) {
        int e = tid * per + k;
        if (e < ne) local += s_off[e];
      }
      uint32_t incl = warp_incl_scan(local, lane);
      if (lane == 31) s_misc[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        uint32_t v = (lane < NW) ? s_misc[lane] : 0u;
        uint32_t vi = warp_incl_scan(v, lane);
        if (lane < NW) s_misc[lane] = vi - v;
        if (lane == 31) s_misc[32] = vi;
      }
      __syncthreads();
      uint32_t run = s_misc[warp] + incl - local;
      for (int k = 0; k < per; ++k) {
        int e = tid * per + k;
        if (e < ne) {
          uint32_t c = s_off[e];
          s_off[e] = run;
          run += c;
        }
      }
    }
    __syncthreads();
    const uint32_t total = s_misc[32];

    for (uint32_t b0 = 0; b0 < total; b0 += prm.cap) {
      const uint32_t b1 = min(total, b0 + (uint32_t)prm.cap);
      const int B = (int)(b1 - b0);
      // ---- B: record -> sorted point index and plane ----
      {
        const int ne = kChunk * np_used;
        const int per = (ne + NT - 1) / NT;
        for (int k = 0; k < per; ++k) {
          int e = tid * per + k;
          if (e >= ne) break;
          uint32_t off = s_off[e];
          uint32_t cnt = (e + 1 < ne ? s_off[e + 1] : total) - off;
          if (cnt == 0 || off >= b1 || off + cnt <= b0) continue;
          uint32_t beg = s_beg[e];
          uint32_t k0 = off < b0 ? b0 - off : 0u;
          uint32_t k1 = min(cnt, b1 - off);
          uint16_t step = (uint16_t)(ch0 + e / np_used);
          for (uint32_t kk = k0; kk < k1; ++kk) {
            s_idx[off + kk - b0] = beg + kk;
            s_step[off + kk - b0] = step;
          }
        }
      }
      __syncthreads();
      // ---- C: per record cell, t, f ----
      for (int e = tid; e < B; e += NT) {
        uint32_t k = s_idx[e];
        CellT a0 = cell_of(__ldg(prm.xs + 3 * (size_t)k), n0);
        CellT a1 = cell_of(__ldg(prm.xs + 3 * (size_t)k + 1), n1);
        CellT a2 = cell_of(__ldg(prm.xs + 3 * (size_t)k + 2), n2);
        (void)a0.c;
        s_t[3 * e] = a0.t;
        s_t[3 * e + 1] = a1.t;
        s_t[3 * e + 2] = a2.t;
        s_c[2 * e] = a1.c;
        s_c[2 * e + 1] = a2.c;
        uint32_t src = __ldg(prm.perm + k);
        s_f[e] = __ldg(reinterpret_cast<const double2*>(prm.f) + src);
      }
      __syncthreads();
      // ---- D: tap weights (w0 all taps; w1/w2 only taps landing inside the patch) ----
      for (int e = tid; e < B * 3 * W; e += NT) {
        int rec = e / (3 * W), r = e % (3 * W), d = r / W, i = r % W;
        bool need = true;
        if (d == 1) {
          int l = (s_c[2 * rec] - M_ + 1 + i - R0) & (n1 - 1);
          need = l < P1;
        } else if (d == 2) {
          int l = (s_c[2 * rec + 1] - M_ + 1 + i - C0) & (n2 - 1);
          need = l < P2;
        }
        if (need) s_w[(size_t)rec * 3 * W + d * W + i] = tap_weight(s_poly, i, s_t[3 * rec + d], M_);
      }
      __syncthreads();
      // ---- E: this warp's ordered list of records touching its 4 x 8 sub-patch ----
      int nlist = 0;
      uint16_t* my = s_list + (size_t)warp * prm.cap;
      for (int base = 0; base < B; base += 32) {
        int e = base + lane;
        bool rel = false;
        if (e < B) {
          int c1 = s_c[2 * e], c2 = s_c[2 * e + 1];
          int d1 = (wr0 - (c1 - M_ + 1) + (kWR - 1)) & (n1 - 1);
          int d2 = (wc0 - (c2 - M_ + 1) + (kWC - 1)) & (n2 - 1);
          rel = (d1 < W + kWR - 1) && (d2 < W + kWC - 1);
        }
        unsigned bal = __ballot_sync(0xffffffffu, rel);
        if (rel) my[nlist + __popc(bal & ((1u << lane) - 1))] = (uint16_t)e;
        nlist += __popc(bal);
      }
      __syncwarp();
      // ---- F: apply the records to the register windows ----
      for (int k = 0; k < nlist; ++k) {
        int e = my[k];
        advance((int)s_step[e]);
        int c1 = s_c[2 * e], c2 = s_c[2 * e + 1];
        unsigned i1 = (unsigned)((l1 - c1 + M_ - 1) & (n1 - 1));
        unsigned i2 = (unsigned)((l2 - c2 + M_ - 1) & (n2 - 1));
        if (i1 < (unsigned)W && i2 < (unsigned)W) {
          const double* w = s_w + (size_t)e * 3 * W;
          double2 fv = s_f[e];
          double w12 = w[W + i1] * w[2 * W + i2];
          double cr = fv.x * w12, ci = fv.y * w12;
#pragma unroll
          for (int i = 0; i < W; ++i) {
            double w0 = w[i];
            acc[i].x = fma(cr, w0, acc[i].x);
            acc[i].y = fma(ci, w0, acc[i].y);
          }
        }
      }
      __syncthreads();
    }
  }
  advance(nsteps);
}

namespace {

template <int P1, int P2, int M_>
size_t sweep_smem_bytes(int cap) {
  using C = SweepCfg<P1, P2, M_>;
  size_t b = 0;
  b += sizeof(double) * C::W * (kPolyDeg + 1);
  b += sizeof(double) * (size_t)cap * 3 * C::W;
  b += sizeof(double2) * cap;
  b += sizeof(double) * (size_t)cap * 3;
  b += sizeof(int) * (size_t)cap * 2;
  b += sizeof(uint32_t) * cap;
  b += sizeof(uint16_t) * cap;
  b += sizeof(uint16_t) * ((size_t)C::kWarps * cap + 1);
  b += sizeof(uint32_t) * (2 * C::kEntries + 40);
  return b + 64;
}

template <int P1, int P2, int M_>
int launch_sweep(Plan* p, const double* f) {
  using C = SweepCfg<P1, P2, M_>;
  const size_t smem_max = 227 * 1024;
  // largest record capacity that fits the shared memory
  int cap = 64;
  while (sweep_smem_bytes<P1, P2, M_>(cap + 64) <= smem_max) cap += 64;
  size_t smem = sweep_smem_bytes<P1, P2, M_>(cap);
  SweepParams prm;
  prm.xs = p->xs;
  prm.perm = p->perm;
  prm.f = f;
  prm.start = p->bin_count;
  prm.poly = p->poly;
  prm.grid = p->grid;
  prm.n0 = (int)p->n[0];
  prm.n1 = (int)p->n[1];
  prm.n2 = (int)p->n[2];
  prm.nb2 = (int)(p->n[2] / kBinW);
  prm.seg = (int)(p->n[0] < 256 ? p->n[0] : 256);
  prm.nseg = (int)(p->n[0] / prm.seg);
  prm.cap = cap;
  auto kern = k_spread_sweep<P1, P2, M_>;
  HPNFFT_CUDA_TRY(p, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                  "sweep smem attr");
  int64_t blocks = (p->n[1] / P1) * (p->n[2] / P2) * prm.nseg;
  kern<<<(unsigned)blocks, C::kThreads, smem, p->stream>>>(prm);
  p->launches++;
  return check_launch(p, "spread_sweep");
}

constexpr int kP1 = 16, kP2 = 32;

}  // namespace

bool sweep_supported(const Plan* p) {
  const int W = 2 * p->m;
  if (p->n[2] < kP2 || p->n[1] < kP1) return false;
  if (p->n[1] < kP1 + W - 1) return false;                    // candidate rows must be distinct
  int b2lo_span = (kP2 + W - 1 + kBinW - 1) / kBinW + 1;      // candidate c2 bins must be distinct
  if (p->n[2] / kBinW < b2lo_span) return false;
  if (p->n[0] < W) return false;
  if (p->n[0] > 65535) return false;
  return true;
}

int spread_sweep(Plan* p, const double* f) {
  switch (p->m) {
    case 2: return launch_sweep<kP1, kP2, 2>(p, f);
    case 3: return launch_sweep<kP1, kP2, 3>(p, f);
    case 4: return launch_sweep<kP1, kP2, 4>(p, f);
    case 5: return launch_sweep<kP1, kP2, 5>(p, f);
    case 6: return launch_sweep<kP1, kP2, 6>(p, f);
    case 7: return launch_sweep<kP1, kP2, 7>(p, f);
    case 8: return launch_sweep<kP1, kP2, 8>(p, f);
    default:
      set_error("m not supported by the sweep kernel");
      return HPNFFT_E_UNSUPPORTED;
  }
}

}  // namespace hpnfft
