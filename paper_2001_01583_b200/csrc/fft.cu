// fft.cu -- A5 + A6 of SURVEY.md §8(a): the d-dimensional FFT of the oversampled grid
// (the "FFT" step of CUNFFT, §3) and the fused "Scaling" step
// (deconvolve + crop to I_N).
//
// ghat(k) = sum_{l in I_n} g(l) exp(-2 pi i k.l/n), unnormalised, only k in I_N kept.
// Three batched, output-pruned 1-D passes (HBM bound):
//   pass z : g[n0][n1][n2]  -> A[n0][n1][N2]   (contiguous lines)
//   pass y : A[n0][n1][N2]  -> B[n0][N1][N2]   (lines strided by N2)
//   pass x : B[n0][N1][N2]  -> F[N0][N1][N2]   (lines strided by N1 N2)
// Output index k' = k + N/2 in [0, N) reads grid frequency (k mod n); each pass multiplies by
// its dimension's 1/c_k (so after pass x, F = ghat / (c_k0 c_k1 c_k2) = fhat).
// In-CTA transform: Stockham autosort, radix 8/4/2 stages over a shared-memory tile of
// n x TI complex (padded rows, lanes run along the TI columns -> conflict-free 16 B accesses).
#include "common.cuh"

namespace hpnfft {

// Complex element of the FFT passes: double (the hot path) or float (the FP32 plans, NEXT #4).
// Aligned to its size: every global and shared access of an element is one 128-bit (64-bit) load
// or store.
template <typename R>
struct alignas(2 * sizeof(R)) CplxT {
  using real = R;
  R x, y;
};
using cplx = CplxT<double>;
using cplxf = CplxT<float>;

template <typename C>
__device__ __forceinline__ C cadd(C a, C b) { return {a.x + b.x, a.y + b.y}; }
template <typename C>
__device__ __forceinline__ C csub(C a, C b) { return {a.x - b.x, a.y - b.y}; }
template <typename C>
__device__ __forceinline__ C cmul(C a, C b) {
  return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
template <typename C>
__device__ __forceinline__ C mul_minus_i(C a) { return {a.y, -a.x}; }   // a * (-i)

// in-register DFT of RAD = 2, 4, 8 points
template <int RAD, typename C>
__device__ __forceinline__ void dft(C* v) {
  using Rl = typename C::real;
  if constexpr (RAD == 2) {
    C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (RAD == 4) {
    C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    C t2 = cadd(v[1], v[3]), t3 = mul_minus_i(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else {
    static_assert(RAD == 8, "radix 2, 4 or 8");
    const Rl h = (Rl)0.70710678118654752440084436210484903;
    C e[4] = {v[0], v[2], v[4], v[6]};
    C o[4] = {v[1], v[3], v[5], v[7]};
    dft<4>(e);
    dft<4>(o);
    // twiddles W8^k = exp(-i pi k/4)
    C o1 = {h * (o[1].x + o[1].y), h * (o[1].y - o[1].x)};
    C o2 = mul_minus_i(o[2]);
    C o3 = {h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)};
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
}

// Radix plan of an n = 2^LOGN point transform: as many radix-8 stages as possible, then one
// radix-4 or radix-2 stage, or two radix-4 stages when LOGN % 3 == 1 (and LOGN >= 4).
__host__ __device__ constexpr int n_radix8(int logn) { return logn / 3 - ((logn % 3 == 1 && logn >= 4) ? 1 : 0); }
__host__ __device__ constexpr int n_stages(int logn) {
  return n_radix8(logn) + ((logn - 3 * n_radix8(logn)) == 4 ? 2 : ((logn - 3 * n_radix8(logn)) > 0 ? 1 : 0));
}
__host__ __device__ constexpr int radix_of(int logn, int k) {
  return k < n_radix8(logn) ? 8 : ((logn - 3 * n_radix8(logn)) == 1 ? 2 : 4);
}
__host__ __device__ constexpr int ns_of(int logn, int k) { return k == 0 ? 1 : ns_of(logn, k - 1) * radix_of(logn, k - 1); }

// kernel argument of the energy variant of the x pass: per-CTA partial sums go to partial[]
struct EnergyArgs {
  double* partial;
  double e_a;
  int64_t k1_base;
  int N1, N2;
  // real charges (NEXT #2, energy_r2c): the x pass runs over the Hermitian half spectrum
  // k2 in [0, N2o/2] (N2 = N2o/2 + 1 columns, no shift) with k0, k1 extended to [-N/2, N/2]
  // (N0 + 2, N1 + 2 outputs, shift N/2 + 1); every output counts for the points of I_N it
  // represents: itself and its mirror -k (|S(-k)| = |S(k)| for real charges, Eq. 12)
  int real_half;
  int N0o, N1o, N2o;
  // w0[k] = inv_c[k]^2 exp(-e_a (k - N/2)^2) over the x pass's kept outputs (k_energy_w0): the
  // Gaussian of Eq. 12 factorises over the three dimensions, so each output needs one table
  // value and the thread's exp(-e_a (n1^2 + n2^2)) instead of an exp of its own
  const double* w0;
};

// a / nn of one Eq. 12 term; HPNFFT_ENERGY_RCP=1: times the correctly rounded reciprocal (no
// division subroutine; within an ulp of the quotient)
#ifndef HPNFFT_ENERGY_RCP
#define HPNFFT_ENERGY_RCP 1
#endif
__device__ __forceinline__ double energy_term(double a, double nn) {
#if HPNFFT_ENERGY_RCP
  return a * __drcp_rn(nn);
#else
  return a / nn;
#endif
}

__global__ void k_energy_w0(double* __restrict__ w0, const double* __restrict__ inv_c, int N, double e_a) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const double b0 = (double)(k - N / 2);
  w0[k] = inv_c[k] * inv_c[k] * exp(-e_a * b0 * b0);
}

// multiplicity of the half-spectrum frequency k (k2 >= 0) in Eq. 12's sum over I_N: k itself
// (k2 < N2/2, k0, k1 in I) plus its mirror -k (k2 >= 1, -k0, -k1 in I)
__device__ __forceinline__ double half_mult(int k0, int k1, int k2, const EnergyArgs& ea) {
  const bool in0 = k0 >= -ea.N0o / 2 && k0 < ea.N0o / 2, in1 = k1 >= -ea.N1o / 2 && k1 < ea.N1o / 2;
  const bool mi0 = -k0 >= -ea.N0o / 2 && -k0 < ea.N0o / 2, mi1 = -k1 >= -ea.N1o / 2 && -k1 < ea.N1o / 2;
  if (k2 > ea.N2o / 2) return 0.0;   // pad columns of the half lines
  return (double)((k2 < ea.N2o / 2 && in0 && in1) ? 1 : 0) + (double)((k2 >= 1 && mi0 && mi1) ? 1 : 0);
}

// Line context of one thread: its column in the shared tile, its global input/output line.
template <typename C>
struct LineIOT {
  const C* gin;          // element a of the line at gin[a * istride]
  C* gout;               // output k' at gout[k' * ostride]
  int64_t istride, ostride;
  int N;                 // kept outputs
  const typename C::real* inv_c;   // 1/c_k per kept output
  bool valid;
  int a_lo, a_len;       // elements a with (a - a_lo) mod n < a_len are loaded, the others are 0
  // peer-memory output (multi-GPU grid-slab y pass): output k of line (o, i) is stored over
  // NVLink into rank k / NP's buffer at ((o NP + k mod NP) ostride + i); null = local output
  C* const* peers;
  int NP;
  int64_t line_o, line_i;
  // inverse transform (Eq. 6 direction): the line's input is the compact N-entry line of fhat
  // (index k + N/2 <-> grid frequency k mod n, the other n - N frequencies are 0), scaled by
  // inv_c on input and conjugated (IFFT(v) = conj(FFT(conj(v)))); all n outputs conjugated
  bool inv;
  // ENUF reciprocal energy (Eq. 12; EN kernels, pass x only): instead of storing
  // fhat(k), accumulate exp(-e_a |n|^2) / |n|^2 |fhat(k)|^2 over n = k - N/2 != 0, where the
  // line is (k1, k2) = (k1_base + line_i / N2e, line_i mod N2e) and the output index is k0
  double e_a;
  int64_t k1_base;
  int N1e, N2e;
  double n12, g12;   // |(n1, n2)|^2 of the line and exp(-e_a n12)
  double esum;
  EnergyArgs ea;
};
using LineIO = LineIOT<cplx>;

// One Stockham stage (radix R, sub-transform length Ns) on the line held in column `col` of the
// shared tile.  Thread slot tj handles 8/R butterflies.  The first stage reads the line straight
// from global memory and the last writes the pruned, scaled outputs straight to global memory,
// so a 3-stage transform makes only two shared-memory round trips.
// Shared-memory slot of element a of the line in column col.  Strided passes (lanes run along
// the columns): row-major [a][col] with one padding column.  Contiguous pass (lanes run along a):
// column-major with one padding element every 8, so the stride-8 stores of the first stage and
// the unit-stride loads are both conflict-free.
template <int LOGN, int TI, bool CONTIG>
__device__ __forceinline__ int slot(int a, int col) {
  constexpr int n = 1 << LOGN;
  if (CONTIG) return col * (n + n / 8) + a + (a >> 3);
  return a * (TI + 1) + col;
}
template <int LOGN, int TI, bool CONTIG>
constexpr size_t tile_elems() {
  return CONTIG ? (size_t)TI * ((1 << LOGN) + (1 << LOGN) / 8) : (size_t)(1 << LOGN) * (TI + 1);
}

template <int LOGN, int R, int Ns, int TI, bool CONTIG, bool IN_G, bool OUT_G, bool EN, typename C>
__device__ __forceinline__ void stockham_stage(C* buf, int col, int tj, const C* __restrict__ tw, LineIOT<C>& io) {
  using Rl = typename C::real;
  constexpr int n = 1 << LOGN;
  constexpr int BPT = (n >= 8 ? 8 : n) / R;   // butterflies per thread
  constexpr int T = (n >= 8 ? n / 8 : 1);     // threads per column
  C v[BPT][R];
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = tj + b * T;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int a = j + r * (n / R);
      if (IN_G) {
        if (io.inv) {
          const int N = io.N;
          const bool lo = a < N / 2, hi = a >= n - N / 2;
          const int k = lo ? a + N / 2 : a - (n - N / 2);
          if (io.valid && (lo || hi)) {
            const C u = io.gin[(int64_t)k * io.istride];
            const Rl sc = io.inv_c[k];
            v[b][r] = {u.x * sc, -u.y * sc};
          } else {
            v[b][r] = {(Rl)0, (Rl)0};
          }
        } else {
          v[b][r] = (io.valid && ((a - io.a_lo) & (n - 1)) < io.a_len) ? io.gin[(int64_t)a * io.istride]
                                                                        : C{(Rl)0, (Rl)0};
        }
      } else {
        v[b][r] = buf[slot<LOGN, TI, CONTIG>(a, col)];
      }
    }
  }
  if (!IN_G) __syncthreads();   // everyone has read the tile before it is overwritten
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    const int j = tj + b * T;
    const int jm = j & (Ns - 1);
    if (Ns > 1) {
      // twiddles w^r, w = exp(-2 pi i step / n): w from the table, its powers by complex
      // products (one L1 load instead of seven; a few ulp per power, far below the 1e-12 bar)
      const int step = jm * (n / (Ns * R));
      if (R == 8) {
        const C w1 = tw[step & (n - 1)];
        const C w2 = cmul(w1, w1), w4 = cmul(w2, w2);
        const C w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
        const C ws[8] = {w1, w1, w2, w3, w4, w5, w6, w7};
#pragma unroll
        for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], ws[r]);
      } else {
#pragma unroll
        for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], tw[(step * r) & (n - 1)]);
      }
    }
    dft<R>(v[b]);
    const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = idxD + r * Ns;   // frequency index on the oversampled grid
      if (OUT_G && EN) {
        const int N = io.N;
        const bool lo = q < N / 2, hi = q >= n - N / 2;
        if (io.valid && (lo || hi)) {
          const int k = lo ? q + N / 2 : q - (n - N / 2);
          const double re = (double)v[b][r].x, im = (double)v[b][r].y;
          const int64_t k1 = io.k1_base + io.line_i / io.N2e;
          const int i0 = k - N / 2, i1 = (int)(k1 - io.N1e / 2);
          const int i2 = io.ea.real_half ? (int)(io.line_i % io.N2e) : (int)(io.line_i % io.N2e - io.N2e / 2);
          const double a0 = (double)i0;
          const double nn = a0 * a0 + io.n12;
          const double mult = io.ea.real_half ? half_mult(i0, i1, i2, io.ea) : 1.0;
          if (nn > 0.0 && mult > 0.0) io.esum += energy_term(mult * io.ea.w0[k] * (re * re + im * im), nn);
        }
      } else if (OUT_G && io.inv) {
        if (io.valid) io.gout[(int64_t)q * io.ostride] = {v[b][r].x, -v[b][r].y};
      } else if (OUT_G) {
        const int N = io.N;
        const bool lo = q < N / 2, hi = q >= n - N / 2;
        if (io.valid && (lo || hi)) {
          const int k = lo ? q + N / 2 : q - (n - N / 2);
          const Rl sc = io.inv_c[k];
          C* dst = io.peers ? io.peers[k / io.NP] + ((io.line_o * io.NP + k % io.NP) * io.ostride + io.line_i)
                            : io.gout + (int64_t)k * io.ostride;
          *dst = {v[b][r].x * sc, v[b][r].y * sc};
        }
      } else {
        buf[slot<LOGN, TI, CONTIG>(q, col)] = v[b][r];
      }
    }
  }
  if (!OUT_G) __syncthreads();   // the tile is complete before the next stage reads it
}

template <int LOGN, int TI, bool CONTIG, bool EN, int K, typename C>
__device__ __forceinline__ void run_stages(C* buf, int col, int tj, const C* __restrict__ tw, LineIOT<C>& io) {
  constexpr int NS = n_stages(LOGN);
  stockham_stage<LOGN, radix_of(LOGN, K), ns_of(LOGN, K), TI, CONTIG, K == 0, K == NS - 1, EN>(buf, col, tj, tw, io);
  if constexpr (K + 1 < NS) run_stages<LOGN, TI, CONTIG, EN, K + 1>(buf, col, tj, tw, io);
}

// all stages into the shared tile (the R2C z pass post-processes the complex half-length transform)
template <int LOGN, int TI, bool CONTIG, int K, typename C>
__device__ __forceinline__ void run_stages_to_smem(C* buf, int col, int tj, const C* __restrict__ tw, LineIOT<C>& io) {
  constexpr int NS = n_stages(LOGN);
  stockham_stage<LOGN, radix_of(LOGN, K), ns_of(LOGN, K), TI, CONTIG, K == 0, false, false>(buf, col, tj, tw, io);
  if constexpr (K + 1 < NS) run_stages_to_smem<LOGN, TI, CONTIG, K + 1>(buf, col, tj, tw, io);
}

// Batched pruned pass.  Lines are indexed by (outer o, column i); element a of a line sits at
//   in + (o * n + a) * inner + i                (inner > 1: strided pass)
// and for the contiguous pass (CONTIG, inner == 1) the TI columns of a CTA are TI consecutive
// outers.  Output k' in [0,N) goes to out + (o * N + k') * inner + i, scaled by inv_c[k'].
// Thread mapping: strided passes put consecutive lanes on consecutive columns (coalesced rows of
// TI complex); the contiguous pass puts consecutive lanes on consecutive butterflies of a line.
template <int LOGN, int TI, bool CONTIG, bool EN = false, typename C = cplx>
__global__ void __launch_bounds__(TI*((1 << LOGN) >= 8 ? (1 << LOGN) / 8 : 1))
k_fft_pass(const C* __restrict__ in, C* __restrict__ out, int64_t outer, int64_t inner, int N,
           const typename C::real* __restrict__ inv_c, const C* __restrict__ tw, int64_t o_start, int64_t o_total,
           int a_lo, int a_len, C* const* peers, int NP, int inv, EnergyArgs ea, const int* __restrict__ abort_flag) {
  constexpr int n = 1 << LOGN;
  constexpr int T = (n >= 8 ? n / 8 : 1);
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  C* smem = reinterpret_cast<C*>(smem_bytes);
  const int tid = threadIdx.x;
  LineIOT<C> io;
  io.N = N;
  io.inv_c = inv_c;
  io.a_lo = a_lo;
  io.a_len = a_len;
  io.peers = peers;
  io.NP = NP;
  io.inv = inv != 0;
  int col, tj;
  if (CONTIG) {
    col = tid / T;
    tj = tid % T;
    const int64_t o = (int64_t)blockIdx.x * TI + col;
    io.valid = o < outer;
    const int64_t oc = io.valid ? (o_start + o) % o_total : 0;
    io.gin = in + oc * (inv ? (int64_t)N : (int64_t)n);
    io.istride = 1;
    io.gout = out + oc * (inv ? (int64_t)n : (int64_t)N);
    io.ostride = 1;
  } else {
    col = tid % TI;
    tj = tid / TI;
    const int64_t tiles_per_outer = (inner + TI - 1) / TI;
    const int64_t o = (o_start + blockIdx.x / tiles_per_outer) % o_total;
    const int64_t i = (blockIdx.x % tiles_per_outer) * TI + col;
    io.valid = i < inner;
    const int64_t ic = io.valid ? i : 0;
    io.gin = in + o * (inv ? (int64_t)N : (int64_t)n) * inner + ic;
    io.istride = inner;
    io.gout = out + o * (inv ? (int64_t)n : (int64_t)N) * inner + ic;
    io.ostride = inner;
    io.line_o = o;
    io.line_i = ic;
  }
  // peer stores after a timed-out cross-GPU barrier: write nothing (the error is reported by the
  // plan's next call)
  if (peers && abort_flag && *abort_flag) io.valid = false;
  io.e_a = ea.e_a;
  io.k1_base = ea.k1_base;
  io.N1e = ea.N1;
  io.N2e = ea.N2 > 0 ? ea.N2 : 1;
  io.esum = 0.0;
  io.ea = ea;
  if constexpr (EN) {
    const int64_t k1 = io.k1_base + io.line_i / io.N2e;
    const double a1 = (double)(k1 - io.N1e / 2);
    const double a2 = ea.real_half ? (double)(io.line_i % io.N2e) : (double)(io.line_i % io.N2e - io.N2e / 2);
    io.n12 = a1 * a1 + a2 * a2;
    io.g12 = exp(-ea.e_a * io.n12);
  }
  run_stages<LOGN, TI, CONTIG, EN, 0>(smem, col, tj, tw, io);
  if constexpr (EN) {   // CTA partial of Eq. 12's sum, fixed order (deterministic)
    __shared__ double red[32];
    double v = io.esum * io.g12;   // the line's Gaussian factor, once
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      ea.partial[blockIdx.x] = t;
    }
  }
}


// ---------------------------------------------------------------------------------------------
// n = 1024 contiguous pass (z lines of config 5 and of the large HP-ENUF grids): four-step
// 1024 = 32 x 32 with each 32-point DFT in one thread's registers and ONE shared-memory
// transpose, instead of 4 Stockham stages (3 round trips, 3 CTAs per SM):
//   x index t + 32 j, frequency k1 + 32 k2:
//   Y[t][k1] = W1024^{t k1} sum_j x[t + 32 j] W32^{j k1}      (thread t, coalesced loads)
//   X[k1 + 32 k2] = sum_t Y[t][k1] W32^{t k2}                  (thread k1, coalesced stores)
// shared tile [k1][t] with row stride 33 (conflict-free in both phases).  The twiddles
// W1024^{t k1} are powers of the table value W1024^t by complex products (31 products:
// ~31 ulp, far below the 1e-12 bar).  Forward, output-pruned (k in I_N, scaled by 1/c_k).
__constant__ cplx c_w32[32] = {
    {1, -0},
    {0.98078528040323043, -0.19509032201612825},
    {0.92387953251128674, -0.38268343236508978},
    {0.83146961230254524, -0.55557023301960218},
    {0.70710678118654757, -0.70710678118654746},
    {0.55557023301960229, -0.83146961230254524},
    {0.38268343236508984, -0.92387953251128674},
    {0.19509032201612833, -0.98078528040323043},
    {6.123233995736766e-17, -1},
    {-0.19509032201612819, -0.98078528040323043},
    {-0.38268343236508973, -0.92387953251128674},
    {-0.55557023301960196, -0.83146961230254546},
    {-0.70710678118654746, -0.70710678118654757},
    {-0.83146961230254535, -0.55557023301960218},
    {-0.92387953251128674, -0.38268343236508989},
    {-0.98078528040323043, -0.19509032201612861},
    {-1, -1.2246467991473532e-16},
    {-0.98078528040323043, 0.19509032201612836},
    {-0.92387953251128685, 0.38268343236508967},
    {-0.83146961230254546, 0.55557023301960196},
    {-0.70710678118654768, 0.70710678118654746},
    {-0.55557023301960218, 0.83146961230254524},
    {-0.38268343236509034, 0.92387953251128652},
    {-0.19509032201612866, 0.98078528040323032},
    {-1.8369701987210297e-16, 1},
    {0.1950903220161283, 0.98078528040323043},
    {0.38268343236509, 0.92387953251128663},
    {0.55557023301960184, 0.83146961230254546},
    {0.70710678118654735, 0.70710678118654768},
    {0.83146961230254524, 0.55557023301960218},
    {0.92387953251128652, 0.38268343236509039},
    {0.98078528040323032, 0.19509032201612872}};

// in-register 32-point DFT, v[j] -> V[k]: 32 = 4 x 8, j = r + 4 i, k = k1 + 8 k2
__device__ __forceinline__ void dft32(cplx (&v)[32]) {
  cplx y[4][8];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) y[r][i] = v[r + 4 * i];
    dft<8>(y[r]);
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1)
      if (r > 0) y[r][k1] = cmul(y[r][k1], c_w32[(r * k1) & 31]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 8; ++k1) {
    cplx z[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
    dft<4>(z);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) v[k1 + 8 * k2] = z[k2];
  }
}

constexpr int kF1024Lines = 2;   // lines per CTA (32 threads each; 33.8 KB static shared)

__global__ void __launch_bounds__(32 * kF1024Lines) k_fft1024_contig(const cplx* __restrict__ in, cplx* __restrict__ out,
                                                                   int64_t outer, int N,
                                                                   const double* __restrict__ inv_c,
                                                                   const cplx* __restrict__ tw, int64_t o_start,
                                                                   int64_t o_total) {
  constexpr int n = 1024;
  __shared__ cplx tile[kF1024Lines][32 * 33];
  const int t = threadIdx.x & 31, line = threadIdx.x >> 5;
  const int64_t o = (int64_t)blockIdx.x * kF1024Lines + line;
  const bool valid = o < outer;
  const int64_t oc = valid ? (o_start + o) % o_total : 0;
  const cplx* gin = in + oc * n;
  cplx v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = valid ? gin[t + 32 * j] : cplx{0.0, 0.0};
  dft32(v);
  cplx* tl = tile[line];
  {
    const cplx w = tw[t];   // W1024^t
    cplx p = {1.0, 0.0};
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) {
      tl[k1 * 33 + t] = k1 ? cmul(v[k1], p) : v[0];
      p = cmul(p, w);
    }
  }
  __syncwarp();
#pragma unroll
  for (int tt = 0; tt < 32; ++tt) v[tt] = tl[t * 33 + tt];   // thread t now holds k1 = t
  dft32(v);
  if (!valid) return;
  cplx* gout = out + oc * N;
  const int k1 = t;
#pragma unroll
  for (int k2 = 0; k2 < 32; ++k2) {
    const int q = k1 + 32 * k2;
    const bool lo = q < N / 2, hi = q >= n - N / 2;
    if (lo || hi) {
      const int k = lo ? q + N / 2 : q - (n - N / 2);
      const double sc = inv_c[k];
      gout[k] = {v[k2].x * sc, v[k2].y * sc};
    }
  }
}

template <int LOGN>
constexpr int tile_cols() {
  return (1 << LOGN) >= 1024 ? 4 : ((4096 >> LOGN) > 64 ? 64 : (4096 >> LOGN));
}
#ifndef HPNFFT_FFT_CONTIG_LINES
#define HPNFFT_FFT_CONTIG_LINES 2
#endif
// contiguous pass: lines per CTA (fewer, smaller CTAs keep more of them resident so that their
// global-load phases overlap)
template <int LOGN>
constexpr int tile_cols_contig() {
  return tile_cols<LOGN>() < HPNFFT_FFT_CONTIG_LINES ? tile_cols<LOGN>() : HPNFFT_FFT_CONTIG_LINES;
}


// Strided n = 1024 lines (passes y and x): the same four-step transform, CW columns per CTA.
// Thread (c, t) = (tid mod CW, tid / CW): lanes run along the columns, so each of the 32 loads
// of a thread is part of a CW x 16 B row segment.  Shared tile [c][k1][t], k1 rows of 33, one
// padding element per column (conflict-free stores and loads).  Input rows a with
// (a - a_lo) mod n >= a_len read as 0 (pass x: unoccupied planes).
template <int CW, bool EN>
__global__ void __launch_bounds__(32 * CW) k_fft1024_strided(const cplx* __restrict__ in, cplx* __restrict__ out,
                                                            int64_t inner, int N, const double* __restrict__ inv_c,
                                                            const cplx* __restrict__ tw, int64_t o_start,
                                                            int64_t o_total, int a_lo, int a_len, EnergyArgs ea) {
  constexpr int n = 1024;
  constexpr int CS = 32 * 33 + 1;   // column stride of the tile (elements)
  extern __shared__ cplx smem[];
  const int c = threadIdx.x % CW, t = threadIdx.x / CW;
  const int64_t tiles_per_outer = (inner + CW - 1) / CW;
  const int64_t o = (o_start + blockIdx.x / tiles_per_outer) % o_total;
  const int64_t i = (blockIdx.x % tiles_per_outer) * CW + c;
  const bool valid = i < inner;
  const int64_t ic = valid ? i : 0;
  const cplx* gin = in + o * (int64_t)n * inner + ic;
  cplx v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int a = t + 32 * j;
    v[j] = (valid && ((a - a_lo) & (n - 1)) < a_len) ? gin[(int64_t)a * inner] : cplx{0.0, 0.0};
  }
  dft32(v);
  cplx* tl = smem + c * CS;
  {
    const cplx w = tw[t];
    cplx p = {1.0, 0.0};
#pragma unroll
    for (int k1 = 0; k1 < 32; ++k1) {
      tl[k1 * 33 + t] = k1 ? cmul(v[k1], p) : v[0];
      p = cmul(p, w);
    }
  }
  __syncthreads();
#pragma unroll
  for (int tt = 0; tt < 32; ++tt) v[tt] = tl[t * 33 + tt];   // thread (c, t) now holds k1 = t
  dft32(v);
  const int k1 = t;
  if constexpr (EN) {   // Eq. 12 energy variant of pass x (see LineIO): weighted |fhat|^2, CTA partial
    double esum = 0.0;
    if (valid) {
      const int N2e = ea.N2 > 0 ? ea.N2 : 1;
      const int i1 = (int)(ea.k1_base + ic / N2e - ea.N1 / 2);
      const int i2 = ea.real_half ? (int)(ic % N2e) : (int)(ic % N2e - N2e / 2);
      const double b1 = (double)i1, b2 = (double)i2;
      const double n12 = b1 * b1 + b2 * b2, g12 = exp(-ea.e_a * n12);
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) {
        const int q = k1 + 32 * k2;
        const bool lo = q < N / 2, hi = q >= n - N / 2;
        if (lo || hi) {
          const int k = lo ? q + N / 2 : q - (n - N / 2);
          const double re = v[k2].x, im = v[k2].y, b0 = (double)(k - N / 2);
          const double nn = b0 * b0 + n12;
          const double mult = ea.real_half ? half_mult(k - N / 2, i1, i2, ea) : 1.0;
          if (nn > 0.0 && mult > 0.0) esum += energy_term(mult * ea.w0[k] * (re * re + im * im), nn);
        }
      }
      esum *= g12;   // the line's Gaussian factor, once
    }
    __shared__ double red[32];
#pragma unroll
    for (int w = 16; w > 0; w >>= 1) esum += __shfl_xor_sync(0xffffffffu, esum, w);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = esum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      ea.partial[blockIdx.x] = tot;
    }
    return;
  }
  if (!valid) return;
  cplx* gout = out + o * (int64_t)N * inner + ic;
#pragma unroll
  for (int k2 = 0; k2 < 32; ++k2) {
    const int q = k1 + 32 * k2;
    const bool lo = q < N / 2, hi = q >= n - N / 2;
    if (lo || hi) {
      const int k = lo ? q + N / 2 : q - (n - N / 2);
      const double sc = inv_c[k];
      gout[(int64_t)k * inner] = {v[k2].x * sc, v[k2].y * sc};
    }
  }
}
#ifndef HPNFFT_F1024_CW
#define HPNFFT_F1024_CW 8
#endif

static bool fft1024_disabled() {   // HPNFFT_FFT1024=0: the generic Stockham pass (measurement)
  static const bool off = [] {
    const char* e = getenv("HPNFFT_FFT1024");
    return e && e[0] == '0';
  }();
  return off;
}

template <int LOGN, typename C = cplx>
static int launch_pass_n(Plan* p, const C* in, C* out, int64_t outer, int64_t inner, int N,
                         const typename C::real* inv_c, const C* tw, bool contig, int64_t o_start, int64_t o_total,
                         int a_lo, int a_len, C* const* peers, int NP, int inv) {
  constexpr bool kF64 = sizeof(typename C::real) == 8;
  constexpr int TI = tile_cols<LOGN>();
  constexpr int TC = tile_cols_contig<LOGN>();
  constexpr int n = 1 << LOGN;
  constexpr int NT = TI * (n >= 8 ? n / 8 : 1);
  if (outer <= 0 || inner <= 0) return HPNFFT_OK;
  if constexpr (kF64) {
  if (LOGN == 10 && contig && !inv && a_lo == 0 && a_len == n && !fft1024_disabled()) {
    k_fft1024_contig<<<(unsigned)((outer + kF1024Lines - 1) / kF1024Lines), 32 * kF1024Lines, 0, p->stream>>>(
        in, out, outer, N, inv_c, tw, o_start, o_total);
    p->launches++;
    return check_launch(p, "fft pass (n = 1024)");
  }
  if (LOGN == 10 && !contig && !inv && peers == nullptr && !fft1024_disabled()) {
    constexpr int CW = HPNFFT_F1024_CW;
    const size_t smem = sizeof(cplx) * (size_t)CW * (32 * 33 + 1);
    HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(k_fft1024_strided<CW, false>),
                                            (int)smem),
                    "fft1024 smem attr");
    const int64_t blocks = outer * ((inner + CW - 1) / CW);
    k_fft1024_strided<CW, false><<<(unsigned)blocks, 32 * CW, smem, p->stream>>>(in, out, inner, N, inv_c, tw, o_start,
                                                                                 o_total, a_lo, a_len, EnergyArgs{});
    p->launches++;
    return check_launch(p, "fft pass (n = 1024, strided)");
  }
  }
  if (contig) {
    const size_t smem = tile_elems<LOGN, TC, true>() * sizeof(C);
    const int64_t blocks = (outer + TC - 1) / TC;
    auto kern = k_fft_pass<LOGN, TC, true, false, C>;
    HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(kern), (int)smem),
                    "fft smem attr");
    kern<<<(unsigned)blocks, TC * (n >= 8 ? n / 8 : 1), smem, p->stream>>>(in, out, outer, inner, N, inv_c, tw,
                                                                            o_start, o_total, a_lo, a_len, nullptr, 1, inv,
                                                                            EnergyArgs{}, nullptr);
  } else {
    const size_t smem = tile_elems<LOGN, TI, false>() * sizeof(C);
    const int64_t blocks = outer * ((inner + TI - 1) / TI);
    auto kern = k_fft_pass<LOGN, TI, false, false, C>;
    HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(kern), (int)smem),
                    "fft smem attr");
    kern<<<(unsigned)blocks, NT, smem, p->stream>>>(in, out, outer, inner, N, inv_c, tw, o_start, o_total, a_lo,
                                                     a_len, peers, NP, inv, EnergyArgs{}, peers ? p->dist_err : nullptr);
  }
  p->launches++;
  return check_launch(p, "fft pass");
}

static int launch_pass(Plan* p, int logn, const double* in, double* out, int64_t outer, int64_t inner, int N,
                       const double* inv_c, const double* tw, bool contig, int64_t o_start, int64_t o_total,
                       int a_lo, int a_len, cplx* const* peers = nullptr, int NP = 1, int inv = 0) {
  const cplx* ci = reinterpret_cast<const cplx*>(in);
  cplx* co = reinterpret_cast<cplx*>(out);
  const cplx* ct = reinterpret_cast<const cplx*>(tw);
  switch (logn) {
    case 2: return launch_pass_n<2>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 3: return launch_pass_n<3>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 4: return launch_pass_n<4>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 5: return launch_pass_n<5>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 6: return launch_pass_n<6>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 7: return launch_pass_n<7>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 8: return launch_pass_n<8>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 9: return launch_pass_n<9>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    case 10: return launch_pass_n<10>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, peers, NP, inv);
    default:
      set_error("FFT length not supported");
      return HPNFFT_E_UNSUPPORTED;
  }
}

// FP32 plans (NEXT #4): the same pruned Stockham passes on complex64 lines (no four-step n = 1024
// special case), float twiddles and deconvolution tables
static int launch_pass_f32(Plan* p, int logn, const float* in, float* out, int64_t outer, int64_t inner, int N,
                           const float* inv_c, const float* tw, bool contig, int64_t o_start, int64_t o_total,
                           int a_lo, int a_len) {
  const cplxf* ci = reinterpret_cast<const cplxf*>(in);
  cplxf* co = reinterpret_cast<cplxf*>(out);
  const cplxf* ct = reinterpret_cast<const cplxf*>(tw);
  switch (logn) {
    case 2: return launch_pass_n<2, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 3: return launch_pass_n<3, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 4: return launch_pass_n<4, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 5: return launch_pass_n<5, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 6: return launch_pass_n<6, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 7: return launch_pass_n<7, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 8: return launch_pass_n<8, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 9: return launch_pass_n<9, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    case 10: return launch_pass_n<10, cplxf>(p, ci, co, outer, inner, N, inv_c, ct, contig, o_start, o_total, a_lo, a_len, nullptr, 1, 0);
    default:
      set_error("FFT length not supported");
      return HPNFFT_E_UNSUPPORTED;
  }
}

// FP32 adjoint: passes z, y, x (+ deconvolve, crop) of the complex64 grid (d < 3: fewer passes)
int fft_and_deconvolve_f32(Plan* p, float* fhat) {
  const int64_t n0 = p->n[0], n1 = p->n[1];
  const int64_t N1 = p->N[1], N2 = p->N[2];
  const int lead = 3 - p->d;
  const int64_t plo = p->plane_lo, plen = p->plane_len;
  float* grid = reinterpret_cast<float*>(p->grid);
  float* bufA = reinterpret_cast<float*>(p->bufA);
  int rc;
  stage_begin(p, 4);
  rc = launch_pass_f32(p, p->logn[2], grid, lead == 2 ? fhat : bufA, plen * n1, 1, (int)N2, p->inv_cf[2], p->twiddle_f[2],
                       true, plo * n1, n0 * n1, 0, (int)p->n[2]);
  stage_end(p, 4);
  if (rc || lead == 2) return rc;
  stage_begin(p, 5);
  rc = launch_pass_f32(p, p->logn[1], bufA, lead == 1 ? fhat : grid, plen, N2, (int)N1, p->inv_cf[1], p->twiddle_f[1],
                       false, plo, n0, 0, (int)n1);
  stage_end(p, 5);
  if (rc || lead == 1) return rc;
  stage_begin(p, 6);
  rc = launch_pass_f32(p, p->logn[0], grid, fhat, 1, N1 * N2, (int)p->N[0], p->inv_cf[0], p->twiddle_f[0], false, 0, 1,
                       (int)plo, (int)plen);
  stage_end(p, 6);
  return rc;
}

int fft_pass(Plan* p, int dim, const double* in, double* out, int64_t outer, int64_t inner, bool contig,
             int64_t o_start, int64_t o_total, int a_lo, int a_len, double* const* peers, int NP) {
  return launch_pass(p, p->logn[dim], in, out, outer, inner, (int)p->N[dim], p->inv_c[dim], p->twiddle[dim], contig,
                     o_start, o_total, a_lo, a_len, reinterpret_cast<cplx* const*>(peers), NP);
}

// Inverse direction (Eq. 6; Subdividing + Inverse FFT of Alg. 5):
// ghat(k mod n) = fhat(k) / prod c_k on I_N, 0 elsewhere, then g(l) = sum_k ghat(k) e^{+2 pi i k.l/n}.
// Three input-pruned passes, smallest data first: z (fhat[N0][N1][N2] -> C[N0][N1][n2], grid
// memory), y (C -> D[N0][n1][n2], bufA), x (D -> g[n0][n1][n2], grid).
int subdivide_and_ifft(Plan* p, const double* fhat) {
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2];
  const int64_t N0 = p->N[0], N1 = p->N[1];
  const int lead = 3 - p->d;   // trivial leading dimensions (d < 3): no pass along them
  // d = 3: z fhat -> grid, y grid -> bufA, x bufA -> grid; d = 2: z fhat -> bufA, y bufA -> grid;
  // d = 1: z fhat -> grid (the last pass always lands in the grid)
  double* zout = lead == 1 ? p->bufA : p->grid;
  int rc = launch_pass(p, p->logn[2], fhat, zout, N0 * N1, 1, (int)p->N[2], p->inv_c[2], p->twiddle[2], true, 0,
                       N0 * N1, 0, (int)n2, nullptr, 1, 1);
  if (rc || lead == 2) return rc;
  double* yout = lead == 1 ? p->grid : p->bufA;
  rc = launch_pass(p, p->logn[1], zout, yout, N0, n2, (int)N1, p->inv_c[1], p->twiddle[1], false, 0, N0, 0,
                   (int)n1, nullptr, 1, 1);
  if (rc || lead == 1) return rc;
  return launch_pass(p, p->logn[0], p->bufA, p->grid, 1, n1 * n2, (int)N0, p->inv_c[0], p->twiddle[0], false, 0, 1,
                     0, (int)n0, nullptr, 1, 1);
}

int fft_and_deconvolve(Plan* p, double* fhat) {
  const int64_t n0 = p->n[0], n1 = p->n[1];
  const int64_t N0 = p->N[0], N1 = p->N[1], N2 = p->N[2];
  const int lead = 3 - p->d;   // trivial leading dimensions (d < 3): the last real pass writes fhat
  // only the occupied l0 planes are transformed by passes z and y; pass x treats the others as 0
  const int64_t plo = p->plane_lo, plen = p->plane_len;
  int rc;
  stage_begin(p, 4);
  rc = launch_pass(p, p->logn[2], p->grid, lead == 2 ? fhat : p->bufA, plen * n1, 1, (int)N2, p->inv_c[2],
                   p->twiddle[2], true, plo * n1, n0 * n1, 0, (int)p->n[2]);
  stage_end(p, 4);
  if (rc || lead == 2) return rc;
  stage_begin(p, 5);
  rc = launch_pass(p, p->logn[1], p->bufA, lead == 1 ? fhat : p->bufB, plen, N2, (int)N1, p->inv_c[1], p->twiddle[1],
                   false, plo, n0, 0, (int)n1);
  stage_end(p, 5);
  if (rc || lead == 1) return rc;
  stage_begin(p, 6);
  rc = x_pass(p, p->bufB, fhat, N1 * N2, 0, (int)plo, (int)plen);
  stage_end(p, 6);
  (void)N0;
  return rc;
}

// ---------------------------------------------------------------------------------------------
// Real charges (Eq. 12 with real q): the z pass of a REAL grid line
// x[0 .. n2) (the real sweep's output, read as h = n2/2 complex z[j] = x[2j] + i x[2j+1]): one
// complex length-h Stockham transform Z in the shared tile, then the split
//   X(k) = (Z(k) + conj Z(h-k))/2 - i exp(-2 pi i k/n2) (Z(k) - conj Z(h-k))/2,   k = 0 .. N2/2,
// deconvolved by 1/c_k2 and stored as the Hermitian half line out[line][0 .. N2/2] (N2/2 + 1
// complex): half the bytes of the complex pass, the other half follows from X(-k) = conj X(k).
template <int LOGH, int TC>
__global__ void __launch_bounds__(TC*((1 << LOGH) >= 8 ? (1 << LOGH) / 8 : 1))
k_fft_r2c_z(const cplx* __restrict__ in, cplx* __restrict__ out, int64_t outer, int N2, int N2s,
            const double* __restrict__ inv_c, const cplx* __restrict__ tw_h, const cplx* __restrict__ tw_n,
            int64_t o_start, int64_t o_total) {
  constexpr int h = 1 << LOGH;
  constexpr int T = (h >= 8 ? h / 8 : 1);
  extern __shared__ __align__(16) unsigned char smem_bytes[];
  cplx* smem = reinterpret_cast<cplx*>(smem_bytes);
  const int tid = threadIdx.x;
  const int col = tid / T, tj = tid % T;
  LineIO io;
  const int64_t o = (int64_t)blockIdx.x * TC + col;
  io.valid = o < outer;
  const int64_t oc = io.valid ? (o_start + o) % o_total : 0;
  io.gin = in + oc * (int64_t)h;
  io.istride = 1;
  io.a_lo = 0;
  io.a_len = h;
  io.inv = false;
  io.peers = nullptr;
  run_stages_to_smem<LOGH, TC, true, 0>(smem, col, tj, tw_h, io);
  if (!io.valid) return;
  // output lines of N2s >= N2/2 + 1 entries (padded to 128-byte rows: the strided passes then read
  // aligned row segments); the pad entries are zero
  const int N2h = N2 / 2 + 1;
  cplx* gout = out + oc * (int64_t)N2s;
  for (int k = N2h + tj; k < N2s; k += T) gout[k] = {0.0, 0.0};
  for (int k = tj; k < N2h; k += T) {
    const cplx zk = smem[slot<LOGH, TC, true>(k & (h - 1), col)];
    const cplx zr = smem[slot<LOGH, TC, true>((h - k) & (h - 1), col)];
    const cplx e = {0.5 * (zk.x + zr.x), 0.5 * (zk.y - zr.y)};    // (Z(k) + conj Z(h-k)) / 2
    const cplx d = {0.5 * (zk.x - zr.x), 0.5 * (zk.y + zr.y)};    // (Z(k) - conj Z(h-k)) / 2
    const cplx wd = cmul(tw_n[k], d);                              // exp(-2 pi i k / n2) d
    const double sc = inv_c[k < N2 / 2 ? k + N2 / 2 : 0];          // c_k even: c(N2/2) = c(-N2/2)
    gout[k] = {(e.x + wd.y) * sc, (e.y - wd.x) * sc};              // e - i wd
  }
}

template <int LOGH>
static int launch_r2c_n(Plan* p, const cplx* in, cplx* out, int64_t outer, int N2, int N2s, const double* inv_c,
                        const cplx* tw_h, const cplx* tw_n, int64_t o_start, int64_t o_total) {
  constexpr int TC = tile_cols_contig<LOGH>();
  constexpr int h = 1 << LOGH;
  if (outer <= 0) return HPNFFT_OK;
  const size_t smem = tile_elems<LOGH, TC, true>() * sizeof(cplx);
  auto kern = k_fft_r2c_z<LOGH, TC>;
  HPNFFT_CUDA_TRY(p, set_max_smem(reinterpret_cast<const void*>(kern), smem), "r2c smem attr");
  kern<<<(unsigned)((outer + TC - 1) / TC), TC * (h >= 8 ? h / 8 : 1), smem, p->stream>>>(in, out, outer, N2, N2s,
                                                                                       inv_c, tw_h, tw_n, o_start, o_total);
  p->launches++;
  return check_launch(p, "fft r2c z pass");
}

static int launch_r2c(Plan* p, int logh, const double* in, double* out, int64_t outer, int N2s, int64_t o_start,
                      int64_t o_total) {
  const cplx* ci = reinterpret_cast<const cplx*>(in);
  cplx* co = reinterpret_cast<cplx*>(out);
  const cplx* th = reinterpret_cast<const cplx*>(p->twiddle_half);
  const cplx* tn = reinterpret_cast<const cplx*>(p->twiddle[2]);
  const int N2 = (int)p->N[2];
  const double* ic = p->inv_c[2];
  switch (logh) {
    case 1: return launch_r2c_n<1>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 2: return launch_r2c_n<2>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 3: return launch_r2c_n<3>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 4: return launch_r2c_n<4>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 5: return launch_r2c_n<5>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 6: return launch_r2c_n<6>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 7: return launch_r2c_n<7>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 8: return launch_r2c_n<8>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    case 9: return launch_r2c_n<9>(p, ci, co, outer, N2, N2s, ic, th, tn, o_start, o_total);
    default:
      set_error("R2C length not supported");
      return HPNFFT_E_UNSUPPORTED;
  }
}

// x pass of Eq. 12 (ENUF reciprocal energy): the x lines of B[n0][L1][N2] (L1 = the k1 rows
// this plan holds, starting at k1_base) with the deconvolution applied and the weighted |fhat|^2
// summed per CTA into partial[] (nothing is stored).  Returns the number of partials (CTAs).
template <int LOGN>
static int64_t launch_energy_n(Plan* p, const cplx* in, int64_t inner, int N0, const double* inv_c0,
                               const EnergyArgs& ea, int a_lo, int a_len) {
  constexpr int TI = tile_cols<LOGN>();
  constexpr int n = 1 << LOGN;
  constexpr int NT = TI * (n >= 8 ? n / 8 : 1);
  if (LOGN == 10 && !fft1024_disabled()) {
    constexpr int CW = HPNFFT_F1024_CW;
    const size_t smem = sizeof(cplx) * (size_t)CW * (32 * 33 + 1);
    if (set_max_smem(reinterpret_cast<const void*>(k_fft1024_strided<CW, true>), (int)smem) != cudaSuccess) {
      fail(p, HPNFFT_E_CUDA, "fft1024 smem attr");
      return -1;
    }
    const int64_t blocks = (inner + CW - 1) / CW;
    k_fft1024_strided<CW, true><<<(unsigned)blocks, 32 * CW, smem, p->stream>>>(
        in, nullptr, inner, N0, inv_c0, reinterpret_cast<const cplx*>(p->twiddle[0]), 0, 1, a_lo, a_len, ea);
    p->launches++;
    return check_launch(p, "fft energy pass (n = 1024)") ? -1 : blocks;
  }
  const size_t smem = tile_elems<LOGN, TI, false>() * sizeof(cplx);
  const int64_t blocks = (inner + TI - 1) / TI;
  auto kern = k_fft_pass<LOGN, TI, false, true>;
  if (set_max_smem(reinterpret_cast<const void*>(kern), (int)smem) != cudaSuccess) {
    fail(p, HPNFFT_E_CUDA, "fft smem attr");
    return -1;
  }
  kern<<<(unsigned)blocks, NT, smem, p->stream>>>(in, nullptr, 1, inner, N0, inv_c0,
                                                   reinterpret_cast<const cplx*>(p->twiddle[0]), 0, 1, a_lo, a_len,
                                                   nullptr, 1, 0, ea, nullptr);
  p->launches++;
  return check_launch(p, "fft energy pass") ? -1 : blocks;
}

static int64_t energy_x_pass(Plan* p, const double* in, int64_t inner, int N0, const double* inv_c0,
                             const EnergyArgs& ea_in, int a_lo, int a_len) {
  const cplx* ci = reinterpret_cast<const cplx*>(in);
  EnergyArgs ea = ea_in;
  ea.w0 = p->e_w0;
  k_energy_w0<<<(unsigned)((N0 + 255) / 256), 256, 0, p->stream>>>(p->e_w0, inv_c0, N0, ea.e_a);
  p->launches++;
  if (check_launch(p, "energy weight table")) return -1;
  switch (p->logn[0]) {
    case 2: return launch_energy_n<2>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 3: return launch_energy_n<3>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 4: return launch_energy_n<4>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 5: return launch_energy_n<5>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 6: return launch_energy_n<6>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 7: return launch_energy_n<7>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 8: return launch_energy_n<8>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 9: return launch_energy_n<9>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    case 10: return launch_energy_n<10>(p, ci, inner, N0, inv_c0, ea, a_lo, a_len);
    default:
      set_error("FFT length not supported");
      return -1;
  }
}

// Eq. 12 for real charges on one GPU: R2C z pass (half lines k2 in [0, N2/2]) -> y pass with k1
// extended to [-N1/2, N1/2] -> x pass with k0 extended to [-N0/2, N0/2] summing every half-spectrum
// frequency with its multiplicity in I_N (half_mult).  Exact: the same sum as the complex path.
int energy_r2c(Plan* p) {
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2];
  const int64_t N0 = p->N[0], N1 = p->N[1], N2 = p->N[2];
  // half lines k2 in [0, N2/2] stored with a stride padded to 8 (128-byte rows); the pad columns
  // are zero (R2C pass) and count 0 times in the energy (half_mult)
  int64_t N2h = ((N2 / 2 + 1) + 7) / 8 * 8;
  if (N2h > N2) N2h = N2 / 2 + 1;   // small N2: bufA holds n0 n1 N2 entries
  const int64_t plo = p->plane_lo, plen = p->plane_len;
  stage_begin(p, 4);
  int rc = launch_r2c(p, p->logn[2] - 1, p->grid, p->bufA, plen * n1, (int)N2h, plo * n1, n0 * n1);
  stage_end(p, 4);
  if (rc) return rc;
  stage_begin(p, 5);
  rc = launch_pass(p, p->logn[1], p->bufA, p->grid, plen, N2h, (int)N1 + 2, p->inv_c_ext[1], p->twiddle[1], false,
                   plo, n0, 0, (int)n1);
  stage_end(p, 5);
  if (rc) return rc;
  stage_begin(p, 6);
  EnergyArgs ea{p->e_partial, p->e_a, 0, (int)N1 + 2, (int)N2h, 1, (int)N0, (int)N1, (int)N2};
  const int64_t nb = energy_x_pass(p, p->grid, (N1 + 2) * N2h, (int)N0 + 2, p->inv_c_ext[0], ea, (int)plo, (int)plen);
  stage_end(p, 6);
  if (nb < 0) return p->failed ? HPNFFT_E_CUDA : HPNFFT_E_UNSUPPORTED;
  p->e_nparts = nb;
  (void)n2;
  return HPNFFT_OK;
}

int x_pass(Plan* p, const double* in, double* fhat, int64_t inner, int64_t k1_base, int a_lo, int a_len) {
  if (!p->energy)
    return launch_pass(p, p->logn[0], in, fhat, 1, inner, (int)p->N[0], p->inv_c[0], p->twiddle[0], false, 0, 1, a_lo,
                       a_len);
  EnergyArgs ea{p->e_partial, p->e_a, k1_base, (int)p->N[1], (int)p->N[2]};
  const int64_t nb = energy_x_pass(p, in, inner, (int)p->N[0], p->inv_c[0], ea, a_lo, a_len);
  if (nb < 0) return p->failed ? HPNFFT_E_CUDA : HPNFFT_E_UNSUPPORTED;
  p->e_nparts = nb;
  return HPNFFT_OK;
}

}  // namespace hpnfft
