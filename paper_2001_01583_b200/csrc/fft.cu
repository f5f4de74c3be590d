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

struct cplx {
  double x, y;
};

__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
__device__ __forceinline__ cplx mul_minus_i(cplx a) { return {a.y, -a.x}; }   // a * (-i)

template <int R>
__device__ __forceinline__ void dft(cplx* v);

template <>
__device__ __forceinline__ void dft<2>(cplx* v) {
  cplx a = v[0], b = v[1];
  v[0] = cadd(a, b);
  v[1] = csub(a, b);
}

template <>
__device__ __forceinline__ void dft<4>(cplx* v) {
  cplx t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
  cplx t2 = cadd(v[1], v[3]), t3 = mul_minus_i(csub(v[1], v[3]));
  v[0] = cadd(t0, t2);
  v[2] = csub(t0, t2);
  v[1] = cadd(t1, t3);
  v[3] = csub(t1, t3);
}

template <>
__device__ __forceinline__ void dft<8>(cplx* v) {
  const double h = 0.70710678118654752440084436210484903;
  cplx e[4] = {v[0], v[2], v[4], v[6]};
  cplx o[4] = {v[1], v[3], v[5], v[7]};
  dft<4>(e);
  dft<4>(o);
  // twiddles W8^k = exp(-i pi k/4)
  cplx o1 = {h * (o[1].x + o[1].y), h * (o[1].y - o[1].x)};
  cplx o2 = mul_minus_i(o[2]);
  cplx o3 = {h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y)};
  v[0] = cadd(e[0], o[0]);
  v[4] = csub(e[0], o[0]);
  v[1] = cadd(e[1], o1);
  v[5] = csub(e[1], o1);
  v[2] = cadd(e[2], o2);
  v[6] = csub(e[2], o2);
  v[3] = cadd(e[3], o3);
  v[7] = csub(e[3], o3);
}

// One Stockham stage of radix R on a tile whose column `col` holds the line; `tj` in
// [0, n/8) is this thread's butterfly slot (8/R butterflies per thread).
template <int LOGN, int R, int TI>
__device__ __forceinline__ void stockham_stage(cplx* buf, int col, int tj, int Ns, const cplx* __restrict__ tw) {
  constexpr int n = 1 << LOGN;
  constexpr int BPT = (n >= 8 ? 8 : n) / R;   // butterflies per thread
  constexpr int T = (n >= 8 ? n / 8 : 1);     // threads per column
  cplx v[BPT][R];
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    int j = tj + b * T;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = buf[(j + r * (n / R)) * (TI + 1) + col];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    int j = tj + b * T;
    int jm = j % Ns;
    if (Ns > 1) {
      int step = jm * (n / (Ns * R));
#pragma unroll
      for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], tw[(step * r) & (n - 1)]);
    }
    dft<R>(v[b]);
    int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[(idxD + r * Ns) * (TI + 1) + col] = v[b][r];
  }
  __syncthreads();
}

template <int LOGN, int TI>
__device__ __forceinline__ void fft_tile(cplx* buf, int col, int tj, const cplx* __restrict__ tw) {
  // radix plan: as many radix-8 stages as possible; the remainder is one radix-4 or radix-2
  // stage, or two radix-4 stages when LOGN % 3 == 1 and LOGN >= 4.
  constexpr int n8 = LOGN / 3 - ((LOGN % 3 == 1 && LOGN >= 4) ? 1 : 0);
  constexpr int rem = LOGN - 3 * n8;
  int Ns = 1;
  if constexpr (n8 > 0) {
#pragma unroll
    for (int s = 0; s < n8; ++s) {
      stockham_stage<LOGN, 8, TI>(buf, col, tj, Ns, tw);
      Ns *= 8;
    }
  }
  if constexpr (rem == 4) {
    stockham_stage<LOGN, 4, TI>(buf, col, tj, Ns, tw);
    Ns *= 4;
    stockham_stage<LOGN, 4, TI>(buf, col, tj, Ns, tw);
  } else if constexpr (rem == 2) {
    stockham_stage<LOGN, 4, TI>(buf, col, tj, Ns, tw);
  } else if constexpr (rem == 1) {
    stockham_stage<LOGN, 2, TI>(buf, col, tj, Ns, tw);
  }
}

// Batched pruned pass.  Lines are indexed by (outer o, column i); element a of a line sits at
//   in + (o * n + a) * inner + i                (inner > 1: strided pass)
// and for the contiguous pass (CONTIG, inner == 1) the TI columns of a CTA are TI consecutive
// outers.  Output k' in [0,N) goes to out + (o * N + k') * inner + i, scaled by inv_c[k'].
template <int LOGN, int TI, bool CONTIG>
__global__ void __launch_bounds__(TI*((1 << LOGN) >= 8 ? (1 << LOGN) / 8 : 1))
k_fft_pass(const cplx* __restrict__ in, cplx* __restrict__ out, int64_t outer, int64_t inner, int N,
           const double* __restrict__ inv_c, const cplx* __restrict__ tw) {
  constexpr int n = 1 << LOGN;
  constexpr int T = (n >= 8 ? n / 8 : 1);
  constexpr int NT = TI * T;
  extern __shared__ cplx smem[];
  cplx* buf = smem;
  const int tid = threadIdx.x;

  int64_t o, i0;
  int cols;
  if (CONTIG) {
    o = (int64_t)blockIdx.x * TI;          // first outer of this CTA
    i0 = 0;
    cols = (int)((outer - o) < TI ? (outer - o) : TI);
  } else {
    int64_t tiles_per_outer = (inner + TI - 1) / TI;
    o = blockIdx.x / tiles_per_outer;
    i0 = (blockIdx.x % tiles_per_outer) * TI;
    cols = (int)((inner - i0) < TI ? (inner - i0) : TI);
  }

  // ---- load the n x TI tile (coalesced along the contiguous direction) ----
  if (CONTIG) {
    const cplx* src = in + o * n;
    for (int e = tid; e < TI * n; e += NT) {
      int c = e >> LOGN, a = e & (n - 1);
      if (c < cols) buf[a * (TI + 1) + c] = src[(int64_t)c * n + a];
    }
  } else {
    const cplx* src = in + o * (int64_t)n * inner + i0;
    for (int e = tid; e < TI * n; e += NT) {
      int a = e / TI, c = e % TI;
      if (c < cols) buf[a * (TI + 1) + c] = src[(int64_t)a * inner + c];
    }
  }
  __syncthreads();

  fft_tile<LOGN, TI>(buf, tid % TI, tid / TI, tw);

  // ---- pruned, scaled store: k' in [0, N) <- grid frequency q = (k' - N/2) mod n ----
  if (CONTIG) {
    cplx* dst = out + o * (int64_t)N;
    for (int e = tid; e < TI * N; e += NT) {
      int c = e / N, k = e % N;
      if (c < cols) {
        int q = (k < N / 2) ? (n - N / 2 + k) : (k - N / 2);
        cplx v = buf[q * (TI + 1) + c];
        double s = inv_c[k];
        dst[(int64_t)c * N + k] = {v.x * s, v.y * s};
      }
    }
  } else {
    cplx* dst = out + o * (int64_t)N * inner + i0;
    for (int e = tid; e < TI * N; e += NT) {
      int k = e / TI, c = e % TI;
      if (c < cols) {
        int q = (k < N / 2) ? (n - N / 2 + k) : (k - N / 2);
        cplx v = buf[q * (TI + 1) + c];
        double s = inv_c[k];
        dst[(int64_t)k * inner + c] = {v.x * s, v.y * s};
      }
    }
  }
}

template <int LOGN>
constexpr int tile_cols() {
  return (1 << LOGN) >= 1024 ? 4 : ((4096 >> LOGN) > 64 ? 64 : (4096 >> LOGN));
}

template <int LOGN>
static int launch_pass_n(Plan* p, const cplx* in, cplx* out, int64_t outer, int64_t inner, int N,
                         const double* inv_c, const cplx* tw, bool contig) {
  constexpr int TI = tile_cols<LOGN>();
  constexpr int n = 1 << LOGN;
  constexpr int NT = TI * (n >= 8 ? n / 8 : 1);
  size_t smem = (size_t)n * (TI + 1) * sizeof(cplx);
  int64_t blocks = contig ? (outer + TI - 1) / TI : outer * ((inner + TI - 1) / TI);
  if (blocks <= 0) return HPNFFT_OK;
  if (contig) {
    auto kern = k_fft_pass<LOGN, TI, true>;
    HPNFFT_CUDA_TRY(p, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "fft smem attr");
    kern<<<(unsigned)blocks, NT, smem, p->stream>>>(in, out, outer, inner, N, inv_c, tw);
  } else {
    auto kern = k_fft_pass<LOGN, TI, false>;
    HPNFFT_CUDA_TRY(p, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "fft smem attr");
    kern<<<(unsigned)blocks, NT, smem, p->stream>>>(in, out, outer, inner, N, inv_c, tw);
  }
  p->launches++;
  return check_launch(p, "fft pass");
}

static int launch_pass(Plan* p, int logn, const double* in, double* out, int64_t outer, int64_t inner, int N,
                       const double* inv_c, const double* tw, bool contig) {
  const cplx* ci = reinterpret_cast<const cplx*>(in);
  cplx* co = reinterpret_cast<cplx*>(out);
  const cplx* ct = reinterpret_cast<const cplx*>(tw);
  switch (logn) {
    case 2: return launch_pass_n<2>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 3: return launch_pass_n<3>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 4: return launch_pass_n<4>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 5: return launch_pass_n<5>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 6: return launch_pass_n<6>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 7: return launch_pass_n<7>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 8: return launch_pass_n<8>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 9: return launch_pass_n<9>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    case 10: return launch_pass_n<10>(p, ci, co, outer, inner, N, inv_c, ct, contig);
    default:
      set_error("FFT length not supported");
      return HPNFFT_E_UNSUPPORTED;
  }
}

int fft_and_deconvolve(Plan* p, double* fhat) {
  const int64_t n0 = p->n[0], n1 = p->n[1];
  const int64_t N0 = p->N[0], N1 = p->N[1], N2 = p->N[2];
  int rc;
  stage_begin(p, 4);
  rc = launch_pass(p, p->logn[2], p->grid, p->bufA, n0 * n1, 1, (int)N2, p->inv_c[2], p->twiddle[2], true);
  stage_end(p, 4);
  if (rc) return rc;
  stage_begin(p, 5);
  rc = launch_pass(p, p->logn[1], p->bufA, p->bufB, n0, N2, (int)N1, p->inv_c[1], p->twiddle[1], false);
  stage_end(p, 5);
  if (rc) return rc;
  stage_begin(p, 6);
  rc = launch_pass(p, p->logn[0], p->bufB, fhat, 1, N1 * N2, (int)N0, p->inv_c[0], p->twiddle[0], false);
  stage_end(p, 6);
  (void)N0;
  return rc;
}

}  // namespace hpnfft
