// energy.cu -- SURVEY.md §8(f) NEXT #2: the ENUF reciprocal-space energy of Eq. 12 (PAPER.md:298,
// §5), the paper's application of the adjoint NFFT ("HP-ENUF"):
//     U^{E,K} = 1/(2 pi L) sum_{n in I_N, n != 0} exp(-pi^2 |n|^2 / (alpha L)^2) / |n|^2 S(n) S(-n)
//               - alpha / sqrt(pi) sum_i q_i^2,
//     S(n) = sum_i q_i exp(-2 pi i n.r_i / L)
// For real charges S(-n) = conj(S(n)), and with the plan's points x_i = r_i / L - 1/2 the adjoint
// NFFT gives fhat(n) = S(n) (-1)^{n0+n1+n2}, so S(n) S(-n) = |fhat(n)|^2.  The adjoint runs as
// usual (spread of f_i = q_i + 0i, FFT passes z and y) and its last pass (x) sums the weighted
// |fhat|^2 per CTA instead of storing fhat (fft.cu x_pass); one CTA then adds the partials and
// the self term in a fixed order (deterministic).  Grid-slab multi-GPU plans sum their k1 slabs'
// terms and their own points' self terms, then all-reduce the scalar.
#include <stdlib.h>
#include "common.cuh"

namespace hpnfft {

namespace {

constexpr int kChargeBlocks = 592;   // 4 x 148 SMs, fixed so that the partial order is fixed
constexpr int kThreads = 256;

// f = q + 0i and per-CTA partial sums of q^2 (grid-stride, fixed grid)
__global__ void __launch_bounds__(kThreads) k_charges(const double* __restrict__ q, double2* __restrict__ f, int64_t M,
                                                       double* __restrict__ q2_partial) {
  double s = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)kThreads + threadIdx.x; j < M; j += (int64_t)gridDim.x * kThreads) {
    const double v = q[j];
    f[j] = make_double2(v, 0.0);
    s = fma(v, v, s);
  }
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += red[w];
    q2_partial[blockIdx.x] = t;
  }
}

// U = sum(e partials) / (2 pi L) - alpha / sqrt(pi) sum(q^2 partials), one CTA, fixed order
__global__ void __launch_bounds__(kThreads) k_energy_final(const double* __restrict__ e_partial, int64_t ne,
                                                            const double* __restrict__ q2_partial, int nq,
                                                            double inv_2pi_l, double self_c, double* __restrict__ U,
                                                            const int* __restrict__ dist_err) {
  __shared__ double se[kThreads], sq[kThreads];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < ne; i += kThreads) a += e_partial[i];
  for (int i = threadIdx.x; i < nq; i += kThreads) b += q2_partial[i];
  se[threadIdx.x] = a;
  sq[threadIdx.x] = b;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      se[threadIdx.x] += se[threadIdx.x + w];
      sq[threadIdx.x] += sq[threadIdx.x + w];
    }
    __syncthreads();
  }
  // a timed-out cross-GPU barrier (grid slab): NaN instead of a plausible wrong energy
  const bool bad = dist_err && *dist_err != 0;
  if (threadIdx.x == 0) *U = bad ? __longlong_as_double(0x7ff8000000000000ll) : se[0] * inv_2pi_l - self_c * sq[0];
}

}  // namespace

}  // namespace hpnfft

using namespace hpnfft;

extern "C" int hpnfft_ewald_reciprocal(hpnfft_plan_t h, const double* q, double L, double alpha, double* U) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p || !U || (!q && p->M > 0)) {
    set_error("NULL argument");
    return HPNFFT_E_INVALID;
  }
  if (p->d != 3 || p->precision != HPNFFT_PRECISION_F64) {
    set_error("hpnfft_ewald_reciprocal: needs a float64 d = 3 plan (Eq. 12)");
    return HPNFFT_E_UNSUPPORTED;
  }
  if (!(L > 0.0) || !(alpha > 0.0)) {
    set_error("hpnfft_ewald_reciprocal: need L > 0 and alpha > 0");
    return HPNFFT_E_INVALID;
  }
  if (p->failed) {
    set_error("plan is in a failed state (an earlier CUDA error)");
    return HPNFFT_E_STATE;
  }
  if (!p->points_set) {
    set_error("hpnfft_ewald_reciprocal before a successful hpnfft_set_points");
    return HPNFFT_E_STATE;
  }
  if (p->nranks > 1 && p->dist_mode != HPNFFT_DIST_GRID_SLAB) {
    set_error("hpnfft_ewald_reciprocal: multi-GPU plans need HPNFFT_DIST_GRID_SLAB");
    return HPNFFT_E_UNSUPPORTED;
  }
  // partials: one per x-pass CTA (at most N1 N2 lines) + the charge CTAs
  // + the x pass's weight table (N0 + 2 entries)
  const int64_t need = p->N[1] * p->N[2] + kChargeBlocks + p->N[0] + 2;
  if (p->e_cap < need) {
    cudaFree(p->e_partial);
    p->e_partial = nullptr;
    if (cudaMalloc(&p->e_partial, sizeof(double) * (size_t)need) != cudaSuccess) {
      cudaGetLastError();
      p->e_cap = 0;
      set_error("device allocation of the energy partials failed");
      return HPNFFT_E_NOMEM;
    }
    p->e_cap = need;
  }
  if (!p->fq && p->M > 0) {
    if (cudaMalloc(&p->fq, sizeof(double) * 2 * (size_t)p->M) != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of the charge values failed");
      return HPNFFT_E_NOMEM;
    }
  }
  p->launches = 0;
  double* q2_partial = p->e_partial + p->N[1] * p->N[2];
  p->e_w0 = q2_partial + kChargeBlocks;
  k_charges<<<kChargeBlocks, kThreads, 0, p->stream>>>(q, reinterpret_cast<double2*>(p->fq), p->M, q2_partial);
  p->launches++;
  int rc = check_launch(p, "charges");
  if (rc) return rc;
  const double pi = 3.14159265358979323846;
  p->energy = true;
  p->e_a = pi * pi / ((alpha * L) * (alpha * L));
  p->e_nparts = 0;
  const char* cenv = getenv("HPNFFT_ENERGY_COMPLEX");   // measurement / tests: the complex path
  if (p->nranks <= 1 && !(cenv && cenv[0] == '1')) {
    // one GPU: real charges -> the REAL spread onto a real grid and the R2C path (NEXT #2)
    p->real_values = true;
    rc = spread(p, p->fq);
    if (!rc) rc = energy_r2c(p);
    p->real_values = false;
  } else {
    rc = dist_adjoint(p, p->fq, nullptr);   // grid slab: complex spread + FFT + exchange steps
  }
  p->energy = false;
  if (rc) return rc;
  k_energy_final<<<1, kThreads, 0, p->stream>>>(p->e_partial, p->e_nparts, q2_partial, kChargeBlocks,
                                                 1.0 / (2.0 * pi * L), alpha / std::sqrt(pi), U,
                                                 p->virt ? nullptr : p->dist_err);
  p->launches++;
  rc = check_launch(p, "energy final sum");
  if (rc) return rc;
  return dist_allreduce_sum(p, U, 1);
}
