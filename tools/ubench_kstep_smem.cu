// The sweep consumer's k-step in isolation: operands from shared-memory records (same layout and
// index arithmetic as spread_sweep.cu), 5 DMUL + 8 DMMA per k-step, W warps per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
constexpr int RD = 46, CAP = 160, W = 12, M_ = 6, CH = 4, NT = 4;
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void dmma16(double (&c)[4], double a0, double a1, double b) {
  asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
template <int MODE>
__global__ void k(double* out, int iters) {
  extern __shared__ double sm[];
  __shared__ uint32_t lst[32][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  for (int i = threadIdx.x; i < CAP * RD; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  for (int i = lane; i < 64; i += 32) {
    uint32_t e = (uint32_t)((i * 37 + warp * 11) % CAP);
    lst[warp][i] = e | ((uint32_t)(i & 3) << 9) | ((uint32_t)((i * 5) % 15) << 18) | ((uint32_t)((i * 7) % 15) << 23);
  }
  __syncthreads();
  double acc[NT][4] = {};
  const uint32_t rbase = (uint32_t)__cvta_generic_to_shared(sm);
  const int part = g & 1, bc0 = g >> 1;
  const uint32_t* my = lst[warp];
  auto fetch = [&](int k, double& a0, double& a1, double& fp, double& w2v, double (&w1v)[NT]) {
    const uint32_t en = my[(k + t) & 63];
    const uint32_t ra = rbase + (en & 0x1ffu) * (uint32_t)(RD * 8);
    const int sh = (int)((en >> 9) & 3u) - M_ + 1;
    const int d1 = (int)((en >> 18) & 31u), d2 = (int)((en >> 23) & 31u);
    a0 = lds_f64(ra + 8u * (uint32_t)(4 + ((g - sh) & 15)));
    a1 = lds_f64(ra + 8u * (uint32_t)(4 + ((8 + g - sh) & 15)));
    fp = lds_f64(ra + 8u * (uint32_t)(2 + part));
    w2v = lds_f64(ra + 8u * (uint32_t)(33 + min((unsigned)(d2 - 3 + bc0), 12u)));
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) w1v[nt] = lds_f64(ra + 8u * (uint32_t)(20 + min((unsigned)(d1 - 3 + nt), 12u)));
  };
  auto apply = [&](double a0, double a1, double fp, double w2v, const double (&w1v)[NT]) {
    const double fw2 = fp * w2v;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) dmma16(acc[nt], a0, a1, fw2 * w1v[nt]);
  };
  for (int it = 0; it < iters; ++it) {
    for (int k = 0; k < 64; k += 8) {
      double a0, a1, fp, w2v, w1v[NT], b0, b1, gp, g2v, g1v[NT];
      fetch(k, a0, a1, fp, w2v, w1v);
      fetch(k + 4, b0, b1, gp, g2v, g1v);
      apply(a0, a1, fp, w2v, w1v);
      apply(b0, b1, gp, g2v, g1v);
    }
  }
  double s = 0;
  for (int a = 0; a < NT; ++a) s += acc[a][0] + acc[a][1] + acc[a][2] + acc[a][3];
  if (s == 1234.5) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t smem = CAP * RD * 8;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 200;
  for (int warps : {4, 8, 12, 16, 24}) {
    k<0><<<p.multiProcessorCount, 32 * warps, smem>>>(d, 2);
    cudaEventRecord(e0);
    k<0><<<p.multiProcessorCount, 32 * warps, smem>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double dm = (double)p.multiProcessorCount * warps * iters * 16 * 8;   // DMMA.8x8x4 per warp
    printf("warps/SM %2d: %.3f ms  DMMA work %.2f TFLOP/s (pipe peak ~36.7)\n", warps, ms, dm * 256 * 2 / ms / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
