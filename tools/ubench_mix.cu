// Do DMMA (FP64 tensor core) and DFMA (FP64 pipe) share throughput?  Warps [0, nd) issue DMMA
// m8n8k4, warps [nd, 8) issue independent DFMA chains; report the time of each mix.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix_kernel(double* out, int iters, int nd, int nf) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < nd) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else if (w < nd + nf) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    const double m = 0.999999, q = 1e-7;
    for (int it = 0; it < iters * 16; ++it) {   // 128 DFMA per outer step = 4096 FMA per warp
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], m, q);
    }
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == 1234.5) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048, grid = p.multiProcessorCount;
  int cfg[][2] = {{8, 0}, {0, 8}, {8, 8}, {4, 4}, {8, 4}, {4, 8}, {16, 0}, {0, 16}};
  for (auto& c : cfg) {
    const int nd = c[0], nf = c[1], threads = 32 * (nd + nf);
    mix_kernel<<<grid, threads>>>(d, 8, nd, nf);
    cudaEventRecord(e0);
    mix_kernel<<<grid, threads>>>(d, iters, nd, nf);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // DMMA: 8 per step x 256 FMA x 32? no: m8n8k4 = 8*8*4 = 256 FMA per warp instruction
    double fd = (double)grid * nd * iters * 8 * 256 * 2, ff = (double)grid * nf * iters * 16 * 8 * 32 * 2;
    printf("dmma warps %2d dfma warps %2d: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", nd, nf, ms,
           fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
