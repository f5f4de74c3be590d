// Throughput of the sweep's DMMA k-step pattern: per step 5 DMUL (B operands) + 8 DMMA m8n8k4 with
// distinct A (2) / B (4) operands, vs the plain 8-DMMA loop, at 2..8 warps per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void kstep(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a0 = 1.0 + lane * 1e-9, a1 = 1.0 - lane * 1e-9, fp = 0.5, w2 = 0.25;
  double w1[4] = {1.0, 0.5, 0.25, 0.125};
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) { dmma(c[i], a0, w2); dmma(c[4 + i], a1, w2); }
    } else {
      const double fw2 = fp * w2;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double b = fw2 * w1[i];
        dmma(c[i], a0, b);
        dmma(c[4 + i], a1, b);
      }
      a0 += 1e-12; a1 -= 1e-12; fp *= 0.9999999;   // keep operands changing
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16, 24, 32}) {
      const int grid = p.multiProcessorCount, threads = 32 * warps;
      auto k = mode ? kstep<1> : kstep<0>;
      k<<<grid, threads>>>(d, 8);
      cudaEventRecord(e0);
      k<<<grid, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double fl = (double)grid * warps * iters * 8 * 256 * 2;
      printf("mode %d (%s) warps/SM %2d: %.3f ms  %.2f TFLOP/s (DMMA)\n", mode, mode ? "k-step" : "plain", warps, ms,
             fl / ms / 1e9);
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
