// FP64 and shared-memory latency microbenchmark (one warp, dependent chains, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7) % 1024;
  __syncthreads();
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, 1e-9);   // dependent DFMA chain
  long long t1 = clock64();
  double y = threadIdx.x + 1;
  for (int i = 0; i < iters; ++i) y = y * a;              // dependent DMUL chain
  long long t2 = clock64();
  int idx = threadIdx.x & 1;                              // dependent LDS chain (pointer chase)
  for (int i = 0; i < iters; ++i) idx = (int)sm[idx];
  long long t3 = clock64();
  float z = threadIdx.x;
  for (int i = 0; i < iters; ++i) z = fmaf(z, (float)a, 1e-9f);
  long long t4 = clock64();
  out[threadIdx.x] = x + y + idx + z;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 4096); cudaMalloc(&c, 64);
  int it = 4096;
  lat<<<1, 32>>>(d, c, 1.0000001, 16);
  lat<<<1, 32>>>(d, c, 1.0000001, it);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("latency (cycles/op, 1 warp): DFMA %.1f  DMUL %.1f  LDS(pointer chase) %.1f  FFMA %.1f\n", (double)h[0] / it,
         (double)h[1] / it, (double)h[2] / it, (double)h[3] / it);
  return 0;
}
