// DMMA m8n8k4 latency on one warp: dependent chain (same accumulator) vs k independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void chain(double* out, int iters, long long* cyc) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[K][2];
  for (int i = 0; i < K; ++i) c[i][0] = c[i][1] = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < K; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < K; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 64); cudaMalloc(&c, 8);
  const int iters = 4096;
  auto run = [&](auto k, int K) {
    k<<<1, 32>>>(d, 16, c);
    k<<<1, 32>>>(d, iters, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("K=%2d independent accumulators: %.1f cycles per DMMA, %.1f cycles per round\n", K,
           (double)h / (iters * K), (double)h / iters);
  };
  run(chain<1>, 1); run(chain<2>, 2); run(chain<4>, 4); run(chain<8>, 8); run(chain<16>, 16);
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
