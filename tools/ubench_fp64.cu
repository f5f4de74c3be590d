// Microbenchmark: FP64 FMA throughput on this GPU (peak for the "alu" roofline).
// Each thread runs 8 independent DFMA chains; grid = 148*k CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  float s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678f) out[0] = s;
}
// shared-memory double atomicAdd throughput (to see whether it is native)
__global__ void smem_atom_kernel(double* out, int iters) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0;
  __syncthreads();
  int idx = (threadIdx.x * 17) & 4095;
  for (int i = 0; i < iters; ++i) { atomicAdd(&buf[idx], 1.0); idx = (idx + 32) & 4095; }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = buf[0];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz smemPerBlockOptin %zu regsPerSM %d\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  double* d; cudaMalloc(&d, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int blocksPerSM : {2, 4, 8}) {
    int grid = p.multiProcessorCount * blocksPerSM, threads = 256;
    dfma_kernel<<<grid, threads>>>(d, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<grid, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)grid * threads * iters * 16 * 8;
    printf("DFMA blocks/SM=%d: %.3f ms  %.2f TFMA/s = %.2f TFLOP/s  (%.1f DFMA/clk/SM at %d MHz)\n", blocksPerSM, ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9,
           fmas / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  {
    int grid = p.multiProcessorCount * 4, threads = 256;
    ffma_kernel<<<grid, threads>>>((float*)d, 16, 1.0000001f, 1e-9f);
    cudaEventRecord(e0);
    ffma_kernel<<<grid, threads>>>((float*)d, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)grid * threads * iters * 16 * 8;
    printf("FFMA: %.3f ms  %.2f TFLOP/s\n", ms, 2 * fmas / ms / 1e9);
  }
  {
    int grid = p.multiProcessorCount * 4, threads = 256, it = 4096;
    smem_atom_kernel<<<grid, threads>>>(d, 16);
    cudaEventRecord(e0);
    smem_atom_kernel<<<grid, threads>>>(d, it);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * threads * it;
    printf("smem f64 atomicAdd: %.3f ms  %.2f Gop/s (%.2f op/clk/SM)\n", ms, ops / ms / 1e6, ops / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3));
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
