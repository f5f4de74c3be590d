// gen.cu -- device twin of inputs/__init__.py (seeded synthetic inputs).  NOT part of the
// product path and holds none of the method's arithmetic: it only draws the same counter-based
// splitmix64 random numbers as the numpy generator, bit for bit, so large benchmark inputs can
// be created directly in HBM.  Built into inputs/libhpnfft_inputs.so.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull, MIX1 = 0xBF58476D1CE4E5B9ull, MIX2 = 0x94D049BB133111EBull,
                   STREAM_MUL = 0xD1B54A32D192ED03ull;
constexpr int STREAM_X = 0, STREAM_F_RE = 3, STREAM_F_IM = 4, STREAM_IRWIN = 16;

__device__ __forceinline__ uint64_t u64(uint64_t seed, uint64_t stream, uint64_t j) {
  uint64_t z = (seed * GOLDEN ^ stream * STREAM_MUL) + (j + 1) * GOLDEN;
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t stream, uint64_t j) {
  return __dmul_rn((double)(u64(seed, stream, j) >> 11), 1.1102230246251565404236316680908203125e-16);
}

__global__ void k_uniform_points(double* x, int64_t M, int64_t start, uint64_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  uint64_t j = (uint64_t)(start + i);
  for (int t = 0; t < 3; ++t) x[3 * i + t] = __dsub_rn(uniform01(seed, STREAM_X + t, j), 0.5);
}
__global__ void k_uniform_values(double* f, int64_t M, int64_t start, uint64_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  uint64_t j = (uint64_t)(start + i);
  f[2 * i] = __dsub_rn(uniform01(seed, STREAM_F_RE, j), 0.5);
  f[2 * i + 1] = __dsub_rn(uniform01(seed, STREAM_F_IM, j), 0.5);
}
// x = wrap(c_{j mod K} + s z), z = sum_{r<12} U_r - 6, wrap(v) = v - floor(v + 0.5)
__global__ void k_clustered_points(double* x, int64_t M, int64_t start, uint64_t seed, const double* centers, int K,
                                   double s) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  uint64_t j = (uint64_t)(start + i);
  int c = (int)(j % (uint64_t)K);
  for (int t = 0; t < 3; ++t) {
    double z = 0.0;
    for (int r = 0; r < 12; ++r) z = __dadd_rn(z, uniform01(seed, STREAM_IRWIN + 12 * t + r, j));
    z = __dsub_rn(z, 6.0);
    double v = __dadd_rn(centers[3 * c + t], __dmul_rn(s, z));
    x[3 * i + t] = __dsub_rn(v, floor(__dadd_rn(v, 0.5)));
  }
}
}  // namespace

extern "C" {
int hpnfft_gen_uniform_points(double* x, int64_t M, int64_t start, uint64_t seed, void* stream) {
  if (M <= 0) return 0;
  k_uniform_points<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, M, start, seed);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
int hpnfft_gen_uniform_values(double* f, int64_t M, int64_t start, uint64_t seed, void* stream) {
  if (M <= 0) return 0;
  k_uniform_values<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(f, M, start, seed);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
int hpnfft_gen_clustered_points(double* x, int64_t M, int64_t start, uint64_t seed, const double* centers, int K,
                                double s, void* stream) {
  if (M <= 0) return 0;
  k_clustered_points<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(x, M, start, seed, centers, K, s);
  return cudaGetLastError() == cudaSuccess ? 0 : -5;
}
}
