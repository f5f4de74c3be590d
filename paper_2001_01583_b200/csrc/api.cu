// api.cu -- the C ABI of include/hpnfft.h: validation, workspace, orchestration.
//
// Per-call structure (Alg. 2 of the paper, without its per-call H2D/D2H and
// allocation: data is device resident and the plan owns its workspace):
//   hpnfft_set_points : keys + histogram -> exclusive scan -> scatter      (sort.cu)
//   hpnfft_adjoint    : spread (spread_sweep.cu / spread_atomic.cu)
//                       -> FFT pass z -> pass y -> pass x + deconvolve    (fft.cu)
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <new>
#include <utility>
#include <string>

#include "common.cuh"

namespace hpnfft {

static thread_local std::string g_last_error = "no error";

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(Plan* p, int code, const std::string& msg) {
  set_error(msg);
  if (p && (code == HPNFFT_E_CUDA || code == HPNFFT_E_NCCL)) p->failed = true;
  return code;
}

int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return 148;
  }
  if (cache[dev] == 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
      cudaGetLastError();
      sms = 148;
    }
    cache[dev] = sms;
  }
  return cache[dev];
}

cudaError_t set_max_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[std::make_pair(func, dev)];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

int check_launch(Plan* p, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(p, HPNFFT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return HPNFFT_OK;
}

// Each stage call owns a begin/end pair of pool events; stages may nest (records inside spread).
void stage_begin(Plan* p, int slot) {
  if (!p->timing || slot < 0 || slot >= kNumStages) return;
  while ((int)p->ev.size() < p->ev_used + 2) {
    cudaEvent_t a;
    cudaEventCreate(&a);
    p->ev.push_back(a);
  }
  cudaEventRecord(p->ev[p->ev_used], p->stream);
  p->ev_open[slot] = p->ev_used;
  p->ev_used += 2;
}

void stage_end(Plan* p, int slot) {
  if (!p->timing || slot < 0 || slot >= kNumStages || p->ev_open[slot] < 0) return;
  cudaEventRecord(p->ev[p->ev_open[slot] + 1], p->stream);
  p->ev_slot.push_back(slot);
  p->ev_pair.push_back(p->ev_open[slot]);
  p->ev_open[slot] = -1;
}

int64_t scan_workspace_elems(int64_t nbins);

// set_points read-back: device flags (+ the multi-GPU barrier error) -> mapped host memory
__global__ void k_flags_to_host(const int* __restrict__ flags, int n, const int* __restrict__ dist_err,
                                volatile int* host) {
  const int t = threadIdx.x;
  if (t < n) host[t] = flags[t];
  if (t == n) host[t] = dist_err ? *dist_err : 0;
  __threadfence_system();
}

// A3 + A4: the sweep when the grid allows it, else the generic atomic kernel (timing slot 3)
int spread(Plan* p, const double* f) {
  if (p->spread_method == HPNFFT_SPREAD_SWEEP && !sweep_supported(p)) {
    set_error("sweep spread kernel not supported for this grid");
    return HPNFFT_E_UNSUPPORTED;
  }
  const bool sweep = (p->spread_method == HPNFFT_SPREAD_SWEEP) ||
                     (p->spread_method == HPNFFT_SPREAD_AUTO && sweep_supported(p));
  stage_begin(p, 3);
  const int rc = sweep ? spread_sweep(p, f) : spread_atomic(p, f);
  stage_end(p, 3);
  return rc;
}

static bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

static void free_plan(Plan* p) {
  if (!p) return;
  if (p->stream) cudaStreamSynchronize(p->stream);
  else cudaDeviceSynchronize();
  cudaFree(p->grid);
  cudaFree(p->bufA);
  for (int t = 0; t < 3; ++t) {
    cudaFree(p->inv_c[t]);
    cudaFree(p->twiddle[t]);
  }
  cudaFree(p->twiddle_half);
  cudaFree(p->wpeak);
  for (int t = 0; t < 3; ++t) {
    cudaFree(p->twiddle_f[t]);
    cudaFree(p->inv_cf[t]);
  }
  cudaFree(p->inv_c_ext[0]);
  cudaFree(p->inv_c_ext[1]);
  cudaFree(p->poly);
  cudaFree(p->bin_count);
  cudaFree(p->key);
  cudaFree(p->rank);
  cudaFree(p->perm);
  cudaFree(p->xs);
  cudaFree(p->scan_tmp);
  cudaFree(p->sort2_buf);
  cudaFree(p->rec);
  cudaFree(p->group_rows);
  cudaFree(p->tile_counter);
  cudaFree(p->tile_sched);
  if (p->side) cudaStreamDestroy(p->side);
  if (p->side_fork) cudaEventDestroy(p->side_fork);
  if (p->side_join) cudaEventDestroy(p->side_join);
  cudaFree(p->err_flag);
  cudaFree(p->fq);
  cudaFree(p->e_partial);
  if (p->err_flag_host) cudaFreeHost(p->err_flag_host);
  if (p->flags_ev) cudaEventDestroy(p->flags_ev);
  dist_free(p);
  for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
  delete p;
}

template <typename T>
static int alloc(Plan* p, T** ptr, size_t count) {
  size_t bytes = sizeof(T) * (count ? count : 1);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("device allocation of ") + std::to_string(bytes) + " bytes failed: " +
              cudaGetErrorString(e));
    return HPNFFT_E_NOMEM;
  }
  p->ws_bytes += bytes;
  return HPNFFT_OK;
}

}  // namespace hpnfft

using namespace hpnfft;

extern "C" {

const char* hpnfft_version(void) { return "hpnfft-b200 0.1 (sm_100a)"; }

const char* hpnfft_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"

namespace hpnfft {
// dst = (float)(src * (scale ? *scale : 1))
__global__ void k_to_float(float* __restrict__ dst, const double* __restrict__ src, int64_t count,
                           const double* __restrict__ scale) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < count) dst[i] = (float)(scale ? src[i] * *scale : src[i]);
}
// FP32 plans: Phi(0) from the tap polynomial of tap m - 1 at t = 0 (s = -1).  The float kernels
// use the window divided by Phi(0) and the deconvolution factors multiplied by it (per
// dimension), which leaves fhat unchanged and keeps the products of three taps inside the float
// range (KB m = 8: Phi(0)^3 ~ 1e45 would overflow)
__global__ void k_window_peak(const double* __restrict__ poly, int m, double* __restrict__ peak) {
  const double* a = poly + (m - 1) * (kPolyDeg + 1);
  double v = a[kPolyDeg];
  for (int j = kPolyDeg - 1; j >= 0; --j) v = fma(v, -1.0, a[j]);
  *peak = v;
}
static int create_plan(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma, int window,
                       void* stream, int precision);
}  // namespace hpnfft

extern "C" {

int hpnfft_plan(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma, int window,
                void* stream) {
  return create_plan(out, d, N, M, m, sigma, window, stream, HPNFFT_PRECISION_F64);
}

int hpnfft_plan_f32(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma, int window,
                    void* stream) {
  if (m > kMaxSweepM) {
    if (out) *out = nullptr;
    set_error("FP32 plans: m must be in [1, 8]");
    return HPNFFT_E_UNSUPPORTED;
  }
  return create_plan(out, d, N, M, m, sigma, window, stream, HPNFFT_PRECISION_F32);
}

}  // extern "C"

namespace hpnfft {

static int create_plan(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma, int window,
                       void* stream, int precision) {
  if (!out) {
    set_error("hpnfft_plan: out is NULL");
    return HPNFFT_E_INVALID;
  }
  *out = nullptr;
  if (!N) {
    set_error("hpnfft_plan: N is NULL");
    return HPNFFT_E_INVALID;
  }
  if (d < 1) {
    set_error("hpnfft_plan: d must be >= 1");
    return HPNFFT_E_INVALID;
  }
  for (int t = 0; t < d; ++t) {
    if (N[t] < 2 || (N[t] & 1)) {
      set_error("invalid bandwidth: every N_t must be even and >= 2 (PAPER.md:27)");
      return HPNFFT_E_INVALID;
    }
  }
  if (d > 3) {
    set_error("d must be 1, 2 or 3");
    return HPNFFT_E_UNSUPPORTED;
  }
  if (M < 0 || M >= (int64_t(1) << 31)) {
    set_error("M must satisfy 0 <= M < 2^31");
    return HPNFFT_E_INVALID;
  }
  if (!(sigma > 1.0)) {
    set_error("sigma must be > 1");
    return HPNFFT_E_INVALID;
  }
  if (window != HPNFFT_WINDOW_KAISER_BESSEL && window != HPNFFT_WINDOW_GAUSSIAN && window != HPNFFT_WINDOW_B_SPLINE &&
      window != HPNFFT_WINDOW_SINC_POWER) {
    set_error("unknown window");
    return HPNFFT_E_INVALID;
  }
  if (m < kMinM || m > kMaxM) {
    set_error("m must be in [" + std::to_string(kMinM) + ", " + std::to_string(kMaxM) + "] for the GPU kernels");
    return HPNFFT_E_UNSUPPORTED;
  }
  // d < 3 (NEXT #4; I_N and Eq. 5 for any d): the d given dimensions are the
  // LAST ones of the internal 3-D layout, the leading 3 - d are trivial (N_t = n_t = 1, x_t = 0,
  // one tap of weight exactly 1, no FFT pass, deconvolution factor 1)
  const int lead = 3 - d;
  int64_t N3[3] = {1, 1, 1};
  for (int t = 0; t < d; ++t) N3[lead + t] = N[t];
  int64_t n[3] = {1, 1, 1};
  for (int t = lead; t < 3; ++t) {
    double nt = sigma * (double)N3[t];
    int64_t ni = (int64_t)(nt + 0.5);
    if (fabs(nt - (double)ni) > 1e-9 || !is_pow2(ni)) {
      set_error("n_t = sigma * N_t must be an integer power of two");
      return HPNFFT_E_UNSUPPORTED;
    }
    if (ni < 4 || ni > 1024) {
      set_error("n_t must be in [4, 1024] for the FFT kernels");
      return HPNFFT_E_UNSUPPORTED;
    }
    n[t] = ni;
  }
  int64_t cells = n[0] * n[1] * n[2];
  Plan* p = new (std::nothrow) Plan();
  if (!p) {
    set_error("host allocation failed");
    return HPNFFT_E_NOMEM;
  }
  p->d = d;
  for (int t = 0; t < 3; ++t) {
    p->N[t] = N3[t];
    p->n[t] = n[t];
    int l = 0;
    while ((int64_t(1) << l) < n[t]) ++l;
    p->logn[t] = l;
  }
  p->M = M;
  p->m = m;
  p->precision = precision;
  p->sigma = sigma;
  p->window = window;
  p->stream = reinterpret_cast<cudaStream_t>(stream);
  int s2 = 0;
  while ((1 << (s2 + 1)) <= 8 && (int64_t(1) << (s2 + 1)) <= n[2]) ++s2;
  // plane chunk of the sweep: CH planes of cells touch CH + 2m - 1 <= 16 node planes (the DMMA
  // accumulator's cyclic window), see spread_sweep.cu
  p->chunk_log = m <= 6 ? 2 : (m == 7 ? 1 : 0);
  if (p->chunk_log > p->logn[0]) p->chunk_log = p->logn[0];   // n0 < CH (d < 3: n0 = 1)
  // one bin per (plane chunk, c1 row, c2 bin) (sort.cu)
  p->nbins = n[1] * (n[2] >> s2) * (n[0] >> p->chunk_log);
  int rc = HPNFFT_OK;
  // complex grid and z-pass buffer: complex128, or complex64 for an FP32 plan
  const size_t cdoubles = precision == HPNFFT_PRECISION_F32 ? 1 : 2;
  rc = rc ? rc : alloc(p, &p->grid, cdoubles * (size_t)cells);
  rc = rc ? rc : alloc(p, &p->bufA, cdoubles * (size_t)(n[0] * n[1] * N3[2]));
  for (int t = 0; t < 3 && !rc; ++t) {
    rc = alloc(p, &p->inv_c[t], (size_t)N3[t]);
    rc = rc ? rc : alloc(p, &p->twiddle[t], 2 * (size_t)n[t]);
  }
  rc = rc ? rc : alloc(p, &p->twiddle_half, (size_t)(n[2] > 1 ? n[2] : 2));
  rc = rc ? rc : alloc(p, &p->inv_c_ext[0], (size_t)(N3[0] + 2));
  rc = rc ? rc : alloc(p, &p->inv_c_ext[1], (size_t)(N3[1] + 2));
  rc = rc ? rc : alloc(p, &p->poly, (size_t)(2 * kMaxM * (kPolyDeg + 1)));
  rc = rc ? rc : alloc(p, &p->bin_count, (size_t)(p->nbins + 1));
  rc = rc ? rc : alloc(p, &p->key, (size_t)M);
  rc = rc ? rc : alloc(p, &p->rank, (size_t)M);
  rc = rc ? rc : alloc(p, &p->perm, (size_t)M);
  rc = rc ? rc : alloc(p, &p->xs, 3 * (size_t)M);
  p->scan_tmp_elems = scan_workspace_elems(p->nbins);
  rc = rc ? rc : alloc(p, reinterpret_cast<uint32_t**>(&p->scan_tmp), (size_t)p->scan_tmp_elems);
  rc = rc ? rc : alloc(p, &p->err_flag, 1 + 2 * kRangeSlots);
  if (!rc) {
    // mapped pinned memory: a kernel writes the flags straight into it, so the read-back at the
    // end of set_points needs no copy engine (a memcpy would queue behind a caller's large D2H)
    cudaError_t e = cudaHostAlloc(&p->err_flag_host, (2 + 2 * kRangeSlots) * sizeof(int), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&p->err_flag_host_dev), p->err_flag_host, 0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->flags_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      set_error("pinned allocation failed");
      rc = HPNFFT_E_NOMEM;
    }
  }
  p->bufB = p->grid;   // pass y output reuses the grid (dead after pass z)
  p->plane_lo = 0;
  p->plane_len = n[0];
  // records for the sweep spread: all M points if they fit in half of the free memory,
  // otherwise groups of points processed one after another
  if (!rc) {
    rc = alloc(p, &p->group_rows, 2);
    rc = rc ? rc : alloc(p, &p->tile_counter, 1);
    p->rec_group = 1;   // provisional so that sweep_supported() only checks the grid shape
    p->rec = reinterpret_cast<double*>(1);
    bool grid_ok = sweep_supported(p);
    p->rec = nullptr;
    p->rec_group = 0;
    if (!rc && grid_ok) {
      size_t rb = record_bytes(m);
      size_t freeb = 0, totalb = 0;
      cudaMemGetInfo(&freeb, &totalb);
      int64_t fit = (int64_t)((freeb / 2) / rb);
      int64_t want = M > 0 ? M : 1;
      int64_t g = want < fit ? want : fit;
      const char* env = getenv("HPNFFT_REC_GROUP");
      if (env && atoll(env) > 0 && atoll(env) < g) g = atoll(env);
      if (g >= 1024 || g == want) {
        if (alloc(p, &p->rec, (size_t)g * (rb / sizeof(double))) == HPNFFT_OK) {
          p->rec_group = g;
        } else {
          p->rec = nullptr;   // the atomic spread is used instead
          set_error("no error");
        }
      }
    }
  }
  if (!rc) rc = build_tables(p);
  if (!rc && precision == HPNFFT_PRECISION_F32) {
    rc = alloc(p, &p->wpeak, 1);
    if (!rc) {
      k_window_peak<<<1, 1, 0, p->stream>>>(p->poly, m, p->wpeak);
      rc = check_launch(p, "window peak");
    }
    for (int t = 0; t < 3 && !rc; ++t) {
      rc = alloc(p, &p->twiddle_f[t], 2 * (size_t)n[t]);
      rc = rc ? rc : alloc(p, &p->inv_cf[t], (size_t)N3[t]);
      if (!rc) {
        k_to_float<<<(unsigned)((2 * n[t] + 255) / 256), 256, 0, p->stream>>>(p->twiddle_f[t], p->twiddle[t], 2 * n[t],
                                                                             nullptr);
        // trivial dimensions (n = 1) keep the factor 1: their single tap is exactly 1, not Phi
        k_to_float<<<(unsigned)((N3[t] + 255) / 256), 256, 0, p->stream>>>(p->inv_cf[t], p->inv_c[t], N3[t],
                                                                          n[t] > 1 ? p->wpeak : nullptr);
        rc = check_launch(p, "float tables");
      }
    }
    if (!rc && cudaStreamSynchronize(p->stream) != cudaSuccess) rc = fail(p, HPNFFT_E_CUDA, "float tables");
  }
  if (rc) {
    free_plan(p);
    return rc;
  }
  *out = reinterpret_cast<hpnfft_plan_t>(p);
  return HPNFFT_OK;
}

}  // namespace hpnfft

extern "C" {

namespace {

// the flags of the last set_points, in the mapped host mirror: range / slab errors, the
// barrier timeout of an earlier grid-slab transform
int check_flags(Plan* p) {
  if (p->err_flag_host[0] == 1) {
    set_error("a point coordinate is outside [-0.5, 0.5] (or NaN)");
    return HPNFFT_E_RANGE;
  }
  if (p->err_flag_host[0] == 2) {
    set_error("a point lies outside this rank's grid slab (HPNFFT_DIST_GRID_SLAB)");
    return HPNFFT_E_RANGE;
  }
  if (p->err_flag_host[1 + 2 * kRangeSlots]) {   // a cross-GPU barrier of an earlier grid-slab transform timed out
    return fail(p, HPNFFT_E_NCCL, "a cross-GPU barrier timed out (peer rank missing)");
  }
  return HPNFFT_OK;
}

// wait for the read-back of the last async set_points and report its deferred error
int check_pending(Plan* p) {
  if (!p->flags_pending) return HPNFFT_OK;
  p->flags_pending = false;
  HPNFFT_CUDA_TRY(p, cudaEventSynchronize(p->flags_ev), "set_points flag event");
  return check_flags(p);
}

int set_points(Plan* p, const double* x, bool async, const float* xf = nullptr) {
  if (p->failed) {
    set_error("plan is in a failed state (an earlier CUDA error)");
    return HPNFFT_E_STATE;
  }
  if (!x && !xf && p->M > 0) {
    set_error("x is NULL");
    return HPNFFT_E_INVALID;
  }
  int rc = check_pending(p);
  if (rc) return rc;
  p->points_set = false;
  p->launches = 0;
  rc = xf ? sort_points_f32(p, xf) : sort_points(p, x);
  if (rc) return rc;
  k_flags_to_host<<<1, 2 + 2 * kRangeSlots, 0, p->stream>>>(p->err_flag, 1 + 2 * kRangeSlots, p->dist_err,
                                                             p->err_flag_host_dev);
  p->launches++;
  rc = check_launch(p, "flag read-back");
  if (rc) return rc;
  const int64_t n0 = p->n[0];
  const bool slab = p->dist_mode == HPNFFT_DIST_GRID_SLAB && p->nranks > 1;
  if (async) {
    HPNFFT_CUDA_TRY(p, cudaEventRecord(p->flags_ev, p->stream), "set_points flag event");
    p->flags_pending = true;
    p->plane_lo = 0;   // no read-back of the occupied planes: all of them
    p->plane_len = n0;
  } else {
    HPNFFT_CUDA_TRY(p, cudaStreamSynchronize(p->stream), "set_points sync");
    rc = check_flags(p);
    if (rc) return rc;
    // occupied planes: taps of cells c0 reach l0 = c0 - m + 1 .. c0 + m
    int64_t lo = 0x7fffffff, hi = -1;
    for (int sl = 0; sl < kRangeSlots; ++sl) {
      lo = lo < p->err_flag_host[1 + 2 * sl] ? lo : p->err_flag_host[1 + 2 * sl];
      hi = hi > p->err_flag_host[2 + 2 * sl] ? hi : p->err_flag_host[2 + 2 * sl];
    }
    const int64_t len = hi - lo + 2 * p->m;
    if (p->M == 0 || hi < lo || len >= n0) {
      p->plane_lo = 0;
      p->plane_len = n0;
    } else {
      p->plane_lo = ((lo - n0 / 2 - p->m + 1) % n0 + n0) % n0;
      p->plane_len = len;
    }
  }
  if (slab) {
    // grid-slab plans spread exactly their own cell planes plus the halo the taps reach (a
    // point outside the slab was flagged by k_keys: its key is outside the slab's key range)
    p->plane_lo = ((p->slab_lo - n0 / 2 - p->m + 1) % n0 + n0) % n0;
    p->plane_len = p->slab_len + 2 * p->m - 1;
  }
  p->points_set = true;
  return HPNFFT_OK;
}

}  // namespace

static int precision_guard(Plan* p, int want) {
  if (p->precision != want) {
    set_error(want == HPNFFT_PRECISION_F64 ? "an FP32 plan takes the _f32 calls (float x, complex64 f, fhat)"
                                           : "the _f32 calls need a plan made by hpnfft_plan_f32");
    return HPNFFT_E_INVALID;
  }
  return HPNFFT_OK;
}

int hpnfft_set_points(hpnfft_plan_t h, const double* x) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F64)) return rc;
  return set_points(p, x, false);
}

int hpnfft_set_points_f32(hpnfft_plan_t h, const float* x) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F32)) return rc;
  return set_points(p, nullptr, false, x);
}

int hpnfft_adjoint_f32(hpnfft_plan_t h, const float* f, float* fhat) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F32)) return rc;
  if (p->failed) {
    set_error("plan is in a failed state (an earlier CUDA error)");
    return HPNFFT_E_STATE;
  }
  if (!p->points_set) {
    set_error("hpnfft_adjoint_f32 called before a successful hpnfft_set_points_f32");
    return HPNFFT_E_STATE;
  }
  if (!fhat || (!f && p->M > 0)) {
    set_error("f or fhat is NULL");
    return HPNFFT_E_INVALID;
  }
  stage_begin(p, 3);
  int rc = spread_f32(p, f);
  stage_end(p, 3);
  if (rc) return rc;
  return fft_and_deconvolve_f32(p, fhat);
}

int hpnfft_set_points_async(hpnfft_plan_t h, const double* x) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F64)) return rc;
  return set_points(p, x, true);
}

int hpnfft_check_points(hpnfft_plan_t h) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  return check_pending(p);
}

int hpnfft_adjoint(hpnfft_plan_t h, const double* f, double* fhat) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (p->failed) {
    set_error("plan is in a failed state (an earlier CUDA error)");
    return HPNFFT_E_STATE;
  }
  if (!p->points_set) {
    set_error("hpnfft_adjoint called before a successful hpnfft_set_points");
    return HPNFFT_E_STATE;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F64)) return rc;
  if (!fhat || (!f && p->M > 0)) {
    set_error("f or fhat is NULL");
    return HPNFFT_E_INVALID;
  }
  if (p->dist_mode >= 0) return dist_adjoint(p, f, fhat);
  int rc = spread(p, f);
  if (rc) return rc;
  return fft_and_deconvolve(p, fhat);
}

int hpnfft_inverse(hpnfft_plan_t h, const double* fhat, double* f) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (p->failed) {
    set_error("plan is in a failed state (an earlier CUDA error)");
    return HPNFFT_E_STATE;
  }
  if (!p->points_set) {
    set_error("hpnfft_inverse called before a successful hpnfft_set_points");
    return HPNFFT_E_STATE;
  }
  if (int rc = precision_guard(p, HPNFFT_PRECISION_F64)) return rc;
  if (!fhat || (!f && p->M > 0)) {
    set_error("fhat or f is NULL");
    return HPNFFT_E_INVALID;
  }
  stage_begin(p, 10);
  int rc = subdivide_and_ifft(p, fhat);
  stage_end(p, 10);
  if (rc) return rc;
  stage_begin(p, 11);
  // the tensor-core gather sweep when the grid allows it (HPNFFT_INTERP=warp forces the
  // warp-per-point gather of interp.cu)
  static const bool force_warp = getenv("HPNFFT_INTERP") && getenv("HPNFFT_INTERP")[0] == 'w';
  const bool sweep = !force_warp && p->spread_method != HPNFFT_SPREAD_ATOMIC && sweep_supported(p);
  rc = sweep ? interp_sweep(p, f) : interpolate(p, f);
  stage_end(p, 11);
  return rc;
}

int hpnfft_destroy(hpnfft_plan_t h) {
  free_plan(reinterpret_cast<Plan*>(h));
  return HPNFFT_OK;
}

size_t hpnfft_workspace_bytes(hpnfft_plan_t h) {
  Plan* p = reinterpret_cast<Plan*>(h);
  return p ? p->ws_bytes : 0;
}

int hpnfft_set_stream(hpnfft_plan_t h, void* stream) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  p->stream = reinterpret_cast<cudaStream_t>(stream);
  return HPNFFT_OK;
}

int hpnfft_set_spread_method(hpnfft_plan_t h, int method) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  if (method < HPNFFT_SPREAD_AUTO || method > HPNFFT_SPREAD_SWEEP) {
    set_error("unknown spread method");
    return HPNFFT_E_INVALID;
  }
  p->spread_method = method;
  return HPNFFT_OK;
}

int64_t hpnfft_launch_count(hpnfft_plan_t h) {
  Plan* p = reinterpret_cast<Plan*>(h);
  return p ? p->launches : -1;
}

int hpnfft_plan_info(hpnfft_plan_t h, int64_t* out, int n) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p || !out) {
    set_error("NULL argument");
    return HPNFFT_E_INVALID;
  }
  const int64_t c = 16;   // complex128
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2], N0 = p->N[0], N1 = p->N[1], N2 = p->N[2];
  const bool slab = p->dist_mode == HPNFFT_DIST_GRID_SLAB && p->nranks > 1;
  const int64_t L = slab ? p->slab_len : p->plane_len;   // node planes of passes z and y
  const int64_t N1r = slab ? N1 / p->nranks : N1;        // k1 rows of pass x
  const int64_t xin = slab ? n0 : p->plane_len;          // planes pass x reads
  int64_t v[8];
  v[0] = c * L * n1 * (n2 + N2);
  v[1] = c * L * N2 * (n1 + N1);
  v[2] = c * N1r * N2 * (xin + N0);
  v[3] = p->nranks <= 1 ? 0 : (!slab ? 1 : (p->virt ? 4 : (p->p2p ? 2 : 3)));
  v[4] = p->plane_len;
  v[5] = p->rec_group;
  v[6] = (p->spread_method == HPNFFT_SPREAD_ATOMIC || (p->spread_method == HPNFFT_SPREAD_AUTO && !sweep_supported(p)))
             ? HPNFFT_SPREAD_ATOMIC
             : HPNFFT_SPREAD_SWEEP;
  v[7] = (int64_t)p->ws_bytes;
  int w = 0;
  for (; w < n && w < 8; ++w) out[w] = v[w];
  return w;
}

int hpnfft_enable_timing(hpnfft_plan_t h, int on) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p) {
    set_error("NULL plan");
    return HPNFFT_E_INVALID;
  }
  p->timing = on != 0;
  return HPNFFT_OK;
}

int hpnfft_stage_times(hpnfft_plan_t h, float* out, int nout) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p || !out) {
    set_error("NULL argument");
    return HPNFFT_E_INVALID;
  }
  HPNFFT_CUDA_TRY(p, cudaStreamSynchronize(p->stream), "timing sync");
  double acc[kNumStages] = {0};
  int cnt[kNumStages] = {0};
  for (size_t pair = 0; pair < p->ev_slot.size(); ++pair) {
    float ms = 0;
    cudaEventElapsedTime(&ms, p->ev[p->ev_pair[pair]], p->ev[p->ev_pair[pair] + 1]);
    int sl = p->ev_slot[pair];
    if (sl >= 0 && sl < kNumStages) {
      acc[sl] += ms;
      cnt[sl] += 1;
    }
  }
  p->ev_slot.clear();
  p->ev_pair.clear();
  p->ev_used = 0;
  int w = 0;
  for (int s = 0; s < kNumStages && w < nout; ++s, ++w) out[w] = cnt[s] ? (float)(acc[s] / cnt[s]) : 0.0f;
  return w;
}

}  // extern "C"
