// common.cuh -- plan object, error plumbing and small device helpers of libhpnfft.
// Product code (the CUDA path).  Shares nothing with oracle/ (see DESIGN.md "Boundary").
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hpnfft.h"

namespace hpnfft {

constexpr int kMaxM = 15;         // GPU kernels are instantiated for m = kMinM..kMaxM
constexpr int kMaxSweepM = 8;     // the sweep spread / gather: CH + 2m - 1 <= 16 accumulator rows
constexpr int kMinM = 1;
constexpr int kPolyDeg = 18;      // window tap polynomial degree (<= 2e-14
                                  // of Phi(0) for every window and m = 1..15, incl. the steep m = 1 Gaussian)
constexpr int kNumStages = 12;     // timing slots, see hpnfft_stage_times
constexpr int kRangeSlots = 64;   // slot pairs for the occupied-plane min/max reduction

// Checked build (HPNFFT_CHECKED=1, libhpnfft_checked.so; compute-sanitizer is not available on the
// GPU pool): device-side bounds / protocol assertions that print the failed condition and trap,
// and a deadlock timeout on every mbarrier wait of the sweep.  Compiled out of the product build.
#ifndef HPNFFT_CHECKED
#define HPNFFT_CHECKED 0
#endif
#if HPNFFT_CHECKED
#define HPNFFT_DCHECK(cond)                                                                            \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("HPNFFT_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define HPNFFT_DCHECK(cond) \
  do {                      \
  } while (0)
#endif

struct Dims3 {
  int64_t v[3];
};

// Plan: everything one adjoint transform needs, owned by the library.
struct Plan {
  int d = 3;
  int64_t N[3] = {0, 0, 0};   // bandwidths N_t
  int64_t n[3] = {0, 0, 0};   // oversampled grid n_t = sigma N_t (powers of two)
  int logn[3] = {0, 0, 0};
  int64_t M = 0;
  int m = 6;
  double sigma = 2.0;
  int window = HPNFFT_WINDOW_KAISER_BESSEL;
  int precision = HPNFFT_PRECISION_F64;   // HPNFFT_PRECISION_F32: complex64 grid, FFT, values (NEXT #4)
  cudaStream_t stream = nullptr;
  int spread_method = HPNFFT_SPREAD_AUTO;
  // ENUF reciprocal energy (energy.cu): while `energy` is set, the last FFT pass (x_pass) sums
  // Eq. 12's weighted |fhat|^2 into e_partial[0 .. e_nparts) instead of storing fhat
  bool energy = false;
  double e_a = 0.0;
  double* e_partial = nullptr;
  double* e_w0 = nullptr;   // Eq. 12 x-dimension weights (inside the e_partial allocation)
  int64_t e_nparts = 0, e_cap = 0;
  double* fq = nullptr;   // [M] complex (q, 0) of hpnfft_ewald_reciprocal
  // real values (the ENUF charges, NEXT #2): spread onto a REAL grid [n0][n1][n2] (doubles) and
  // the R2C path of fft.cu (energy_r2c); set only inside hpnfft_ewald_reciprocal
  bool real_values = false;
  bool failed = false;
  bool points_set = false;

  // ---- device workspace (plan-owned) ----
  double* grid = nullptr;       // [n0][n1][n2] complex (2 doubles)
  double* bufA = nullptr;       // [n0][n1][N2] complex (FFT pass z output)
  double* bufB = nullptr;       // [n0][N1][N2] complex (aliases grid)
  double* inv_c[3] = {nullptr, nullptr, nullptr};   // 1/c_k per dim, index k + N/2
  double* twiddle[3] = {nullptr, nullptr, nullptr}; // exp(-2 pi i t/n_t), t < n_t (complex)
  // real-charge energy path (energy_r2c): exp(-2 pi i t/(n2/2)), t < n2/2, and 1/c_k on the
  // extended ranges k in [-N_t/2 - 1, N_t/2] (index k + N_t/2 + 1) of dimensions 0 and 1
  double* twiddle_half = nullptr;
  // FP32 plans: float copies of the twiddle and deconvolution tables
  float* twiddle_f[3] = {nullptr, nullptr, nullptr};
  float* inv_cf[3] = {nullptr, nullptr, nullptr};   // 1/c_k * Phi(0): the float kernels use Phi / Phi(0)
  double* wpeak = nullptr;                          // device Phi(0) (FP32 plans)
  double* inv_c_ext[2] = {nullptr, nullptr};
  double* poly = nullptr;       // window tap polynomials [2m][kPolyDeg+1]
  // bin sort
  int64_t nbins = 0;            // n1 * (n2/8) * n0 bins (sort.cu: key order plane chunk, c1, c2/8, c0)
  int chunk_log = 2;            // log2 of the sweep's plane chunk CH (4 planes for m <= 6)
  uint32_t* bin_count = nullptr;  // [nbins + 1], becomes exclusive prefix (bin_start)
  uint32_t* key = nullptr;        // [M]
  uint32_t* rank = nullptr;       // [M] arrival rank inside the bin
  uint32_t* perm = nullptr;       // [M] sorted position -> original index
  double* xs = nullptr;           // [M][3] sorted coordinates
  void* scan_tmp = nullptr;       // block sums for the scan
  void* sort2_buf = nullptr;      // two-level sort workspace (lazy, large M): keys, indices, coordinates
  int64_t sort2_hist_n = 0;       //   in chunk order + [chunks][blocks] counts + scan block sums
  int64_t scan_tmp_elems = 0;
  double* rec = nullptr;          // point records for the sweep spread [rec_group][22 + 4m]
  int64_t rec_group = 0;          // points per record group (== M unless memory-limited)
  int* group_rows = nullptr;      // [2] device scratch for the multi-group sweep (chunk range)
  int* tile_counter = nullptr;    // sweep tile scheduler counter
  void* tile_sched = nullptr;     // sweep tile order: uint64 keys [16384] + int order [16384] (lazy)
  cudaStream_t side = nullptr;    // side stream: the tile-order kernels overlap the records kernel
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
  const int* sched_order = nullptr;   // tile order prepared for the next sweep launch (or null)
  bool sched_pending = false;         // the next sweep must wait for side_join
  int* err_flag = nullptr;        // device [1 + 2 kRangeSlots]: range-error flag, then slot pairs of
                                  // min / max of the x-ordered cell c0
  cudaEvent_t flags_ev = nullptr;   // recorded after the flag read-back of an async set_points
  bool flags_pending = false;       // an async set_points' flags are not checked yet
  int* err_flag_host = nullptr;   // mapped pinned mirror [1 + 2 kRangeSlots + 1 (dist barrier error)]
  int* err_flag_host_dev = nullptr;   // its device alias
  // occupied l0 planes (circular interval [plane_lo, plane_lo + plane_len) mod n0): planes that
  // receive any tap of the current points.  Planes outside are zero and are skipped by the sweep
  // and the first two FFT passes (x-slab subcells of the multi-GPU layer).
  int64_t plane_lo = 0, plane_len = 0;
  size_t ws_bytes = 0;

  int64_t launches = 0;         // kernel launches since the last set_points

  // ---- multi-GPU (hpnfft_plan_dist; csrc/dist.cu) ----
  int dist_mode = -1;           // HPNFFT_DIST_* or -1 for a single-GPU plan
  int nranks = 1, dist_rank = 0;
  void* comm = nullptr;         // ncclComm_t
  int64_t slab_lo = 0, slab_len = 0;   // GRID_SLAB: owned x-ordered cell planes c0x in [lo, lo + len) mod n0
  int64_t slab_edges[17] = {};        // GRID_SLAB: every rank's slab, c0x in [edges[s], edges[s+1]) mod n0
  double* halo = nullptr;       // GRID_SLAB: received halo planes [2m - 1][n1][n2] complex
  double* partial = nullptr;    // REDUCE_SCATTER: this rank's full partial fhat
  // GRID_SLAB over NVLink peer memory (CUDA IPC): the ranks' grids and barrier flags
  bool p2p = false;
  bool virt = false;                  // member of a one-GPU rank group (hpnfft_plan_group): peers are
                                      // the group's own plans, stream order replaces the barriers
  double** peer_grid = nullptr;       // device array [nranks] (own grid at dist_rank)
  double* peer_grid_host[16] = {};    // host copies (opened IPC pointers, closed at destroy)
  uint32_t* flags = nullptr;          // device [64]: barrier epochs written by the peers
  uint32_t** peer_flags = nullptr;    // device array [nranks]
  uint32_t* peer_flags_host[16] = {};
  uint32_t epoch = 0;
  int* dist_err = nullptr;            // device flag: a cross-GPU barrier timed out

  // timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pool, kNumStages+1 events per call
  int ev_used = 0;
  std::vector<int> ev_slot;     // stage id of each recorded begin/end pair
  std::vector<int> ev_pair;     // pool index of the pair's begin event
  int ev_open[kNumStages] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  double stage_ms_acc[kNumStages] = {0};
  int stage_calls[kNumStages] = {0};
};

void set_error(const std::string& msg);
int fail(Plan* p, int code, const std::string& msg);

// SM count of the calling thread's current device (cached per device)
int device_sm_count();
// raise a kernel's dynamic shared-memory limit to `bytes` on the current device (the attribute is
// set only when it grows: no driver call per launch)
cudaError_t set_max_smem(const void* func, size_t bytes);

// Launch-error check helper: returns HPNFFT_OK or records the CUDA error on the plan.
int check_launch(Plan* p, const char* what);

// timing helpers (no-ops unless p->timing)
void stage_begin(Plan* p, int slot);
void stage_end(Plan* p, int slot);

// kernels' host launchers (each returns HPNFFT_OK or an error code)
int build_tables(Plan* p);
int sort_points(Plan* p, const double* x);
int sort_points_f32(Plan* p, const float* x);   // FP32 plans: float coordinates, same keys
// FP32 plans: shared-memory box spread (spread_f32.cu) and the complex64 FFT passes (fft.cu)
int spread_f32(Plan* p, const float* f);
int fft_and_deconvolve_f32(Plan* p, float* fhat);
// bin keys [k_lo, k_hi) this plan's points may use (a grid-slab rank: its own planes' keys only;
// the bin table is zeroed and scanned over that range only, sort.cu)
void key_range(const Plan* p, uint32_t& k_lo, uint32_t& k_hi);
int spread_atomic(Plan* p, const double* f);
int spread_sweep(Plan* p, const double* f);
bool sweep_supported(const Plan* p);
size_t record_bytes(int m);
int fft_and_deconvolve(Plan* p, double* fhat);
// Eq. 12 for real charges (NEXT #2): R2C z pass + extended y pass + multiplicity-weighted x pass
// over the real grid the REAL spread produced (fft.cu)
int energy_r2c(Plan* p);
// the last (x) pass of the adjoint: lines k1 in [k1_base, k1_base + inner / N2) of B[n0][.][N2],
// deconvolved into fhat, or (p->energy) summed into Eq. 12's partials
int x_pass(Plan* p, const double* in, double* fhat, int64_t inner, int64_t k1_base, int a_lo, int a_len);
// one batched pruned FFT pass along dimension dim (fft.cu, see k_fft_pass)
// (peers: device array of nranks output pointers for the grid-slab y pass over NVLink; NP = N/P)
int fft_pass(Plan* p, int dim, const double* in, double* out, int64_t outer, int64_t inner, bool contig,
             int64_t o_start, int64_t o_total, int a_lo, int a_len, double* const* peers = nullptr, int NP = 1);
// multi-GPU exchange steps (dist.cu)
int dist_adjoint(Plan* p, const double* f, double* fhat);
// grid-slab exchange phases over peer memory (dist.cu; one rank each)
int slab_phase_halo(Plan* p);
int slab_phase_z(Plan* p);
int slab_phase_y(Plan* p);
int slab_phase_x(Plan* p, double* fhat);
void dist_free(Plan* p);
int dist_allreduce_sum(Plan* p, double* buf, int64_t count);
int spread(Plan* p, const double* f);
// inverse direction (Eq. 6): fft.cu subdivide + inverse FFT into the grid, interp.cu interpolation
int subdivide_and_ifft(Plan* p, const double* fhat);
int interpolate(Plan* p, double* f);
int interp_sweep(Plan* p, double* f);   // the DMMA gather sweep (spread_sweep.cu)

}  // namespace hpnfft

#define HPNFFT_CUDA_TRY(p, expr, what)                                       \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      return ::hpnfft::fail((p), HPNFFT_E_CUDA,                              \
                            std::string(what) + ": " + cudaGetErrorString(e_)); \
    }                                                                        \
  } while (0)
