/*
 * hpnfft.h -- C ABI of the B200-native adjoint NFFT (HP-NFFT hot path, arXiv 2001.01583).
 *
 * Operation (§1 Eq. 5):
 *     fhat(k) = sum_{j=0}^{M-1} f_j * exp(-2 pi i k.x_j),   k in I_N,
 *     I_N = { k in Z^3 : -N_t/2 <= k_t < N_t/2 }            (§1)
 * computed by the CUNFFT gridding scheme (§2 Fig. 1; Alg. 2):
 * bin-sort the points, spread each f_j with a Kaiser-Bessel (Gaussian, B-spline, sinc-power) window of 2m taps per
 * dimension onto the sigma-oversampled grid I_n (n_t = sigma N_t), FFT that grid, divide by the
 * window's Fourier weights c_k and crop to I_N ("Scaling", §3).
 * The paper's "NDFT" direction (Eq. 5, minus sign) is called "adjoint" here.
 *
 * Conventions (readings Q1-Q10):
 *   - points x_j in [-0.5, 0.5]^3 (Pi^3); x = 0.5 and x = -0.5 give the same result;
 *   - u_t = n_t x_t, taps l_t = floor(u_t) - m + 1 .. floor(u_t) + m (strict |u - l| < m),
 *     grid offset l_t mod n_t;
 *   - Kaiser-Bessel: b = pi (2 - 1/sigma), Phi(u) = sinh(b sqrt(m^2-u^2)) / (pi sqrt(m^2-u^2)),
 *     c_k = I0(m sqrt(b^2 - (2 pi k/n)^2)); Gaussian: b = 2 sigma/(2 sigma-1) m/pi,
 *     Phi(u) = exp(-u^2/b)/sqrt(pi b), c_k = exp(-b pi^2 k^2/n^2);
 *   - output fhat is row-major [N0][N1][N2] (last dimension fastest) at index k_t + N_t/2,
 *     complex128 stored as interleaved (re, im) doubles; no normalisation.
 *
 * Memory and ownership: unless stated otherwise every data pointer is a CUDA DEVICE pointer
 * (cudaMalloc / torch CUDA tensor memory) that the caller owns.  Calls are asynchronous on the
 * plan's stream (stream order is the only synchronisation): a buffer passed to a call must stay
 * valid until the stream has passed the call.  The plan owns its workspace (grid, FFT buffers,
 * bins, permutation, tables), allocated by hpnfft_plan and released by hpnfft_destroy.
 *
 * Errors: every function returns HPNFFT_OK (0) or a negative status; hpnfft_last_error() gives
 * a thread-local text for the last failure.  Argument validation is synchronous and happens
 * before any launch; a failed hpnfft_plan leaves *out == NULL.  After HPNFFT_E_CUDA/E_NCCL the
 * plan is sticky-failed: every later call except hpnfft_destroy returns HPNFFT_E_STATE.
 * Threading: one host thread per plan at a time; distinct plans are independent.
 */
#ifndef HPNFFT_H_
#define HPNFFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hpnfft_plan_s* hpnfft_plan_t;

/* Windows named by the paper (§4, Fig. 12); formulas in DESIGN.md reading Q21 /
 * csrc/window.cuh (NFFT conventions, window in grid cells, support |u| < m). */
enum {
  HPNFFT_WINDOW_KAISER_BESSEL = 0,
  HPNFFT_WINDOW_GAUSSIAN = 1,
  HPNFFT_WINDOW_B_SPLINE = 2,   /* centred cardinal B-spline M_2m */
  HPNFFT_WINDOW_SINC_POWER = 3  /* sinc(pi beta u)^2m, beta = (2 sigma - 1)/(2 m sigma) */
};

enum {
  HPNFFT_OK = 0,
  HPNFFT_E_INVALID = -1,            /* malformed argument (odd N_t, sigma <= 1, NULL, ...) */
  HPNFFT_E_UNSUPPORTED = -2,        /* valid but not implemented (d != 3, n_t not 2^k, m range) */
  HPNFFT_E_RANGE = -3,              /* a point coordinate outside [-0.5, 0.5] (or NaN) */
  HPNFFT_E_NOMEM = -4,              /* device allocation failed */
  HPNFFT_E_CUDA = -5,               /* CUDA runtime/launch error (plan becomes sticky-failed) */
  HPNFFT_E_NCCL = -6,               /* NCCL missing or an NCCL call failed (multi-GPU plans) */
  HPNFFT_E_STATE = -7,              /* call out of order (adjoint before set_points) or failed plan */
  HPNFFT_E_DEGENERATE_WINDOW = -8   /* a Fourier weight c_k is not finite or below 1e-300 */
};

/* Arithmetic precision of a plan (the FP32 variant). */
enum { HPNFFT_PRECISION_F64 = 0, HPNFFT_PRECISION_F32 = 1 };

/* Spread kernel selection (for measurement; HPNFFT_SPREAD_AUTO is the product default). */
enum { HPNFFT_SPREAD_AUTO = 0, HPNFFT_SPREAD_ATOMIC = 1, HPNFFT_SPREAD_SWEEP = 2 };

/*
 * Create a plan (A0 in SURVEY.md §8(a)): validates, allocates the workspace and builds the
 * per-dimension deconvolution tables 1/c_k, the FFT twiddles and the window tap polynomials
 * in device kernels.
 *   out    : receives the plan handle (host pointer to a handle).
 *   d      : dimension 1, 2 or 3 (I_N and Eq. 5 for any d), else
 *            E_UNSUPPORTED.  A d < 3 plan runs the 3-D kernels with 3 - d trivial leading
 *            dimensions (N_t = n_t = 1, x_t = 0, one tap of weight exactly 1, no FFT pass), on the
 *            generic atomic spread and warp gather; multi-GPU plans and hpnfft_ewald_reciprocal
 *            need d = 3.
 *   N      : HOST array of d bandwidths N_t, each even and >= 2, else E_INVALID.
 *   M      : number of points this plan will be given (0 <= M < 2^31), else E_INVALID.
 *   m      : cut-off, 1 <= m <= 15 (PAPER.md:266 sweeps m = 1..15), else E_UNSUPPORTED.  The DMMA
 *            sweep spread and gather serve m <= 8 (a chunk's CH + 2m - 1 node planes fit the
 *            16-row accumulator); m = 9..15 run the generic atomic spread and warp gather.
 *   sigma  : oversampling factor > 1; n_t = sigma N_t must be an integer power of two >= 2m
 *            (PAPER.md:266 uses sigma = 2), else E_UNSUPPORTED (E_INVALID for sigma <= 1).
 *   window : HPNFFT_WINDOW_KAISER_BESSEL, _GAUSSIAN, _B_SPLINE or _SINC_POWER.
 *   stream : cudaStream_t (as void*) all work is enqueued on; NULL = legacy default stream.
 */
int hpnfft_plan(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma,
                int window, void* stream);

/*
 * Bin-sort the points (A1 keys + A2 counting sort).
 *   x : DEVICE [M][d] float64 row-major, each coordinate in [-0.5, 0.5].  Read only; the plan
 *       keeps its own sorted copy, so x may be released once the stream passes this call.
 * Out-of-range or NaN coordinates return HPNFFT_E_RANGE; this is detected with a device flag
 * that is read back once at the end of the call (the only host synchronisation of the path).
 */
int hpnfft_set_points(hpnfft_plan_t p, const double* x);

/*
 * hpnfft_set_points without the host synchronisation, for pipelines that keep the host ahead of
 * the GPU (e.g. host -> device copies of the next batch overlapping this transform).  The flags
 * are still copied to host memory on the stream, but checked only by the NEXT call of
 * hpnfft_set_points / hpnfft_set_points_async / hpnfft_check_points on this plan, which returns
 * this call's HPNFFT_E_RANGE (or a grid-slab barrier timeout) — a deferred error; the transform of
 * such points is memory-safe but its result is undefined.  Without the read-back the plan cannot
 * prune the unoccupied grid planes: a single-GPU plan spreads and transforms all n0 planes (the
 * same work for points that fill [-1/2, 1/2)), a grid-slab plan its fixed slab + halo planes.
 */
int hpnfft_set_points_async(hpnfft_plan_t p, const double* x);

/* Wait for the flags of the last hpnfft_set_points_async and return its deferred error (or OK). */
int hpnfft_check_points(hpnfft_plan_t p);

/*
 * Transform (A3 window, A4 spread, A5 FFT, A6 deconvolve + crop; Alg. 2).
 *   f    : DEVICE [M][2] float64 (re, im) values in the ORIGINAL point order of set_points.
 *   fhat : DEVICE [N0*...*N_{d-1}][2] float64 output (row-major over the d dimensions), fully
 *          overwritten (no accumulation).
 * Requires a prior successful hpnfft_set_points (else HPNFFT_E_STATE).  Asynchronous.
 */
int hpnfft_adjoint(hpnfft_plan_t p, const double* f, double* fhat);

/*
 * Inverse direction (Eq. 6, §1): the adjoint of Eq. 5's
 * matrix, called "inverse NDFT" in the paper (not a matrix inverse):
 *     f(x_j) = sum_{k in I_N} fhat(k) exp(+2 pi i k.x_j),   j < M,
 * by the inverse CUNFFT of Alg. 5: Subdividing (fhat / c_k into the
 * oversampled spectrum), Inverse FFT, Interpolating (a gather with the same 2m taps per
 * dimension as the spread, no atomics).  Same conventions and error level as hpnfft_adjoint
 * (the two are exact transposes of each other up to rounding).
 *   fhat : DEVICE [N0*N1*N2][2] float64, row-major at index k_t + N_t/2 (the FULL fhat also on
 *          multi-GPU plans: every rank interpolates its own points, Alg. 4).
 *   f    : DEVICE [M][2] float64 output in the ORIGINAL point order of set_points.
 * Requires a prior successful hpnfft_set_points (else HPNFFT_E_STATE).  Uses the plan's grid
 * workspace, so it must not overlap an hpnfft_adjoint of the same plan.  Asynchronous.
 */
int hpnfft_inverse(hpnfft_plan_t p, const double* fhat, double* f);

/*
 * FP32 plans (the lower-precision variant): the same operation (Eq. 5)
 * and conventions in float -- complex64 values, grid, FFT passes and fhat -- on float coordinates.
 * Arguments as hpnfft_plan; m in [1, 8].  Spreading: shared-memory box accumulation (native float
 * shared atomics, one vector float2 reduction per node into the zeroed grid); FFT: the pruned
 * Stockham passes on complex64.  Accuracy: the method's error at m (E2 vs Eq. 5) plus float
 * rounding (~1e-6 relative).  FP32 plans take only the _f32 calls below (plus
 * destroy / last_error / workspace / stream / timing / info); the float64 calls on them (and the
 * _f32 calls on a float64 plan) return HPNFFT_E_INVALID; no inverse, energy or multi-GPU plans.
 */
int hpnfft_plan_f32(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M, int m, double sigma, int window,
                    void* stream);
/* x : DEVICE [M][d] float32 coordinates in [-0.5, 0.5] (as hpnfft_set_points). */
int hpnfft_set_points_f32(hpnfft_plan_t p, const float* x);
/* f : DEVICE [M][2] float32 (re, im) in the original point order; fhat : DEVICE [N0*..][2] float32. */
int hpnfft_adjoint_f32(hpnfft_plan_t p, const float* f, float* fhat);

/* Release the plan and its workspace (synchronises the plan's stream).  NULL is a no-op. */
int hpnfft_destroy(hpnfft_plan_t p);

/* Thread-local text of the last failure (never NULL). */
const char* hpnfft_last_error(void);

/* Bytes of device workspace the plan owns (host query, no synchronisation). */
size_t hpnfft_workspace_bytes(hpnfft_plan_t p);

/* Change the stream later calls enqueue on (cudaStream_t as void*). */
int hpnfft_set_stream(hpnfft_plan_t p, void* stream);

/* Select the spread kernel (HPNFFT_SPREAD_*); AUTO picks the sweep kernel when the grid allows. */
int hpnfft_set_spread_method(hpnfft_plan_t p, int method);

/*
 * Number of kernel launches the last hpnfft_set_points + hpnfft_adjoint enqueued (host counter;
 * used by bench.py for "gpu_launches").
 */
int64_t hpnfft_launch_count(hpnfft_plan_t p);

/*
 * Per-stage device timing (CUDA events on the plan's stream) of the most recent calls, in ms:
 * out[0] keys+histogram, out[1] scan, out[2] scatter, out[3] spread, out[4] FFT pass z,
 * out[5] FFT pass y, out[6] FFT pass x + deconvolve, out[7] point records (part of out[3]),
 * out[8] multi-GPU exchange (the collective, or the halo exchange for HPNFFT_DIST_GRID_SLAB),
 * out[9] HPNFFT_DIST_GRID_SLAB pack + all-to-all, out[10] inverse: subdivide + inverse FFT,
 * out[11] inverse: interpolation.
 * Enabled by hpnfft_enable_timing(p, 1);
 * reading synchronises the stream.  Returns the number of values written (<= n).
 */
int hpnfft_enable_timing(hpnfft_plan_t p, int on);
int hpnfft_stage_times(hpnfft_plan_t p, float* out, int n);

/*
 * Plan facts for measurement (HOST int64 out[n]; returns the number written, <= 8):
 *   out[0..2] algorithmic HBM bytes of the FFT passes z, y, x (+ deconvolve) of this plan's next
 *             hpnfft_adjoint for the current points: each pass reads its input once and writes its
 *             pruned output once (complex128; only the node planes the points reach, the rank's
 *             slab and k1 rows for a grid-slab plan);
 *   out[3]    exchange path: 0 none (one rank), 1 NCCL collective on fhat (option A), 2 grid slab
 *             over NVLink peer memory (CUDA IPC), 3 grid slab over NCCL send/recv, 4 one-GPU rank
 *             group (hpnfft_plan_group);
 *   out[4]    node planes of dimension 0 the passes z and y process;
 *   out[5]    points per record group of the sweep spread ("groups"; M = one group);
 *   out[6]    the spread kernel HPNFFT_SPREAD_AUTO resolves to (HPNFFT_SPREAD_ATOMIC or _SWEEP);
 *   out[7]    workspace bytes.
 */
int hpnfft_plan_info(hpnfft_plan_t p, int64_t* out, int n);

/* Library version string. */
const char* hpnfft_version(void);

/*
 * ENUF reciprocal-space energy (Eq. 12, §5 "HP-ENUF"):
 *   U = 1/(2 pi L) sum_{n in I_N, n != 0} exp(-pi^2 |n|^2 / (alpha L)^2) / |n|^2 |S(n)|^2
 *       - alpha / sqrt(pi) sum_i q_i^2,        S(n) = sum_i q_i exp(-2 pi i n.r_i / L),
 * with the points of the last hpnfft_set_points taken as x_i = r_i / L - 1/2 (so that
 * |S(n)| = |fhat(n)| of Eq. 5 with f_i = q_i).
 *   q     : DEVICE [M] float64 real charges (this rank's points for a multi-GPU plan).
 *   L     : box side (> 0), alpha : Ewald parameter (> 0), in the same length unit.
 *   U     : DEVICE 1 float64, written in stream order (the sum over all ranks for a grid-slab plan;
 *           collective: every rank of a grid-slab plan must call it, it ends with an all-reduce).
 * Runs the adjoint's spread and FFT passes on f_i = q_i + 0i; the last FFT pass sums the weighted
 * |fhat|^2 instead of storing fhat (no fhat buffer); fixed-order reductions (deterministic).
 * Errors: E_INVALID (NULL, L or alpha <= 0), E_STATE (no set_points), E_UNSUPPORTED (a multi-GPU
 * plan other than HPNFFT_DIST_GRID_SLAB), E_NOMEM, E_CUDA, E_NCCL.  Asynchronous.
 */
int hpnfft_ewald_reciprocal(hpnfft_plan_t p, const double* q, double L, double alpha, double* U);

/* ---------------------------------------------------------------------------------------------
 * Multi-GPU (A7 of SURVEY.md §8(a), §8(e)): one process per GPU, NCCL over NVLink/NVSwitch.
 * By Eq. 8 (§3) fhat is linear in the point set: every rank transforms its own
 * points (the paper's subcells) and the partial results are combined by one
 * exchange step ("Accumulate", Alg. 3).  NCCL is loaded at run time
 * (dlopen "libnccl.so.2", so the process shares torch's copy when torch is loaded); a missing
 * NCCL makes hpnfft_get_unique_id / hpnfft_plan_dist return HPNFFT_E_NCCL.
 *
 * Modes (what hpnfft_adjoint leaves in fhat on rank r of P):
 *   HPNFFT_DIST_ALLREDUCE    : the full fhat [N0][N1][N2] on every rank (ncclAllReduce).
 *   HPNFFT_DIST_REDUCE_ROOT0 : the full fhat on rank 0 (ncclReduce, Alg. 3's semantics); the
 *                              buffer of the other ranks holds their own partial transform.
 *   HPNFFT_DIST_REDUCE_SCATTER : fhat[r N0/P .. (r+1) N0/P)[N1][N2] (k0 slab r; N0 % P == 0).
 *   HPNFFT_DIST_GRID_SLAB    : SURVEY.md §8(e) option G.  Rank r owns the x-ordered cell planes
 *       c0x in [r n0/P, (r+1) n0/P), c0x = (floor(n0 x0) + n0/2) mod n0 (the equal-size x-slab
 *       [-1/2 + r/P, -1/2 + (r+1)/P)); all its points must lie there (else
 *       set_points returns HPNFFT_E_RANGE).  The rank spreads into its planes plus the m - 1
 *       planes below and m above, adds the neighbours' halo planes to its own (pulled from their
 *       grids over NVLink peer memory; ncclSend/Recv when peer memory is unavailable), runs the z
 *       and y FFT passes on its own planes only, exchanges blocks all-to-all (the y pass stores
 *       straight into the destination ranks' grids; grouped ncclSend/Recv otherwise) and runs the
 *       x pass on its k1 slab: fhat[N0][r N1/P .. (r+1)
 *       N1/P)[N2] (row-major [N0][N1/P][N2]).  Requires P a power of two, N1 % P == 0 and
 *       n0 / P >= 2m.  Over NVLink peer memory (CUDA IPC, chosen collectively: all ranks agree)
 *       the phases are ordered by cross-GPU flag barriers with a 5 s timeout; after a timeout the
 *       rank touches no peer memory any more, its fhat block is undefined, and its next
 *       hpnfft_set_points returns HPNFFT_E_NCCL (the plan is then failed).
 */
enum {
  HPNFFT_DIST_ALLREDUCE = 0,
  HPNFFT_DIST_REDUCE_ROOT0 = 1,
  HPNFFT_DIST_REDUCE_SCATTER = 2,
  HPNFFT_DIST_GRID_SLAB = 3
};

/* 128-byte NCCL unique id (HOST buffer), created on one rank and given to all ranks by the
 * caller (any channel, e.g. torch.distributed broadcast). */
int hpnfft_get_unique_id(unsigned char id[128]);

/*
 * Create the plan of rank `rank` of `nranks` (arguments as hpnfft_plan; M = this rank's point
 * count).  Initialises an NCCL communicator over the caller's current CUDA device from `id`
 * (HOST, 128 bytes); all ranks must call this collectively.  mode = HPNFFT_DIST_*.
 * Errors: E_INVALID (bad rank/nranks/mode/id), E_UNSUPPORTED (mode constraints above),
 * E_NCCL (NCCL missing or its initialisation failed), plus those of hpnfft_plan.
 */
int hpnfft_plan_dist(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M_local, int m, double sigma,
                     int window, void* stream, int nranks, int rank, const unsigned char id[128], int mode);

/*
 * HPNFFT_DIST_GRID_SLAB only: replace the equal-size slabs by arbitrary cell-plane slabs, e.g.
 * equal-COUNT slabs for clustered points (PAPER.md:93's "subcells with same
 * size" balance the work only for uniform points).  edges: HOST int64[nranks + 1], x-ordered cell
 * planes c0x (as above), cyclic: rank s owns c0x in [edges[s], edges[s+1]) mod n0, with
 * 0 <= edges[0] < n0, edges[nranks] = edges[0] + n0, every slab a multiple of 4 planes and
 * >= 2m planes, and c0x = n0/2 (x = 0, the grid's memory plane 0) one of the edges mod n0 (each
 * slab is then one contiguous plane range of the grid in memory).  Collective in effect: every
 * rank must pass the same edges before its next hpnfft_set_points (which this call invalidates).
 * The default, set by hpnfft_plan_dist, is edges[s] = s n0 / nranks.  The output layout (k1 slabs)
 * does not change.  Errors: E_INVALID (not a grid-slab plan, bad edges), E_CUDA.
 */
int hpnfft_set_slabs(hpnfft_plan_t p, const int64_t* edges);

/*
 * One-GPU rank group: the ranks of a multi-GPU plan emulated as `nranks` plans on the caller's
 * CURRENT device, for validating the exchange code where fewer GPUs than ranks exist (SURVEY.md
 * §8(e); the driver's test box has one GPU).  Member r behaves exactly like rank r of
 * hpnfft_plan_dist in `mode` (same partition rules, hpnfft_set_slabs, hpnfft_set_points,
 * hpnfft_output_shape), except that
 *   - HPNFFT_DIST_GRID_SLAB: the "peer grids" are the group's own plans' grids (no CUDA IPC) and
 *     hpnfft_adjoint_group runs every exchange phase of the peer-memory path (spread, halo pull,
 *     z pass, y pass with stores into the destination members' grids, x pass) for ALL members
 *     before the next phase starts, in stream order on the one stream: the cross-GPU flag
 *     barriers of the real path are replaced by that order, so no kernel ever waits for another;
 *   - option A (ALLREDUCE, REDUCE_ROOT0, REDUCE_SCATTER): every member's partial fhat (Eq. 8 term)
 *     is summed by a device kernel into the same result layout as the NCCL collective.
 *   out : HOST array of nranks handles (filled in rank order; all NULL on failure).
 *   M   : HOST int64[nranks], member r's point count.  Other arguments as hpnfft_plan.
 * All members must stay on one stream and be destroyed together (hpnfft_destroy each).
 * Errors: those of hpnfft_plan / hpnfft_plan_dist (no NCCL is needed).
 */
int hpnfft_plan_group(hpnfft_plan_t* out, int d, const int64_t* N, const int64_t* M, int m, double sigma, int window,
                      void* stream, int nranks, int mode);

/*
 * The adjoint of a one-GPU rank group: f[r] (DEVICE, member r's values in its set_points order)
 * -> fhat[r] (DEVICE, member r's output block, shape hpnfft_output_shape).  plans/f/fhat are HOST
 * arrays of nranks pointers in rank order.  Errors: E_INVALID (not one group in rank order, or
 * members on different streams), E_STATE (a member without set_points), E_CUDA.  Asynchronous.
 */
int hpnfft_adjoint_group(hpnfft_plan_t* plans, int nranks, const double* const* f, double* const* fhat);

/* Shape (HOST int64[3]) of the fhat block hpnfft_adjoint writes on this rank (see the modes); for a
 * d < 3 plan the leading 3 - d entries are 1. */
int hpnfft_output_shape(hpnfft_plan_t p, int64_t shape[3]);

#ifdef __cplusplus
}
#endif

#endif /* HPNFFT_H_ */
