// dist.cu -- A7 of SURVEY.md §8(a) / §8(e): the multi-GPU exchange steps, NCCL over NVLink.
//
// By Eq. 8 (§3) fhat is linear in the point set, so every rank transforms its
// own points (the paper's equal-size subcells) and the partial results are summed
// ("Accumulate", Alg. 3; the paper's binomial tree of MPI Send/Recv becomes
// one NCCL collective).  Modes (include/hpnfft.h):
//   ALLREDUCE / REDUCE_ROOT0 / REDUCE_SCATTER : SURVEY.md §8(e) option A, sum of the partial fhat;
//   GRID_SLAB : option G, sum of the overlapping grid halos + a distributed pruned FFT:
//       spread (own cell planes + halo) -> halo send/recv + add -> FFT z, y on own planes ->
//       pack -> all-to-all -> FFT x (+ deconvolve) on this rank's k1 slab.
// NCCL is resolved at run time with dlopen("libnccl.so.2"): inside a torch process this is the
// copy torch already loaded; the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <string.h>

#include <stdlib.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace hpnfft {

namespace {

// ---- the subset of the NCCL C API used here (stable ABI since NCCL 2.7) ----
struct NcclUid {
  char internal[128];
};
typedef void* NcclComm;
typedef int NcclResult;                 // ncclSuccess = 0
constexpr int kNcclFloat64 = 8;         // ncclFloat64
constexpr int kNcclSum = 0;             // ncclSum

struct NcclApi {
  NcclResult (*GetUniqueId)(NcclUid*);
  NcclResult (*CommInitRank)(NcclComm*, int, NcclUid, int);
  NcclResult (*CommDestroy)(NcclComm);
  NcclResult (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
  NcclResult (*Reduce)(const void*, void*, size_t, int, int, int, NcclComm, cudaStream_t);
  NcclResult (*ReduceScatter)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
  NcclResult (*AllGather)(const void*, void*, size_t, int, NcclComm, cudaStream_t);
  NcclResult (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t);
  NcclResult (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t);
  NcclResult (*GroupStart)();
  NcclResult (*GroupEnd)();
  const char* (*GetErrorString)(NcclResult);
  bool ok;
};

const NcclApi* nccl() {
  static NcclApi api = [] {
    NcclApi a;
    memset(&a, 0, sizeof(a));
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    bool ok = true;
    auto get = [&](const char* name) {
      void* f = dlsym(h, name);
      ok = ok && f != nullptr;
      return f;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(get("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(get("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(get("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(get("ncclAllReduce"));
    a.Reduce = reinterpret_cast<decltype(a.Reduce)>(get("ncclReduce"));
    a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(get("ncclReduceScatter"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(get("ncclAllGather"));
    a.Send = reinterpret_cast<decltype(a.Send)>(get("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(get("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(get("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(get("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(get("ncclGetErrorString"));
    a.ok = ok;
    return a;
  }();
  return &api;
}

int nccl_fail(Plan* p, NcclResult r, const char* what) {
  const NcclApi* a = nccl();
  const char* txt = (a->ok && a->GetErrorString) ? a->GetErrorString(r) : "?";
  return fail(p, HPNFFT_E_NCCL, std::string(what) + ": " + txt);
}

#define HPNFFT_NCCL_TRY(p, expr, what)         \
  do {                                         \
    NcclResult r_ = (expr);                    \
    if (r_ != 0) return nccl_fail((p), r_, (what)); \
  } while (0)

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// memory plane of the x-ordered cell plane c0x (c0x = (c0 + n0/2) mod n0)
inline int64_t mem_plane(int64_t c0x, int64_t n0) { return ((c0x + n0 / 2) % n0 + n0) % n0; }

struct PlaneMap {
  int count;
  int plane[16];   // destination memory plane of received halo plane j
};

// grid[plane[j]] += halo[j], all planes of one halo exchange in one launch (blockIdx.y = j)
__global__ void k_halo_add(double2* __restrict__ grid, const double2* __restrict__ halo, int64_t plane_elems,
                           PlaneMap map) {
  const int j = blockIdx.y;
  if (j >= map.count) return;
  double2* dst = grid + (size_t)map.plane[j] * plane_elems;
  const double2* src = halo + (size_t)j * plane_elems;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < plane_elems; e += (int64_t)gridDim.x * blockDim.x) {
    double2 a = dst[e];
    const double2 b = src[e];
    a.x += b.x;
    a.y += b.y;
    dst[e] = a;
  }
}

// send[s][p][k1l][k2] = B[(l0 + p) mod n0][s * N1P + k1l][k2]: destination-major blocks of the
// y-pass output, so that every block of the all-to-all is contiguous
__global__ void k_pack(const double2* __restrict__ B, double2* __restrict__ send, int64_t l0, int64_t n0, int64_t L,
                       int64_t N1, int64_t N1P, int64_t N2, int P) {
  const int64_t per_dest = L * N1P * N2;
  const int64_t total = per_dest * P;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e / per_dest;
    int64_t r = e - s * per_dest;
    const int64_t pl = r / (N1P * N2);
    r -= pl * (N1P * N2);
    const int64_t k1l = r / N2, k2 = r - k1l * N2;
    const int64_t plane = (l0 + pl) % n0;
    send[e] = B[(plane * N1 + s * N1P + k1l) * N2 + k2];
  }
}

// GRID_SLAB step 1: every rank adds the halo planes its neighbours' points reached
int halo_exchange(Plan* p) {
  const NcclApi* a = nccl();
  const int P = p->nranks, r = p->dist_rank, m = p->m;
  const int64_t n0 = p->n[0], pe = p->n[1] * p->n[2];   // complex elements per plane
  const int lower = (r - 1 + P) % P, upper = (r + 1) % P;
  const int64_t lo = p->slab_lo, L = p->slab_len;
  double2* grid = reinterpret_cast<double2*>(p->grid);
  double2* halo = reinterpret_cast<double2*>(p->halo);
  NcclComm comm = p->comm;
  // a run of k x-ordered planes starting at c0x is at most two memory-contiguous pieces
  auto runs = [&](int64_t c0x, int k, auto&& fn) {
    const int64_t first = mem_plane(c0x, n0);
    const int k0 = (int)(first + k <= n0 ? k : n0 - first);
    fn(first, 0, k0);
    if (k0 < k) fn(0, k0, k - k0);
  };
  HPNFFT_NCCL_TRY(p, a->GroupStart(), "ncclGroupStart");
  // my lower halo (m - 1 planes below my slab) -> rank r-1; my upper halo (m planes) -> rank r+1
  int rcode = 0;
  runs(lo - (m - 1), m - 1, [&](int64_t plane, int, int k) {
    if (!rcode) rcode = a->Send(grid + plane * pe, 2 * pe * k, kNcclFloat64, lower, comm, p->stream);
  });
  runs(lo + L, m, [&](int64_t plane, int, int k) {
    if (!rcode) rcode = a->Send(grid + plane * pe, 2 * pe * k, kNcclFloat64, upper, comm, p->stream);
  });
  // rank r+1's lower halo -> halo[0, m-1); rank r-1's upper halo -> halo[m-1, 2m-1), received in
  // the sender's piece structure (the same x-ordered plane run, so the same split)
  runs(lo + L - (m - 1), m - 1, [&](int64_t, int j, int k) {
    if (!rcode) rcode = a->Recv(halo + (int64_t)j * pe, 2 * pe * k, kNcclFloat64, upper, comm, p->stream);
  });
  runs(lo, m, [&](int64_t, int j, int k) {
    if (!rcode) rcode = a->Recv(halo + (int64_t)(m - 1 + j) * pe, 2 * pe * k, kNcclFloat64, lower, comm, p->stream);
  });
  if (rcode) {
    a->GroupEnd();
    return nccl_fail(p, rcode, "halo send/recv");
  }
  HPNFFT_NCCL_TRY(p, a->GroupEnd(), "ncclGroupEnd");
  PlaneMap map;
  map.count = 2 * m - 1;
  for (int j = 0; j < m - 1; ++j) map.plane[j] = (int)mem_plane(lo + L - (m - 1) + j, n0);
  for (int j = 0; j < m; ++j) map.plane[m - 1 + j] = (int)mem_plane(lo + j, n0);
  dim3 g((unsigned)((pe + 255) / 256 < 512 ? (pe + 255) / 256 : 512), (unsigned)map.count);
  k_halo_add<<<g, 256, 0, p->stream>>>(grid, halo, pe, map);
  p->launches++;
  return check_launch(p, "halo add");
}

// GRID_SLAB steps 2-4: FFT z and y on the own planes, all-to-all, FFT x on the own k1 slab
int slab_fft(Plan* p, double* fhat) {
  const NcclApi* a = nccl();
  const int P = p->nranks, r = p->dist_rank;
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2];
  const int64_t N1 = p->N[1], N2 = p->N[2], N1P = N1 / P;
  const int64_t L = p->slab_len, l0 = mem_plane(p->slab_lo, n0);
  int rc;
  stage_begin(p, 4);
  rc = fft_pass(p, 2, p->grid, p->bufA, L * n1, 1, true, l0 * n1, n0 * n1, 0, (int)n2);
  stage_end(p, 4);
  if (rc) return rc;
  stage_begin(p, 5);
  rc = fft_pass(p, 1, p->bufA, p->bufB, L, N2, false, l0, n0, 0, (int)n1);
  stage_end(p, 5);
  if (rc) return rc;
  stage_begin(p, 9);
  const int64_t blk = L * N1P * N2;   // complex elements per (source, destination) block
  double2* send = reinterpret_cast<double2*>(p->bufA);
  double2* recv = reinterpret_cast<double2*>(p->grid);   // [n0][N1P][N2] in memory-plane order
  {
    const int64_t total = blk * P;
    const int64_t blocks = (total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096;
    k_pack<<<(unsigned)blocks, 256, 0, p->stream>>>(reinterpret_cast<const double2*>(p->bufB), send, l0, n0, L, N1,
                                                     N1P, N2, P);
    p->launches++;
    rc = check_launch(p, "pack");
    if (rc) return rc;
  }
  HPNFFT_NCCL_TRY(p, a->GroupStart(), "ncclGroupStart");
  for (int s = 0; s < P; ++s) {
    if (s == r) continue;
    // rank s's slab (its own length: slabs may differ, hpnfft_set_slabs) is one memory-contiguous
    // plane run (x = 0 is a slab edge)
    const int64_t dst_plane = mem_plane(p->slab_edges[s], n0);
    const int64_t blk_s = (p->slab_edges[s + 1] - p->slab_edges[s]) * N1P * N2;
    HPNFFT_NCCL_TRY(p, a->Send(send + s * blk, 2 * blk, kNcclFloat64, s, p->comm, p->stream), "ncclSend a2a");
    HPNFFT_NCCL_TRY(p, a->Recv(recv + dst_plane * N1P * N2, 2 * blk_s, kNcclFloat64, s, p->comm, p->stream),
                    "ncclRecv a2a");
  }
  HPNFFT_NCCL_TRY(p, a->GroupEnd(), "ncclGroupEnd");
  HPNFFT_CUDA_TRY(p, cudaMemcpyAsync(recv + l0 * N1P * N2, send + r * blk, sizeof(double2) * blk,
                                     cudaMemcpyDeviceToDevice, p->stream),
                  "a2a self block");
  stage_end(p, 9);
  stage_begin(p, 6);
  rc = x_pass(p, p->grid, fhat, N1P * N2, (int64_t)r * N1P, 0, (int)n0);
  stage_end(p, 6);
  return rc;
}

// ---------------------------------------------------------------------------------------------
// GRID_SLAB over NVLink peer memory: the grids of all ranks are mapped into every rank (CUDA IPC
// handles exchanged once with ncclAllGather), the halo is PULLED from the neighbours' grids and
// added locally, and the y FFT pass stores its outputs straight into the destination ranks'
// buffers (the all-to-all is fused into the FFT epilogue).  Cross-GPU ordering comes from a
// flag barrier in peer memory (release/acquire at system scope) between the phases.
__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// every rank writes `epoch` into its slot of every rank's flags, then waits for all slots of its
// own flags; gives up after 5 s (sets *err) instead of hanging the GPU
__global__ void k_xbarrier(uint32_t* const* peer_flags, int P, int r, uint32_t epoch, int* err, int fault) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int s = 0; s < P; ++s) st_release_sys(peer_flags[s] + r, epoch);
  if (fault) {   // fault injection (tests): behave as if the wait had timed out
    *err = 1;
    return;
  }
  const uint32_t* mine = peer_flags[r];
  const uint64_t t0 = globaltimer();
  for (int s = 0; s < P; ++s) {
    while (ld_acquire_sys(mine + s) < epoch) {
      if (globaltimer() - t0 > 5000000000ull) {
        *err = 1;
        return;
      }
    }
  }
  __threadfence_system();
}

// my owned planes += the same memory planes of the neighbours' grids (their halo regions)
__global__ void k_halo_pull(double2* __restrict__ grid, const double2* __restrict__ from_upper,
                            const double2* __restrict__ from_lower, int64_t plane_elems, PlaneMap map, int n_upper,
                            const int* __restrict__ abort_flag) {
  const int j = blockIdx.y;
  if (j >= map.count) return;
  if (abort_flag && *abort_flag) return;   // a cross-GPU barrier timed out: touch no peer memory
  const size_t off = (size_t)map.plane[j] * plane_elems;
  double2* dst = grid + off;
  const double2* src = (j < n_upper ? from_upper : from_lower) + off;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < plane_elems; e += (int64_t)gridDim.x * blockDim.x) {
    double2 a = dst[e];
    const double2 b = src[e];
    a.x += b.x;
    a.y += b.y;
    dst[e] = a;
  }
}

int xbarrier(Plan* p) {
  if (p->virt) return HPNFFT_OK;   // one-GPU rank group: stream order is the barrier
  ++p->epoch;
  // HPNFFT_XBARRIER_FAULT=1 (read per call; tools/dist_check.py): this rank's barriers report a
  // timeout after releasing their own flags, to exercise the error path (skipped peer traffic,
  // NaN output, HPNFFT_E_NCCL from the next call)
  const char* fe = getenv("HPNFFT_XBARRIER_FAULT");
  const int fault = fe && fe[0] == '1';
  k_xbarrier<<<1, 32, 0, p->stream>>>(p->peer_flags, p->nranks, p->dist_rank, p->epoch, p->dist_err, fault);
  p->launches++;
  return check_launch(p, "cross-GPU barrier");
}

}  // namespace

// The grid-slab adjoint over peer memory in four phases.  A real rank runs them back to back
// (slab_adjoint_p2p) with cross-GPU flag barriers where a phase reads or writes a peer's grid; a
// one-GPU rank group (hpnfft_plan_group) runs each phase for every rank before the next phase.
// 1. halo: after every rank's sweep, pull the neighbours' halo planes into my own planes
int slab_phase_halo(Plan* p) {
  const int P = p->nranks, r = p->dist_rank, m = p->m;
  const int64_t n0 = p->n[0], pe = p->n[1] * p->n[2];
  const int64_t lo = p->slab_lo, L = p->slab_len;
  stage_begin(p, 8);
  int rc = xbarrier(p);
  if (rc) return rc;
  PlaneMap map;
  map.count = 2 * m - 1;
  for (int j = 0; j < m - 1; ++j) map.plane[j] = (int)mem_plane(lo + L - (m - 1) + j, n0);   // from rank r+1
  for (int j = 0; j < m; ++j) map.plane[m - 1 + j] = (int)mem_plane(lo + j, n0);           // from rank r-1
  dim3 g((unsigned)((pe + 255) / 256 < 512 ? (pe + 255) / 256 : 512), (unsigned)map.count);
  k_halo_pull<<<g, 256, 0, p->stream>>>(reinterpret_cast<double2*>(p->grid),
                                       reinterpret_cast<const double2*>(p->peer_grid_host[(r + 1) % P]),
                                       reinterpret_cast<const double2*>(p->peer_grid_host[(r - 1 + P) % P]), pe, map,
                                       m - 1, p->virt ? nullptr : p->dist_err);
  p->launches++;
  rc = check_launch(p, "halo pull");
  stage_end(p, 8);
  return rc;
}

// 2. z pass on the own planes (the grid is read for the last time)
int slab_phase_z(Plan* p) {
  const int64_t n0 = p->n[0], n1 = p->n[1], n2 = p->n[2];
  const int64_t L = p->slab_len, l0 = mem_plane(p->slab_lo, n0);
  stage_begin(p, 4);
  const int rc = fft_pass(p, 2, p->grid, p->bufA, L * n1, 1, true, l0 * n1, n0 * n1, 0, (int)n2);
  stage_end(p, 4);
  return rc;
}

// 3. every rank has finished reading its grid: the y pass stores into the destination ranks'
//    grids ([n0][N1/P][N2] receive layout) over NVLink, then everyone waits for everyone
int slab_phase_y(Plan* p) {
  const int P = p->nranks;
  const int64_t n0 = p->n[0], n1 = p->n[1];
  const int64_t N2 = p->N[2], N1P = p->N[1] / P;
  const int64_t L = p->slab_len, l0 = mem_plane(p->slab_lo, n0);
  stage_begin(p, 9);
  int rc = xbarrier(p);
  stage_end(p, 9);
  if (rc) return rc;
  stage_begin(p, 5);
  rc = fft_pass(p, 1, p->bufA, p->grid, L, N2, false, l0, n0, 0, (int)n1, p->peer_grid, (int)N1P);
  if (!rc) rc = xbarrier(p);
  stage_end(p, 5);
  return rc;
}

// 4. x pass (+ deconvolve, or the Eq. 12 energy sum) on the own k1 slab
int slab_phase_x(Plan* p, double* fhat) {
  const int64_t n0 = p->n[0], N2 = p->N[2], N1P = p->N[1] / p->nranks;
  stage_begin(p, 6);
  const int rc = x_pass(p, p->grid, fhat, N1P * N2, (int64_t)p->dist_rank * N1P, 0, (int)n0);
  stage_end(p, 6);
  return rc;
}

namespace {

// a cross-GPU barrier of this transform timed out (*err set by k_xbarrier): the phases after it
// skipped their peer traffic, so the rank's output is filled with NaN instead of being left
// plausible-looking (the plan's next call returns HPNFFT_E_NCCL)
__global__ void k_poison_on_err(double* __restrict__ a, int64_t n, const int* __restrict__ err) {
  if (*err == 0) return;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = nan;
}

int slab_adjoint_p2p(Plan* p, double* fhat) {
  int rc = slab_phase_halo(p);
  if (!rc) rc = slab_phase_z(p);
  if (!rc) rc = slab_phase_y(p);
  if (!rc) rc = slab_phase_x(p, fhat);
  if (!rc && fhat && p->dist_err && !p->virt) {
    const int64_t n = 2 * p->N[0] * (p->N[1] / p->nranks) * p->N[2];   // this rank's k1 slab of fhat
    k_poison_on_err<<<(unsigned)(device_sm_count() * 4), 256, 0, p->stream>>>(fhat, n, p->dist_err);
    p->launches++;
    rc = check_launch(p, "barrier error poison");
  }
  return rc;
}

// map the peers' grids and barrier flags (CUDA IPC, handles exchanged with ncclAllGather).
// Collective and consistent: every rank reaches both collectives whatever happens locally (an
// allocation, a handle export or an open that fails), and the ranks agree on the outcome (the
// minimum over the ranks of a local ok flag), so that all of them take the same exchange protocol
// (peer memory or NCCL send/recv).  `want` = this rank's HPNFFT_DIST_P2P choice (also agreed).
bool setup_p2p(Plan* p, bool want) {
  const NcclApi* a = nccl();
  const int P = p->nranks, r = p->dist_rank;
  struct Msg {
    cudaIpcMemHandle_t h[2];
    int ok;
    int pad;
  };
  Msg mine;
  memset(&mine, 0, sizeof(mine));
  bool ok = want && P <= 16;
  ok = ok && cudaMalloc(&p->flags, 64 * sizeof(uint32_t)) == cudaSuccess;
  ok = ok && cudaMemset(p->flags, 0, 64 * sizeof(uint32_t)) == cudaSuccess;
  ok = ok && cudaMalloc(&p->dist_err, sizeof(int)) == cudaSuccess;
  ok = ok && cudaMemset(p->dist_err, 0, sizeof(int)) == cudaSuccess;
  ok = ok && cudaIpcGetMemHandle(&mine.h[0], p->grid) == cudaSuccess &&
       cudaIpcGetMemHandle(&mine.h[1], p->flags) == cudaSuccess;
  cudaGetLastError();
  mine.ok = ok ? 1 : 0;
  // device scratch for the two collectives: the (not yet used) grid when it is large enough
  const size_t hb = sizeof(Msg), need = hb * (size_t)(P + 1) + 2 * sizeof(int);
  const size_t grid_bytes = sizeof(double) * 2 * (size_t)(p->n[0] * p->n[1] * p->n[2]);
  unsigned char* dbuf = reinterpret_cast<unsigned char*>(p->grid);
  bool own = false;
  if (grid_bytes < need) {
    own = true;
    if (cudaMalloc(&dbuf, need) != cudaSuccess) dbuf = nullptr;   // tiny grids only
  }
  std::vector<unsigned char> all(hb * P);
  bool coll = dbuf != nullptr && cudaMemcpy(dbuf + hb * P, &mine, hb, cudaMemcpyHostToDevice) == cudaSuccess;
  coll = a->AllGather(dbuf + hb * P, dbuf, hb, 0 /* ncclInt8 */, p->comm, p->stream) == 0 && coll;
  coll = coll && cudaStreamSynchronize(p->stream) == cudaSuccess &&
         cudaMemcpy(all.data(), dbuf, hb * P, cudaMemcpyDeviceToHost) == cudaSuccess;
  bool all_ok = coll;
  for (int s = 0; s < P && all_ok; ++s) all_ok = reinterpret_cast<const Msg*>(all.data() + hb * s)->ok == 1;
  bool opened = all_ok;
  for (int s = 0; s < P && opened; ++s) {
    if (s == r) {
      p->peer_grid_host[s] = p->grid;
      p->peer_flags_host[s] = p->flags;
      continue;
    }
    const Msg* ms = reinterpret_cast<const Msg*>(all.data() + hb * s);
    void* g = nullptr;
    void* fl = nullptr;
    opened = cudaIpcOpenMemHandle(&g, ms->h[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (opened) p->peer_grid_host[s] = static_cast<double*>(g);
    opened = opened && cudaIpcOpenMemHandle(&fl, ms->h[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
    if (opened) p->peer_flags_host[s] = static_cast<uint32_t*>(fl);
  }
  if (opened) {
    opened = cudaMalloc(&p->peer_grid, sizeof(double*) * P) == cudaSuccess &&
             cudaMalloc(&p->peer_flags, sizeof(uint32_t*) * P) == cudaSuccess &&
             cudaMemcpy(p->peer_grid, p->peer_grid_host, sizeof(double*) * P, cudaMemcpyHostToDevice) == cudaSuccess &&
             cudaMemcpy(p->peer_flags, p->peer_flags_host, sizeof(uint32_t*) * P, cudaMemcpyHostToDevice) == cudaSuccess;
  }
  cudaGetLastError();
  // agreement on the outcome: min over the ranks (every rank reaches this all-reduce)
  int agreed = opened ? 1 : 0;
  if (dbuf) {
    int* d = reinterpret_cast<int*>(dbuf + hb * (size_t)(P + 1));
    bool c2 = cudaMemcpy(d, &agreed, sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
    c2 = a->AllReduce(d, d + 1, 1, 2 /* ncclInt32 */, 3 /* ncclMin */, p->comm, p->stream) == 0 && c2;
    c2 = c2 && cudaStreamSynchronize(p->stream) == cudaSuccess &&
         cudaMemcpy(&agreed, d + 1, sizeof(int), cudaMemcpyDeviceToHost) == cudaSuccess;
    if (!c2) agreed = 0;
  } else {
    agreed = 0;
  }
  if (own && dbuf) cudaFree(dbuf);
  cudaGetLastError();
  if (!agreed) {   // everyone falls back to NCCL send/recv: release what this rank mapped
    for (int s = 0; s < 16; ++s) {
      if (s != r && p->peer_grid_host[s]) cudaIpcCloseMemHandle(p->peer_grid_host[s]);
      if (s != r && p->peer_flags_host[s]) cudaIpcCloseMemHandle(p->peer_flags_host[s]);
      p->peer_grid_host[s] = nullptr;
      p->peer_flags_host[s] = nullptr;
    }
    cudaFree(p->peer_grid);
    cudaFree(p->peer_flags);
    p->peer_grid = nullptr;
    p->peer_flags = nullptr;
    cudaGetLastError();
    return false;
  }
  return true;
}

}  // namespace

int dist_adjoint(Plan* p, const double* f, double* fhat) {
  const NcclApi* a = nccl();
  const int64_t nk = p->N[0] * p->N[1] * p->N[2];
  int rc;
  if (p->nranks == 1) {   // nothing to exchange
    rc = spread(p, f);
    return rc ? rc : fft_and_deconvolve(p, fhat);
  }
  switch (p->dist_mode) {
    case HPNFFT_DIST_ALLREDUCE:
    case HPNFFT_DIST_REDUCE_ROOT0:
      rc = spread(p, f);
      if (!rc) rc = fft_and_deconvolve(p, fhat);
      if (rc) return rc;
      stage_begin(p, 8);
      if (p->dist_mode == HPNFFT_DIST_ALLREDUCE)
        HPNFFT_NCCL_TRY(p, a->AllReduce(fhat, fhat, 2 * nk, kNcclFloat64, kNcclSum, p->comm, p->stream), "ncclAllReduce");
      else
        HPNFFT_NCCL_TRY(p, a->Reduce(fhat, fhat, 2 * nk, kNcclFloat64, kNcclSum, 0, p->comm, p->stream), "ncclReduce");
      stage_end(p, 8);
      return HPNFFT_OK;
    case HPNFFT_DIST_REDUCE_SCATTER:
      rc = spread(p, f);
      if (!rc) rc = fft_and_deconvolve(p, p->partial);
      if (rc) return rc;
      stage_begin(p, 8);
      HPNFFT_NCCL_TRY(p, a->ReduceScatter(p->partial, fhat, 2 * nk / p->nranks, kNcclFloat64, kNcclSum, p->comm, p->stream),
                      "ncclReduceScatter");
      stage_end(p, 8);
      return HPNFFT_OK;
    case HPNFFT_DIST_GRID_SLAB:
      rc = spread(p, f);
      if (rc) return rc;
      if (p->p2p) return slab_adjoint_p2p(p, fhat);
      stage_begin(p, 8);
      rc = halo_exchange(p);
      stage_end(p, 8);
      if (rc) return rc;
      return slab_fft(p, fhat);
    default:
      set_error("unknown distribution mode");
      return HPNFFT_E_INVALID;
  }
}

// in-place sum over the ranks of `count` doubles (the ENUF energy scalar of grid-slab plans)
int dist_allreduce_sum(Plan* p, double* buf, int64_t count) {
  if (p->nranks < 2) return HPNFFT_OK;
  const NcclApi* a = nccl();
  HPNFFT_NCCL_TRY(p, a->AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, p->comm, p->stream), "ncclAllReduce");
  return HPNFFT_OK;
}

void dist_free(Plan* p) {
  for (int s = 0; s < 16; ++s) {
    if (s == p->dist_rank || p->virt) continue;   // a rank group's peers are its own plans' grids
    if (p->peer_grid_host[s]) cudaIpcCloseMemHandle(p->peer_grid_host[s]);
    if (p->peer_flags_host[s]) cudaIpcCloseMemHandle(p->peer_flags_host[s]);
  }
  for (int s = 0; s < 16; ++s) {
    p->peer_grid_host[s] = nullptr;
    p->peer_flags_host[s] = nullptr;
  }
  cudaFree(p->peer_grid);
  cudaFree(p->peer_flags);
  cudaFree(p->flags);
  cudaFree(p->dist_err);
  p->peer_grid = nullptr;
  p->peer_flags = nullptr;
  p->flags = nullptr;
  p->dist_err = nullptr;
  if (p->comm && nccl()->ok) nccl()->CommDestroy(p->comm);
  p->comm = nullptr;
  cudaFree(p->halo);
  cudaFree(p->partial);
  p->halo = p->partial = nullptr;
}

}  // namespace hpnfft

using namespace hpnfft;

extern "C" {

int hpnfft_get_unique_id(unsigned char id[128]) {
  if (!id) {
    set_error("id is NULL");
    return HPNFFT_E_INVALID;
  }
  const NcclApi* a = nccl();
  if (!a->ok) {
    set_error("NCCL (libnccl.so.2) could not be loaded");
    return HPNFFT_E_NCCL;
  }
  NcclUid u;
  const NcclResult r = a->GetUniqueId(&u);
  if (r != 0) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  memcpy(id, u.internal, 128);
  return HPNFFT_OK;
}

}  // extern "C"

namespace hpnfft {
namespace {

// validation shared by hpnfft_plan_dist and hpnfft_plan_group (before anything is created)
int check_dist_args(const char* fn, int nranks, int mode) {
  if (nranks < 1 || nranks > 16) {
    set_error(std::string(fn) + ": need 1 <= nranks <= 16");
    return HPNFFT_E_INVALID;
  }
  if (mode < HPNFFT_DIST_ALLREDUCE || mode > HPNFFT_DIST_GRID_SLAB) {
    set_error(std::string(fn) + ": unknown mode");
    return HPNFFT_E_INVALID;
  }
  return HPNFFT_OK;
}

// rank `rank` of `nranks` in `mode` on a freshly created plan: mode constraints, the equal-size
// slabs, the bin table reset, the exchange buffers (no communication)
int init_dist_fields(Plan* p, int nranks, int rank, int mode) {
  const int64_t n0 = p->n[0];
  const int m = p->m;
  if ((p->d != 3 || p->precision != HPNFFT_PRECISION_F64) && nranks > 1) {
    set_error("multi-GPU plans need d = 3 (x-slab subcells of dimension 0, PAPER.md:93)");
    return HPNFFT_E_UNSUPPORTED;
  }
  if (mode == HPNFFT_DIST_REDUCE_SCATTER && p->N[0] % nranks) {
    set_error("HPNFFT_DIST_REDUCE_SCATTER needs N0 % nranks == 0");
    return HPNFFT_E_UNSUPPORTED;
  }
  if (mode == HPNFFT_DIST_GRID_SLAB && nranks > 1 &&
      (!is_pow2(nranks) || p->N[1] % nranks || n0 / nranks < 2 * m || n0 % nranks)) {
    set_error("HPNFFT_DIST_GRID_SLAB needs nranks a power of two, N1 % nranks == 0 and n0 / nranks >= 2m");
    return HPNFFT_E_UNSUPPORTED;
  }
  p->dist_mode = mode;
  p->nranks = nranks;
  p->dist_rank = rank;
  for (int s = 0; s <= nranks; ++s) p->slab_edges[s] = (int64_t)s * (n0 / nranks);
  p->slab_len = n0 / nranks;
  p->slab_lo = (int64_t)rank * p->slab_len;
  // grid-slab ranks zero and scan only their own key range per set_points (sort.cu key_range):
  // the rest of the bin table must read as empty
  if (cudaMemset(p->bin_count, 0, sizeof(uint32_t) * (size_t)(p->nbins + 1)) != cudaSuccess) {
    cudaGetLastError();
    set_error("bin table initialisation failed");
    return HPNFFT_E_CUDA;
  }
  cudaError_t e = cudaSuccess;
  if (mode == HPNFFT_DIST_GRID_SLAB && nranks > 1)
    e = cudaMalloc(&p->halo, sizeof(double) * 2 * (size_t)(2 * m - 1) * (size_t)(p->n[1] * p->n[2]));
  if (mode == HPNFFT_DIST_REDUCE_SCATTER && nranks > 1)
    e = cudaMalloc(&p->partial, sizeof(double) * 2 * (size_t)(p->N[0] * p->N[1] * p->N[2]));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation of the exchange buffers failed");
    return HPNFFT_E_NOMEM;
  }
  return HPNFFT_OK;
}

// dst[i] += src[i] (the option-A sum of a one-GPU rank group)
__global__ void k_add_into(double* __restrict__ dst, const double* __restrict__ src, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

int add_into(Plan* p, double* dst, const double* src, int64_t count) {
  const int64_t blocks = (count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096;
  if (count <= 0) return HPNFFT_OK;
  k_add_into<<<(unsigned)blocks, 256, 0, p->stream>>>(dst, src, count);
  p->launches++;
  return check_launch(p, "group sum");
}

}  // namespace
}  // namespace hpnfft

extern "C" {

int hpnfft_plan_dist(hpnfft_plan_t* out, int d, const int64_t* N, int64_t M_local, int m, double sigma, int window,
                     void* stream, int nranks, int rank, const unsigned char id[128], int mode) {
  if (!out) {
    set_error("hpnfft_plan_dist: out is NULL");
    return HPNFFT_E_INVALID;
  }
  *out = nullptr;
  int rc = check_dist_args("hpnfft_plan_dist", nranks, mode);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks || !id) {
    set_error("hpnfft_plan_dist: need 0 <= rank < nranks and a unique id");
    return HPNFFT_E_INVALID;
  }
  hpnfft_plan_t h = nullptr;
  rc = hpnfft_plan(&h, d, N, M_local, m, sigma, window, stream);
  if (rc) return rc;
  Plan* p = reinterpret_cast<Plan*>(h);
  const NcclApi* a = nccl();
  if (!a->ok) {
    hpnfft_destroy(h);
    set_error("NCCL (libnccl.so.2) could not be loaded");
    return HPNFFT_E_NCCL;
  }
  rc = init_dist_fields(p, nranks, rank, mode);
  if (rc) {
    const std::string msg = hpnfft_last_error();
    hpnfft_destroy(h);
    set_error(msg);
    return rc;
  }
  if (nranks > 1) {
    NcclUid u;
    memcpy(u.internal, id, 128);
    NcclComm comm = nullptr;
    const NcclResult r = a->CommInitRank(&comm, nranks, u, rank);
    if (r != 0) {
      rc = nccl_fail(nullptr, r, "ncclCommInitRank");
      hpnfft_destroy(h);
      return rc;
    }
    p->comm = comm;
  }
  if (mode == HPNFFT_DIST_GRID_SLAB && nranks > 1) {
    const char* env = getenv("HPNFFT_DIST_P2P");
    p->p2p = setup_p2p(p, !(env && env[0] == '0'));
  }
  *out = h;
  return HPNFFT_OK;
}

int hpnfft_plan_group(hpnfft_plan_t* out, int d, const int64_t* N, const int64_t* M, int m, double sigma, int window,
                      void* stream, int nranks, int mode) {
  if (!out || !M) {
    set_error("hpnfft_plan_group: out or M is NULL");
    return HPNFFT_E_INVALID;
  }
  int rc = check_dist_args("hpnfft_plan_group", nranks, mode);
  if (rc) return rc;
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  Plan* ps[16] = {};
  auto undo = [&](int code) {
    const std::string msg = hpnfft_last_error();
    for (int r = 0; r < nranks; ++r) {
      if (ps[r]) hpnfft_destroy(reinterpret_cast<hpnfft_plan_t>(ps[r]));
      out[r] = nullptr;
    }
    set_error(msg);
    return code;
  };
  for (int r = 0; r < nranks; ++r) {
    hpnfft_plan_t h = nullptr;
    rc = hpnfft_plan(&h, d, N, M[r], m, sigma, window, stream);
    if (rc) return undo(rc);
    ps[r] = reinterpret_cast<Plan*>(h);
    ps[r]->virt = true;
    rc = init_dist_fields(ps[r], nranks, r, mode);
    if (rc) return undo(rc);
  }
  if (mode == HPNFFT_DIST_GRID_SLAB && nranks > 1) {
    double* grids[16] = {};
    for (int s = 0; s < nranks; ++s) grids[s] = ps[s]->grid;
    for (int r = 0; r < nranks; ++r) {
      Plan* p = ps[r];
      for (int s = 0; s < nranks; ++s) p->peer_grid_host[s] = grids[s];
      if (cudaMalloc(&p->peer_grid, sizeof(double*) * nranks) != cudaSuccess ||
          cudaMemcpy(p->peer_grid, grids, sizeof(double*) * nranks, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        set_error("device allocation of the group's peer table failed");
        return undo(HPNFFT_E_NOMEM);
      }
      p->p2p = true;
    }
  }
  for (int r = 0; r < nranks; ++r) out[r] = reinterpret_cast<hpnfft_plan_t>(ps[r]);
  return HPNFFT_OK;
}

int hpnfft_adjoint_group(hpnfft_plan_t* plans, int nranks, const double* const* f, double* const* fhat) {
  if (!plans || !f || !fhat || nranks < 1 || nranks > 16) {
    set_error("hpnfft_adjoint_group: NULL argument or bad nranks");
    return HPNFFT_E_INVALID;
  }
  Plan* ps[16];
  for (int r = 0; r < nranks; ++r) {
    ps[r] = reinterpret_cast<Plan*>(plans[r]);
    Plan* p = ps[r];
    if (!p || !p->virt || p->nranks != nranks || p->dist_rank != r || p->dist_mode != ps[0]->dist_mode ||
        p->stream != ps[0]->stream) {
      set_error("hpnfft_adjoint_group: plans must be the members of one hpnfft_plan_group, in rank order, on one "
                "stream");
      return HPNFFT_E_INVALID;
    }
    if (p->failed) {
      set_error("plan is in a failed state (an earlier CUDA error)");
      return HPNFFT_E_STATE;
    }
    if (!p->points_set) {
      set_error("hpnfft_adjoint_group called before a successful hpnfft_set_points of every member");
      return HPNFFT_E_STATE;
    }
    if (!fhat[r] || (!f[r] && p->M > 0)) {
      set_error("f or fhat is NULL");
      return HPNFFT_E_INVALID;
    }
  }
  const int mode = ps[0]->dist_mode;
  int rc = HPNFFT_OK;
  if (mode == HPNFFT_DIST_GRID_SLAB && nranks > 1) {
    // the exchange phases of slab_adjoint_p2p, each for all ranks before the next (stream order)
    for (int r = 0; r < nranks && !rc; ++r) rc = spread(ps[r], f[r]);
    for (int r = 0; r < nranks && !rc; ++r) rc = slab_phase_halo(ps[r]);
    for (int r = 0; r < nranks && !rc; ++r) rc = slab_phase_z(ps[r]);
    for (int r = 0; r < nranks && !rc; ++r) rc = slab_phase_y(ps[r]);
    for (int r = 0; r < nranks && !rc; ++r) rc = slab_phase_x(ps[r], fhat[r]);
    return rc;
  }
  // option A: every rank's partial transform, then the collective's result layout
  const int64_t nk = ps[0]->N[0] * ps[0]->N[1] * ps[0]->N[2];
  const bool rs = mode == HPNFFT_DIST_REDUCE_SCATTER && nranks > 1;
  for (int r = 0; r < nranks && !rc; ++r) {
    rc = spread(ps[r], f[r]);
    if (!rc) rc = fft_and_deconvolve(ps[r], rs ? ps[r]->partial : fhat[r]);
  }
  if (rc || nranks == 1) return rc;
  Plan* p0 = ps[0];
  stage_begin(p0, 8);
  if (rs) {   // fhat[r] = sum_s partial_s[k0 slab r]
    const int64_t blk = 2 * nk / nranks;
    for (int r = 0; r < nranks && !rc; ++r) {
      if (cudaMemcpyAsync(fhat[r], ps[0]->partial + r * blk, sizeof(double) * blk, cudaMemcpyDeviceToDevice,
                          p0->stream) != cudaSuccess)
        return fail(p0, HPNFFT_E_CUDA, "group copy");
      for (int s = 1; s < nranks && !rc; ++s) rc = add_into(p0, fhat[r], ps[s]->partial + r * blk, blk);
    }
  } else {   // ALLREDUCE: every rank the sum; REDUCE_ROOT0: rank 0 the sum, the others their partial
    for (int s = 1; s < nranks && !rc; ++s) rc = add_into(p0, fhat[0], fhat[s], 2 * nk);
    if (mode == HPNFFT_DIST_ALLREDUCE)
      for (int r = 1; r < nranks && !rc; ++r)
        if (cudaMemcpyAsync(fhat[r], fhat[0], sizeof(double) * 2 * nk, cudaMemcpyDeviceToDevice, p0->stream) !=
            cudaSuccess)
          return fail(p0, HPNFFT_E_CUDA, "group copy");
  }
  stage_end(p0, 8);
  return rc;
}

int hpnfft_set_slabs(hpnfft_plan_t h, const int64_t* edges) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p || !edges) {
    set_error("NULL argument");
    return HPNFFT_E_INVALID;
  }
  if (p->dist_mode != HPNFFT_DIST_GRID_SLAB || p->nranks < 2) {
    set_error("hpnfft_set_slabs: only for HPNFFT_DIST_GRID_SLAB plans of 2 or more ranks");
    return HPNFFT_E_INVALID;
  }
  const int P = p->nranks;
  const int64_t n0 = p->n[0], min_len = (2 * p->m + 3) / 4 * 4;
  bool ok = edges[0] >= 0 && edges[0] < n0 && edges[P] == edges[0] + n0;
  bool x0_edge = false;   // the plane c0x = n0/2 (x = 0, memory plane 0) must start a slab
  for (int s = 0; s < P && ok; ++s) {
    const int64_t len = edges[s + 1] - edges[s];
    ok = len >= min_len && len % 4 == 0;
    x0_edge = x0_edge || edges[s] % n0 == n0 / 2;
  }
  if (!ok || !x0_edge) {
    set_error("hpnfft_set_slabs: need edges[0] in [0, n0), edges[P] = edges[0] + n0, every slab a multiple "
              "of 4 planes and >= 2m, and n0/2 (x = 0) among the edges");
    return HPNFFT_E_INVALID;
  }
  if (cudaStreamSynchronize(p->stream) != cudaSuccess ||
      cudaMemset(p->bin_count, 0, sizeof(uint32_t) * (size_t)(p->nbins + 1)) != cudaSuccess) {
    set_error("hpnfft_set_slabs: bin table reset failed");
    return HPNFFT_E_CUDA;
  }
  for (int s = 0; s <= P; ++s) p->slab_edges[s] = edges[s];
  p->slab_lo = edges[p->dist_rank] % n0;
  p->slab_len = edges[p->dist_rank + 1] - edges[p->dist_rank];
  p->points_set = false;
  return HPNFFT_OK;
}

int hpnfft_output_shape(hpnfft_plan_t h, int64_t shape[3]) {
  Plan* p = reinterpret_cast<Plan*>(h);
  if (!p || !shape) {
    set_error("NULL argument");
    return HPNFFT_E_INVALID;
  }
  shape[0] = p->N[0];
  shape[1] = p->N[1];
  shape[2] = p->N[2];
  if (p->dist_mode == HPNFFT_DIST_REDUCE_SCATTER) shape[0] = p->N[0] / p->nranks;
  if (p->dist_mode == HPNFFT_DIST_GRID_SLAB) shape[1] = p->N[1] / p->nranks;
  return HPNFFT_OK;
}

}  // extern "C"
