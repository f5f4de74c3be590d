"""Multi-GPU layer: the paper's accumulative decomposition on one process per GPU.

HP-NFFT (§3, Eqs. 7-8) splits the points into equal-size spatial subcells,
computes a partial NFFT per node and sums the partial results ("Accumulate", Alg. 3,
PAPER.md:174-200, a binomial tree of MPI Send/Recv).  Here every rank is one GPU of one node:

* the subcells are x-slabs (dimension 0): equal-size as the paper states (PAPER.md:93,
  "subcells with same size") or equal-count (quantiles, for clustered inputs);
* each rank runs the library's multi-GPU plan (``hpnfft_plan_dist``): the exchange runs inside
  libhpnfft.so with NCCL over NVLink/NVSwitch — ``allreduce`` (every rank gets fhat),
  ``reduce`` (rank 0 gets fhat, Alg. 3's semantics), ``reduce_scatter`` (k0 slabs) or
  ``grid_slab`` (SURVEY.md §8(e) option G: grid halo exchange + distributed FFT, k1 slabs;
  the points must be partitioned by ``grid_slab_mask``; ``grid_slab_edges`` gives equal-count
  cell-plane slabs for clustered inputs).  torch.distributed only carries the
  128-byte NCCL unique id from rank 0 to the others.

The partition helpers are host logic exercised on CPU with the gloo backend in
tests/test_dist_gloo.py (which emulates the exchange itself, with torch.distributed collectives
around the CPU oracle: test code, not product code); the library's exchange code runs on one GPU
in tests/test_gpu_parity.py through hpnfft_plan_group (all ranks as plans on one device).
"""
from __future__ import annotations

MODES = ("allreduce", "reduce", "reduce_scatter", "grid_slab")


def slab_bounds(rank: int, world: int):
    """Equal-size x-slab [lo, hi) of `rank` among `world`."""
    lo = -0.5 + rank / world
    hi = -0.5 + (rank + 1) / world
    return lo, hi


def slab_mask(x, rank: int, world: int, edges=None):
    """Boolean mask of the points (tensor [M, 3]) whose x0 lies in this rank's slab.

    Coordinates equal to +0.5 belong to the last slab (x = 0.5 is x = -0.5 by periodicity, but
    the partition only has to be a partition).  `edges` (world + 1 increasing values) selects
    an equal-count partition instead of equal size.
    """
    if world == 1:
        import torch

        return torch.ones(x.shape[0], dtype=torch.bool, device=x.device)
    x0 = x[:, 0]
    if edges is None:
        lo, hi = slab_bounds(rank, world)
    else:
        lo, hi = float(edges[rank]), float(edges[rank + 1])
    m = (x0 >= lo) & (x0 < hi)
    if rank == world - 1:
        m |= x0 >= hi
    if rank == 0:
        m |= x0 < lo
    return m


def _cell_plane_x(x, n0: int):
    """x-ordered cell plane c0x = (floor(n0 x0) + n0/2) mod n0 (the library's exact cell rule)."""
    import torch

    c0 = torch.floor(x[:, 0] * float(n0)).to(torch.int64) % n0
    return (c0 + n0 // 2) % n0


def grid_slab_rank(x, world: int, n0: int, edges=None):
    """Owner rank of each point for ``grid_slab`` plans.  Default: its x-ordered cell plane c0x
    lies in [r n0/P, (r+1) n0/P) (the equal-size x-slab [-1/2 + r/P, -1/2 + (r+1)/P),
    PAPER.md:93).  With `edges` (hpnfft_set_slabs, cyclic): c0x in [edges[r], edges[r+1]) mod n0."""
    import torch

    c0x = _cell_plane_x(x, n0)
    if edges is None:
        return torch.div(c0x, n0 // world, rounding_mode="floor")
    e0 = int(edges[0])
    rel = (c0x - e0) % n0
    bounds = torch.tensor([int(e) - e0 for e in edges[1:world]], dtype=torch.int64, device=x.device)
    return torch.bucketize(rel, bounds, right=True)


def grid_slab_mask(x, rank: int, world: int, n0: int, edges=None):
    return grid_slab_rank(x, world, n0, edges) == rank


def grid_slab_edges(x, world: int, n0: int, m: int = 6, group=None, reduce: bool = True,
                    plane_weight: float = 8000.0):
    """Equal-COUNT cell-plane slabs for ``grid_slab`` plans (hpnfft_set_slabs): the cyclic edges
    start at x = 0 (c0x = n0/2, the grid's memory plane 0) and cut the point histogram over the
    cell planes at the quantiles r M / P, rounded up to multiples of 4 planes, every slab >= 2m
    planes.  `x` is this rank's points; with `reduce` and torch.distributed initialised the
    histograms of all ranks are summed first (collective), so every rank returns the same edges
    (reduce=False when every rank already holds the same full point set).  `plane_weight` adds
    that many points' worth of cost to every cell plane (a rank's grid planes cost spread-flush
    and FFT time whatever their point count): the cut is then at equal cost, not equal count.
    The default 8000 is the fit of tools/slab_cost.py on a B200 at BASELINE config 4
    (profiles/r1_slab_cost.txt: 9.2e-7 ms per point, 7.1e-3 ms per plane of sort + spread and
    5.7e-4 ms per plane of the z and y FFT passes); plane_weight=0 gives equal-count slabs."""
    import torch
    import torch.distributed as dist

    c0x = _cell_plane_x(x, n0)
    mem = (c0x + n0 // 2) % n0          # memory plane: x = 0 first
    hist = torch.bincount(mem, minlength=n0).to(torch.int64)
    if reduce and dist.is_available() and dist.is_initialized():
        dist.all_reduce(hist, group=group)
    return grid_slab_edges_hist(hist, world, n0, m, plane_weight)


def grid_slab_edges_hist(hist, world: int, n0: int, m: int = 6, plane_weight: float = 8000.0):
    """The cut of grid_slab_edges on a histogram of the points over the MEMORY planes
    (hist[c0], c0 = floor(n0 x0) mod n0; x = 0 is memory plane 0), e.g. accumulated chunk by chunk."""
    import torch

    cost = hist.to(torch.float64) + float(plane_weight)
    cum = torch.cumsum(cost, 0).cpu().tolist()   # cum[e] = cost of the memory planes <= e
    total = cum[-1] if cum else 0
    step = 4
    min_len = -(-2 * m // step) * step
    if world * min_len > n0:
        raise ValueError("n0 too small for world slabs of >= 2m planes")
    E = [0]
    for r in range(1, world):
        target = r * total / world
        e = E[-1] + min_len
        while e + step <= n0 - (world - r) * min_len and cum[e - 1] < target:
            e += step
        E.append(min(e, n0 - (world - r) * min_len))
    E.append(n0)
    return [e + n0 // 2 for e in E]


def equal_count_edges(x, world: int):
    """Slab edges at the x0 quantiles so every rank owns ~M/world points (load balance)."""
    import torch

    x0 = torch.sort(x[:, 0]).values
    M = x0.shape[0]
    edges = [-0.5]
    for r in range(1, world):
        edges.append(float(x0[min(M - 1, (r * M) // world)]))
    edges.append(0.5)
    return edges


class DistPlan:
    """Distributed adjoint NFFT: the library's multi-GPU plan (hpnfft_plan_dist) on this rank's
    points; the exchange (NCCL collective or the grid-slab peer-memory steps) runs inside
    libhpnfft.so.  torch.distributed only carries the 128-byte NCCL unique id.

    group   : torch.distributed process group (None = WORLD)
    mode    : "allreduce" | "reduce" | "reduce_scatter" | "grid_slab"
    """

    def __init__(self, N, M_local: int, m: int = 6, sigma: float = 2.0, window="kb", group=None,
                 mode: str = "allreduce", device=None, slab_edges=None):
        import torch.distributed as dist

        from . import Plan, get_unique_id

        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        self.N = tuple(int(v) for v in N)
        self.mode = mode
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if mode == "reduce_scatter" and self.N[0] % self.world:
            raise ValueError("reduce_scatter needs N0 divisible by the world size")
        if mode == "grid_slab" and self.N[1] % self.world:
            raise ValueError("grid_slab needs N1 divisible by the world size")
        uid = [get_unique_id() if self.rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(uid, src=src, group=group)
        self.plan = Plan(self.N, M_local, m=m, sigma=sigma, window=window, device=device,
                         dist=(self.world, self.rank, uid[0], mode))
        if slab_edges is not None and self.world > 1:
            self.plan.set_slabs(slab_edges)

    def set_points(self, x):
        self.plan.set_points(x)

    def adjoint(self, f, out=None):
        """This rank's block of fhat = sum over ranks of the partial transforms (Eq. 8; Accumulate
        of Alg. 3): the full fhat (allreduce; reduce on rank 0, None elsewhere), the k0 slab
        (reduce_scatter) or the k1 slab (grid_slab)."""
        out = self.plan.adjoint(f, out=out)
        return None if (self.mode == "reduce" and self.rank != 0) else out

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None
