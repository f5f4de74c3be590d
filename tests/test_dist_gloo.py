"""Multi-process host logic of the distributed layer on CPU (gloo, world_size 2).

The partition (equal-size x-slabs, and equal-count slabs) and the collectives of
DistPlan (Eq. 8 / Alg. 3 "Accumulate") are checked with the CPU
oracle injected as the local transform: the sum over ranks must equal the single-process NFFT.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N = (16, 16, 16)
M = 3000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class EmulatedDistPlan:
    """Test-only emulation of the exchange of paper_2001_01583_b200.dist.DistPlan: the local
    transform is the CPU oracle and the Accumulate step (Eq. 8, Alg. 3) is a torch.distributed
    collective, so that the partition helpers and the result layouts of the four modes can be
    checked on CPU with gloo.  (The library's own exchange runs on one GPU via hpnfft_plan_group
    in tests/test_gpu_parity.py.)"""

    def __init__(self, N, mode, local_fn):
        self.N, self.mode, self.local_fn = tuple(N), mode, local_fn
        self.world, self.rank = dist.get_world_size(), dist.get_rank()

    def set_points(self, x):
        self._x = x

    def adjoint(self, f):
        fh = self.local_fn(self._x, f)
        if self.mode == "allreduce":
            dist.all_reduce(fh, op=dist.ReduceOp.SUM)
            return fh
        if self.mode == "reduce":
            dist.reduce(fh, dst=0, op=dist.ReduceOp.SUM)
            return fh if self.rank == 0 else None
        dist.all_reduce(fh, op=dist.ReduceOp.SUM)   # gloo has no reduce_scatter: reduce + slice
        if self.mode == "grid_slab":   # rank r receives fhat[:, k1 slab r, :]
            cols = self.N[1] // self.world
            return fh[:, self.rank * cols:(self.rank + 1) * cols].contiguous()
        rows = self.N[0] // self.world   # reduce_scatter: fhat[k0 slab r]
        return fh[self.rank * rows:(self.rank + 1) * rows].clone()


def _worker(rank, world, port, mode, equal_count, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import inputs
        import oracle
        from paper_2001_01583_b200.dist import equal_count_edges, grid_slab_edges, grid_slab_mask, slab_mask

        x = torch.from_numpy(inputs.clustered_points(M, s=0.08) if equal_count else inputs.uniform_points(M))
        f = torch.from_numpy(inputs.uniform_values(M))
        edges = equal_count_edges(x, world) if equal_count else None
        if mode == "grid_slab":
            # equal-count cell-plane slabs from this rank's share of the histogram (summed over
            # the ranks inside grid_slab_edges: a collective)
            gedges = grid_slab_edges(x[rank::world], world, 2 * N[0], plane_weight=0) if equal_count else None
            mask = grid_slab_mask(x, rank, world, 2 * N[0], gedges)
        else:
            mask = slab_mask(x, rank, world, edges)
        xl, fl = x[mask], f[mask]

        def local(xx, ff):
            return torch.from_numpy(oracle.nfft_adjoint(xx.numpy(), ff.numpy(), N))

        dp = EmulatedDistPlan(N, mode, local)
        dp.set_points(xl)
        out = dp.adjoint(fl)
        counts = torch.tensor([int(mask.sum())])
        dist.all_reduce(counts)
        outq.put((rank, None if out is None else out.numpy(), int(counts.item()), int(mask.sum())))
    finally:
        dist.destroy_process_group()


def _run(world, mode, equal_count=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, equal_count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.fixture(scope="module")
def reference():
    import inputs
    import oracle

    x, f = inputs.uniform_points(M), inputs.uniform_values(M)
    return oracle.nfft_adjoint(x, f, N)


@pytest.mark.parametrize("mode", ["allreduce", "reduce", "reduce_scatter", "grid_slab"])
def test_dist_modes_sum_partials(mode, reference):
    import oracle

    res = _run(2, mode)
    assert all(r[2] == M for r in res)          # every point owned by exactly one rank
    if mode == "allreduce":
        for r in res:
            assert oracle.rel_l2_error(r[1], reference) < 1e-14
    elif mode == "reduce":
        assert oracle.rel_l2_error(res[0][1], reference) < 1e-14
        assert res[1][1] is None
    elif mode == "grid_slab":   # rank r holds fhat[:, k1 slab r, :]
        full = np.concatenate([r[1] for r in res], axis=1)
        assert oracle.rel_l2_error(full, reference) < 1e-14
    else:
        full = np.concatenate([r[1] for r in res], axis=0)
        assert oracle.rel_l2_error(full, reference) < 1e-14


def test_equal_count_partition_balances_clustered_points():
    import inputs
    import oracle

    res = _run(2, "allreduce", equal_count=True)
    assert sum(r[3] for r in res) == M
    assert abs(res[0][3] - res[1][3]) <= 2
    x, f = inputs.clustered_points(M, s=0.08), inputs.uniform_values(M)
    assert oracle.rel_l2_error(res[0][1], oracle.nfft_adjoint(x, f, N)) < 1e-14


def test_grid_slab_equal_count_clustered():
    """Equal-count grid slabs (hpnfft_set_slabs edges from the summed histogram) on clustered
    points: still a partition, better balanced than the equal-size cell slabs, same fhat."""
    import inputs
    import oracle
    from paper_2001_01583_b200.dist import grid_slab_rank

    res = _run(2, "grid_slab", equal_count=True)
    assert all(r[2] == M for r in res)
    x, f = inputs.clustered_points(M, s=0.08), inputs.uniform_values(M)
    full = np.concatenate([r[1] for r in res], axis=1)
    assert oracle.rel_l2_error(full, oracle.nfft_adjoint(x, f, N)) < 1e-14
    eq = torch.bincount(grid_slab_rank(torch.from_numpy(x), 2, 2 * N[0]), minlength=2)
    assert abs(res[0][3] - res[1][3]) <= abs(int(eq[0]) - int(eq[1]))


def test_grid_slab_edges_valid_and_balanced():
    """grid_slab_edges: cyclic edges from x = 0 (c0x = n0/2), multiples of 4 planes, every slab
    >= 2m planes; owners by bucketize agree with a plain per-point loop; uniform points give
    near-equal counts and clustered points counts within one 4-plane band of M/P."""
    import inputs
    from paper_2001_01583_b200.dist import grid_slab_edges, grid_slab_rank

    n0, m = 512, 6
    for world in (2, 4, 8):
        for pts in (inputs.uniform_points(20000), inputs.clustered_points(20000, s=0.1)):
            x = torch.from_numpy(pts)
            e = grid_slab_edges(x, world, n0, m=m, plane_weight=0)
            assert len(e) == world + 1 and e[0] == n0 // 2 and e[-1] == e[0] + n0
            lens = [e[r + 1] - e[r] for r in range(world)]
            assert all(L % 4 == 0 and L >= 2 * m for L in lens)
            own = grid_slab_rank(x, world, n0, e)
            c0x = [(int(np.floor(n0 * v)) % n0 + n0 // 2) % n0 for v in pts[:500, 0]]
            brute = [next(r for r in range(world) if (c - e[r]) % n0 < lens[r]) for c in c0x]
            assert own[:500].tolist() == brute
            cnt = torch.bincount(own, minlength=world).tolist()
            assert sum(cnt) == len(pts)
            band = torch.bincount(torch.tensor([(int(np.floor(n0 * v)) % n0) // 4 for v in pts[:, 0]]),
                                  minlength=n0 // 4).max().item()
            # every edge is within one 4-plane band of its quantile, unless the 2m minimum binds
            assert max(cnt) - min(cnt) <= 2 * band + 1


def test_slab_mask_is_partition():
    from paper_2001_01583_b200.dist import slab_mask

    x = torch.tensor([[-0.5, 0, 0], [0.5, 0, 0], [-0.25, 0, 0], [0.0, 0, 0], [0.4999, 0, 0]], dtype=torch.float64)
    for world in (1, 2, 3, 4, 8):
        owners = torch.stack([slab_mask(x, r, world) for r in range(world)]).sum(0)
        assert torch.all(owners == 1)


def test_grid_slab_rank_follows_the_cell_planes():
    """grid_slab owners: x-ordered cell plane c0x = (floor(n0 x0) + n0/2) mod n0 in the rank's
    n0/P planes, i.e. the equal-size slab [-1/2 + r/P, -1/2 + (r+1)/P); x0 = 1/2
    is x0 = -1/2 by periodicity and belongs to rank 0."""
    from paper_2001_01583_b200.dist import grid_slab_rank

    n0, world = 32, 4
    x0 = torch.tensor([-0.5, -0.25 - 1e-12, -0.25, 0.0, 0.2499999, 0.25, 0.49, 0.5], dtype=torch.float64)
    x = torch.stack([x0, torch.zeros_like(x0), torch.zeros_like(x0)], 1)
    assert grid_slab_rank(x, world, n0).tolist() == [0, 0, 1, 2, 2, 3, 3, 0]


def test_grid_slab_edges_from_histogram_match():
    """bench.py's chunked shard generation cuts the slabs on a histogram accumulated chunk by chunk
    (dist.grid_slab_edges_hist); it must give the same edges as dist.grid_slab_edges on the points."""
    import inputs
    from paper_2001_01583_b200.dist import grid_slab_edges, grid_slab_edges_hist

    x = torch.from_numpy(inputs.clustered_points(50000, s=0.05))
    n0 = 128
    c0 = torch.floor(x[:, 0] * float(n0)).to(torch.int64) % n0
    hist = torch.zeros(n0, dtype=torch.int64)
    for part in torch.split(c0, 7777):   # chunk by chunk, as bench.shard_inputs does
        hist += torch.bincount(part, minlength=n0)
    for world in (2, 4):
        for w in (0.0, 8000.0):
            a = grid_slab_edges(x, world, n0, m=6, reduce=False, plane_weight=w)
            b = grid_slab_edges_hist(hist, world, n0, m=6, plane_weight=w)
            assert a == b
            assert len(a) == world + 1 and a[-1] - a[0] == n0
