"""Per-rank cost of grid-slab partitions, emulated on ONE GPU: for each rank's slab the points it
would own are transformed by a single-GPU plan (occupied planes only, as the grid-slab rank
spreads), and the spread stages are timed.  Fits spread_ms = a * points + b * planes to pick the
plane weight of dist.grid_slab_edges (equal-cost slabs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs.device as idev  # noqa: E402
import paper_2001_01583_b200 as hp  # noqa: E402
from paper_2001_01583_b200.dist import grid_slab_edges, grid_slab_mask  # noqa: E402

N, M = (256,) * 3, 10 ** 7
n0 = 512
dev = torch.device("cuda", 0)
rows = []
for dist_kind in ("uniform", "clustered"):
    x = idev.uniform_points(M, device=dev) if dist_kind == "uniform" else idev.clustered_points(M, device=dev)
    f = idev.uniform_values(M, device=dev)
    for P in (2, 4, 8):
        weights = [None, 0.0] + [float(w) for w in os.environ.get("PLANE_WEIGHTS", "").split(",") if w]
        for w in weights:
            if w is None:
                edges = [n0 // 2 + r * n0 // P for r in range(P + 1)]   # equal-size, rotated labels
                tag = "equal_size"
            else:
                edges = grid_slab_edges(x, P, n0, reduce=False, plane_weight=w)
                tag = f"w={w:g}"
            times = []
            for r in range(P):
                mk = grid_slab_mask(x, r, P, n0, edges)
                xl, fl = x[mk].contiguous(), f[mk].contiguous()
                plan = hp.Plan(N, xl.shape[0], device=dev)
                for rep in range(3):
                    plan.enable_timing(rep == 2)
                    plan.set_points(xl)
                    plan.adjoint(fl)
                torch.cuda.synchronize()
                st = plan.stage_times()
                spread = st["spread"] + st["keys"] + st["scan"] + st["scatter"]
                planes = edges[r + 1] - edges[r]
                fzy = (st["fft_z"] + st["fft_y"]) * planes / n0   # the rank's share of the z, y passes
                times.append(spread + fzy)
                rows.append((xl.shape[0], planes, spread, fzy / planes))
                plan.close()
            print(f"{dist_kind} P={P} {tag}: edges={edges} max={max(times):.3f} ms "
                  f"per-rank={[round(t, 3) for t in times]}", flush=True)
A = np.array([[r[0], r[1]] for r in rows], dtype=np.float64)
y = np.array([r[2] for r in rows])
coef, *_ = np.linalg.lstsq(A, y, rcond=None)
fzy = float(np.mean([r[3] for r in rows]))
print(f"fit spread+sort ms = {coef[0]:.3e} * points + {coef[1]:.3e} * planes; fft z+y {fzy:.3e} ms/plane "
      f"-> plane weight {(coef[1] + fzy) / coef[0]:.0f} points")
