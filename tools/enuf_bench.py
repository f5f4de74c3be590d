"""Time the ENUF reciprocal energy (hpnfft_ewald_reciprocal, Eq. 12) on the paper's fluorite
systems of Fig. 16: 12 c^3 ions for c = 32, 45, 56, 64 cells per side (L = c l,
l = 4/sqrt(3) r0), alpha = 1.2 / r0, N = 256^3 (c = 32) or 512^3.  One step = set_points +
ewald_reciprocal with the positions and charges resident in HBM; CUDA events over 10 steps after
3 warm-ups.  Prints one line per system (no oracle here: the values are pinned by the -m gpu
tests)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2001_01583_b200 as hp  # noqa: E402

dev = torch.device("cuda", 0)
alpha = 1.2
for c in [int(v) for v in os.environ.get("ENUF_CELLS", "32,45,56,64").split(",")]:
    N = (256,) * 3 if c <= 32 else (512,) * 3
    r, q, L = inputs.crystal("caf2", c)
    x = torch.from_numpy(r / L - 0.5).to(dev)
    qd = torch.from_numpy(q).to(dev)
    plan = hp.Plan(N, x.shape[0], device=dev)
    plan.set_spread_method(os.environ.get("ENUF_METHOD", "auto"))
    out = torch.empty(1, dtype=torch.float64, device=dev)
    for _ in range(3):
        plan.set_points(x)
        plan.ewald_reciprocal(qd, L, alpha, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 10
    e0.record()
    for _ in range(steps):
        plan.set_points(x)
        plan.ewald_reciprocal(qd, L, alpha, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    plan.enable_timing(True)
    plan.set_points(x)
    plan.ewald_reciprocal(qd, L, alpha, out=out)
    torch.cuda.synchronize()
    st = {k: round(v, 3) for k, v in plan.stage_times().items() if v}
    print(f"cells={c}^3 ions={x.shape[0]} N={N[0]}^3 L={L:.2f} U^K={out.item():.10e} "
          f"step={ms:.3f} ms ({x.shape[0] / ms * 1e3:.3e} ions/s) U^K per ion={out.item() / x.shape[0]:.10f} "
          f"stages={st}", flush=True)
    plan.close()
    del x, qd
    torch.cuda.empty_cache()
