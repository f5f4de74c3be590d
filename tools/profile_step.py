"""One warm-up + one profiled pass of the hot path at a BASELINE config (for ncu captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs.device as idev  # noqa: E402
import paper_2001_01583_b200 as hp  # noqa: E402

CONFIGS = {"3": ((128,) * 3, 10 ** 6), "4": ((256,) * 3, 10 ** 7), "5": ((512,) * 3, 10 ** 8)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--dist", default="uniform")
ap.add_argument("--method", default="auto")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--timing", action="store_true")
ap.add_argument("--inverse", action="store_true")
a = ap.parse_args()
N, M = CONFIGS[a.config]
dev = torch.device("cuda", 0)
x = idev.uniform_points(M, device=dev) if a.dist == "uniform" else idev.clustered_points(M, device=dev)
f = idev.uniform_values(M, device=dev)
plan = hp.Plan(N, M, device=dev)
plan.set_spread_method(a.method)
ap2 = None
for r in range(a.reps):
    if r == a.reps - 1 and a.timing:
        plan.enable_timing(True)
    plan.set_points(x)
    out = plan.adjoint(f)
    if a.inverse:
        fl = plan.inverse(out)
torch.cuda.synchronize()
msg = {"config": a.config, "dist": a.dist, "patch": os.environ.get("HPNFFT_SWEEP_PATCH", "default")}
if a.timing:
    msg.update(plan.stage_times())
print("ok", float(out.abs().sum()), msg)
