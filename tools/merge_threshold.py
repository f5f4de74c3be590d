"""Sweep kernel choice vs point density: the one-chunk (dense) and merged-chunk (sparse) sweeps timed
on the same uniform points (HPNFFT_SWEEP_MERGE read per call) at N = 256^3 (grid 512^3) for a range
of M; prints the expected records per (tile, chunk) the automatic choice uses (threshold 64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs.device as idev  # noqa: E402
import paper_2001_01583_b200 as hp  # noqa: E402

dev = torch.device("cuda", 0)
N = (256, 256, 256)
for M in [int(v) for v in os.environ.get("MT_M", "500000,1000000,2000000,3000000,5000000,10000000").split(",")]:
    x = idev.uniform_points(M, device=dev)
    f = idev.uniform_values(M, device=dev)
    plan = hp.Plan(N, M, device=dev)
    plan.set_points(x)
    per_chunk = M / (512.0 ** 3) * 19 * 43 * 4
    res = {}
    for mode in ("0", "1"):
        os.environ["HPNFFT_SWEEP_MERGE"] = mode
        out = plan.adjoint(f)
        for _ in range(3):
            plan.adjoint(f, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.adjoint(f, out=out)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 10
    os.environ.pop("HPNFFT_SWEEP_MERGE", None)
    print(f"M={M:>9d} records/(tile,chunk)={per_chunk:7.1f} adjoint dense {res['0']:.3f} ms merged {res['1']:.3f} ms",
          flush=True)
    plan.close()
    del x, f
    torch.cuda.empty_cache()
