"""Small cases of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), one tool per gpurun call (profiles/r2_sanitizer.md):
  the DMMA sweep spread (single-chunk and multi-chunk batches, clustered, multi-group records),
  the gather sweep (inverse), the atomic spread and warp gather, the FFT passes, the Eq. 12
  energy, and a one-GPU grid-slab rank group (halo pull, fused peer-store y pass, x pass).
Each case is checked against the CPU oracle so a silent corruption also fails the run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_2001_01583_b200 as hp  # noqa: E402

dev = torch.device("cuda", 0)
fails = []


def check(name, got, ref, tol):
    e = oracle.rel_l2_error(got, ref)
    print(f"{name:40s} E2 {e:.2e}", flush=True)
    if not e <= tol:
        fails.append(name)


def adjoint(N, x, f, method="auto", m=6):
    p = hp.Plan(N, x.shape[0], m=m, device=dev)
    p.set_spread_method(method)
    p.set_points(torch.from_numpy(x).to(dev))
    out = p.adjoint(torch.from_numpy(f).to(dev)).cpu().numpy()
    p.close()
    return out


N = (32, 32, 32)
M = 2000
x, f = inputs.uniform_points(M, seed=1), inputs.uniform_values(M, seed=1)
xc = inputs.clustered_points(M, s=0.05, seed=2)
ref, refc = oracle.nfft_adjoint(x, f, N), oracle.nfft_adjoint(xc, f, N)
check("sweep uniform", adjoint(N, x, f, "sweep"), ref, 1e-12)
check("sweep clustered", adjoint(N, xc, f, "sweep"), refc, 1e-12)
os.environ["HPNFFT_SWEEP_MERGE"] = "1"
check("sweep multi-chunk batches", adjoint(N, x, f, "sweep"), ref, 1e-12)
os.environ.pop("HPNFFT_SWEEP_MERGE")
os.environ["HPNFFT_REC_GROUP"] = "1024"
check("sweep multi-group records", adjoint(N, xc, f, "sweep"), refc, 1e-12)
os.environ.pop("HPNFFT_REC_GROUP")
check("atomic spread", adjoint(N, x, f, "atomic"), ref, 1e-12)
check("atomic spread m=11", adjoint(N, x, f, "atomic", m=11), oracle.nfft_adjoint(x, f, N, m=11), 1e-12)

rng = np.random.default_rng(3)
spec = rng.standard_normal(N) + 1j * rng.standard_normal(N)
for meth in ("auto", "atomic"):
    p = hp.Plan(N, M, device=dev)
    p.set_spread_method(meth)
    p.set_points(torch.from_numpy(xc).to(dev))
    got = p.inverse(torch.from_numpy(spec).to(dev)).cpu().numpy()
    p.close()
    check(f"inverse ({meth})", got, oracle.nfft_inverse(xc, spec, N), 1e-12)

# Eq. 12 energy (fused x pass) on random charges
q = rng.standard_normal(M)
p = hp.Plan(N, M, device=dev)
p.set_points(torch.from_numpy(x).to(dev))
U = p.ewald_reciprocal(torch.from_numpy(q).to(dev), 10.0, 0.9).item()
p.close()
fh = oracle.nfft_adjoint(x, q.astype(complex), N)
k = np.meshgrid(*[np.arange(-v // 2, v // 2) for v in N], indexing="ij")
nn = sum(kk.astype(float) ** 2 for kk in k)
w = np.where(nn > 0, np.exp(-np.pi ** 2 * nn / (0.9 * 10.0) ** 2) / np.where(nn > 0, nn, 1), 0.0)
Uref = (w * np.abs(fh) ** 2).sum() / (2 * np.pi * 10.0) - 0.9 / np.sqrt(np.pi) * (q ** 2).sum()
check("ewald reciprocal", np.array([U]), np.array([Uref]), 1e-11)

# one-GPU grid-slab rank group, P = 2
from paper_2001_01583_b200.dist import grid_slab_rank  # noqa: E402

owner = grid_slab_rank(torch.from_numpy(xc), 2, 2 * N[0]).numpy()
parts = [np.nonzero(owner == r)[0] for r in range(2)]
g = hp.PlanGroup(N, [len(pp) for pp in parts], mode="grid_slab", device=dev)
g.set_points([torch.from_numpy(np.ascontiguousarray(xc[pp])).to(dev) for pp in parts])
outs = g.adjoint([torch.from_numpy(np.ascontiguousarray(f[pp])).to(dev) for pp in parts])
full = np.concatenate([o.cpu().numpy() for o in outs], axis=1)
g.close()
check("grid-slab rank group P=2", full, refc, 1e-12)
torch.cuda.synchronize()
print("FAILED: " + ", ".join(fails) if fails else "all cases ok")
sys.exit(1 if fails else 0)
