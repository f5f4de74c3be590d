"""H2D speed: alone, concurrent with the adjoint kernels, concurrent with a D2H."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import inputs.device as idev
import paper_2001_01583_b200 as hp

dev = torch.device("cuda", 0)
N, M = (256, 256, 256), 10 ** 7
x = idev.uniform_points(M, device=dev)
f = idev.uniform_values(M, device=dev)
plan = hp.Plan(N, M, device=dev)
xh, fh = x.cpu().pin_memory(), f.cpu().pin_memory()
oh = torch.empty(N, dtype=torch.complex128, pin_memory=True)
xd = torch.empty_like(x)
o = plan.adjoint(f) if False else None
plan.set_points(x); o = plan.adjoint(f)
torch.cuda.synchronize()
s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
def ev():
    return torch.cuda.Event(enable_timing=True)
# 1. alone
a, b = ev(), ev()
with torch.cuda.stream(s_h2d):
    a.record(); xd.copy_(xh, non_blocking=True); b.record()
torch.cuda.synchronize(); print("H2D x alone %.2f ms" % a.elapsed_time(b))
# 2. concurrent with adjoint kernels on the default stream
c0, c1 = ev(), ev()
c0.record()
plan.set_points(x); plan.adjoint(f, out=o)
with torch.cuda.stream(s_h2d):
    a.record(); xd.copy_(xh, non_blocking=True); b.record()
c1.record()
torch.cuda.synchronize(); print("H2D x during set_points+adjoint %.2f ms (compute %.2f)" % (a.elapsed_time(b), c0.elapsed_time(c1)))
# 3. concurrently issued BEFORE the kernels
with torch.cuda.stream(s_h2d):
    a.record(); xd.copy_(xh, non_blocking=True); b.record()
c0.record(); plan.adjoint(f, out=o); c1.record()
torch.cuda.synchronize(); print("H2D x issued first, adjoint after: h2d %.2f ms, adjoint %.2f" % (a.elapsed_time(b), c0.elapsed_time(c1)))
# 4. with D2H
d0, d1 = ev(), ev()
with torch.cuda.stream(s_d2h):
    d0.record(); oh.copy_(o, non_blocking=True); d1.record()
with torch.cuda.stream(s_h2d):
    a.record(); xd.copy_(xh, non_blocking=True); b.record()
torch.cuda.synchronize(); print("D2H %.2f ms with H2D %.2f ms concurrently" % (d0.elapsed_time(d1), a.elapsed_time(b)))
