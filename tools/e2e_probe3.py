"""Streamed e2e with events at every boundary (inline copy of HostPipeline.submit)."""
import os, sys, time
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
oh = [torch.empty(N, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
del x, f
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
comp = torch.cuda.Stream()
print("streams", h2d, d2h, comp, torch.cuda.current_stream())
X = [torch.empty((M, 3), dtype=torch.float64, device=dev) for _ in range(2)]
F = [torch.empty((M,), dtype=torch.complex128, device=dev) for _ in range(2)]
O = [torch.empty(N, dtype=torch.complex128, device=dev) for _ in range(2)]
E = lambda: torch.cuda.Event(enable_timing=True)
base = E(); base.record(h2d); torch.cuda.synchronize()
log = []
used = [None, None]; drained = [None, None]; pending = None
t_host0 = time.perf_counter()
for i in range(6):
    s = i & 1
    ev = {}
    with torch.cuda.stream(h2d):
        if used[s] is not None: h2d.wait_event(used[s])
        ev['x0'] = E(); ev['x0'].record(h2d)
        X[s].copy_(xh, non_blocking=True)
        ev['x1'] = E(); ev['x1'].record(h2d)
        F[s].copy_(fh, non_blocking=True)
        ev['f1'] = E(); ev['f1'].record(h2d)
    if pending is not None:
        ps, pout, pdone = pending
        with torch.cuda.stream(d2h):
            d2h.wait_event(pdone)
            ev['d0'] = E(); ev['d0'].record(d2h)
            pout.copy_(O[ps], non_blocking=True)
            ev['d1'] = E(); ev['d1'].record(d2h)
            dr = torch.cuda.Event(); dr.record(d2h); drained[ps] = dr
    comp.wait_event(ev['x1'])
    if drained[s] is not None: comp.wait_event(drained[s])
    with torch.cuda.stream(comp):
        ev['c0'] = E(); ev['c0'].record(comp)
        th = time.perf_counter()
        plan.set_points(X[s])
        th = time.perf_counter() - th
        comp.wait_event(ev['f1'])
        plan.adjoint(F[s], out=O[s])
        ev['c1'] = E(); ev['c1'].record(comp)
    used[s] = ev['c1']
    pending = (s, oh[s], ev['c1'])
    log.append((ev, th, time.perf_counter() - t_host0))
torch.cuda.synchronize()
for i, (ev, th, tw) in enumerate(log):
    r = {k: round(base.elapsed_time(v), 2) for k, v in ev.items()}
    print(i, r, "set_points host %.2f" % (th * 1e3), "host clock %.2f" % (tw * 1e3))
