"""Where does the streamed e2e step spend its time?  Events on each stream, per step."""
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
pipe = hp.HostPipeline(plan, M)
for i in range(3):
    pipe.submit(xh, fh, oh[i & 1])
pipe.flush()
torch.cuda.synchronize()
base = torch.cuda.Event(enable_timing=True)
base.record()
marks = []
K = 6
for i in range(K):
    s = i & 1
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("h0", "h1", "c0", "c1", "d0", "d1")}
    with torch.cuda.stream(pipe.h2d):
        ev["h0"].record(pipe.h2d)
    t_host = time.perf_counter()
    pipe.submit(xh, fh, oh[s])
    t_host = time.perf_counter() - t_host
    ev["h1"].record(pipe.h2d)
    ev["c1"].record(pipe.compute)
    ev["d1"].record(pipe.d2h)
    marks.append((ev, t_host))
pipe.flush()
torch.cuda.synchronize()
for i, (ev, th) in enumerate(marks):
    print(f"step {i}: h2d end {base.elapsed_time(ev['h1']):8.2f}  compute end {base.elapsed_time(ev['c1']):8.2f}  "
          f"d2h end {base.elapsed_time(ev['d1']):8.2f}  host in submit {th*1e3:6.2f} ms")
