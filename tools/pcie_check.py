"""Pinned host <-> device copy rates on this box (H2D, D2H, both at once), for the e2e ceiling.
Under torchrun every rank measures its own GPU at the same time (shared host links)."""
import os

import torch

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if "WORLD_SIZE" in os.environ:
    import torch.distributed as dist

    dist.init_process_group("gloo")

n = 400 * 2 ** 20 // 8
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    if "WORLD_SIZE" in os.environ:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


b = n * 8 / 1e9
th = t(lambda: d.copy_(h, non_blocking=True))
td = t(lambda: h2.copy_(d2, non_blocking=True))
tb = t(both)
print(f"rank {local} cpu affinity {sorted(os.sched_getaffinity(0))[:4]}..({len(os.sched_getaffinity(0))}) H2D {b / th * 1e3:.1f} GB/s  D2H {b / td * 1e3:.1f} GB/s  both: {2 * b / tb * 1e3:.1f} GB/s total")
