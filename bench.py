#!/usr/bin/env python
"""Benchmark of the B200 adjoint NFFT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dist uniform|clustered] [--config 4|3|5] [--method auto|atomic|sweep]

Workload (BASELINE.json configs[3], the metric's config): d = 3, N = 256^3, M = 10^7 points,
float64, Kaiser-Bessel m = 6, sigma = 2 (grid 512^3).  One step = one pass of the whole hot
path: set_points (keys, bin sort) + adjoint (records, sweep spread, 3 pruned
FFT passes with the fused deconvolve/crop).  For N > 1 GPUs every rank generates and owns the
points of one x-slab subcell ("subcells with same size") and the library's exchange
combines the partial results (Eq. 8 / Alg. 3): by default option G
(--exchange grid_slab: halo + distributed FFT over NVLink peer memory), or option A (NCCL
collective on fhat).  Total work is fixed as N grows (strong scaling).  Inputs are resident in
HBM before the timed region and are larger than L2 (x 240 MB, f 160 MB, grid 2.1 GB), so no
explicit L2 flush is needed.

cpu_baseline: the oracle's whole transform of the workload once on all host cores.
--impl reference: the oracle (oracle/, the independent CPU NFFT) timed on the host cores, each
step a complete transform of a bounded sample of the workload's points.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {
    "3": {"N": (128, 128, 128), "M": 10 ** 6},
    "4": {"N": (256, 256, 256), "M": 10 ** 7},
    "5": {"N": (512, 512, 512), "M": 10 ** 9},
}
METRIC = "adjoint NFFT nonuniform points/s at N=256³ float64, 1/2/4/8 B200; E2 error"
EXCHANGE_TEXT = {
    "nccl_collective": "option A: one NCCL collective on fhat inside libhpnfft.so ({mode})",
    "grid_slab_nvlink_p2p": "option G: grid halo pulled from the neighbours' grids + distributed pruned FFT whose "
                            "y-pass epilogue stores into the destination ranks' grids (the all-to-all), over NVLink "
                            "peer memory (CUDA IPC) inside libhpnfft.so; fhat left in k1 slabs",
    "grid_slab_nccl_sendrecv": "option G over NCCL send/recv (peer memory unavailable): halo runs + pack + grouped "
                               "all-to-all inside libhpnfft.so; fhat left in k1 slabs",
    "none": "none",
}
M_WINDOW, SIGMA = 6, 2.0
# FP64 tensor-core (DMMA m8n8k4) peak MEASURED on this pool's B200 with tools/ubench_dmma.cu /
# tools/ubench_kstep.cu (profiles/ubench_dmma.txt, profiles/ubench_kstep.txt): 36.7 TFLOP/s for
# back-to-back DMMAs (DFMA and DMMA share this throughput: profiles/ubench_mix.txt).  The
# fallback rule (bf16 measured x nominal FP64/bf16 ratio = 1653.7 / 56.25 = 29.4) would be lower,
# so the measured number is the conservative denominator.
FP64_TC_PEAK_TFLOPS = 36.7
FP64_FMA_PEAK_TFLOPS = 34.2   # DFMA chains, tools/ubench_fp64.cu (profiles/ubench_fp64.txt)


def spread_flops_per_point(m: int) -> float:
    """Algorithmic FP64 work of the spread per point: 2(2m)^3 FMAs for the
    complex-times-real tap updates + 2(2m)^2 for the per-(i1,i2) coefficient, 2 flop each."""
    w = 2 * m
    return 2.0 * (2 * w ** 3 + 2 * w ** 2)


def fft_bytes(N, sigma=2.0):
    """Algorithmic HBM bytes of the three pruned FFT passes."""
    n = [int(sigma * v) for v in N]
    c = 16
    z = c * (n[0] * n[1] * n[2] + n[0] * n[1] * N[2])
    y = c * (n[0] * n[1] * N[2] + n[0] * N[1] * N[2])
    x = c * (n[0] * N[1] * N[2] + N[0] * N[1] * N[2])
    return {"fft_z": z, "fft_y": y, "fft_x_deconv": x}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(cfg, dist_kind, device):
    import inputs.device as idev

    M = cfg["M"]
    if dist_kind == "clustered":
        x = idev.clustered_points(M, s=0.05, device=device)
    else:
        x = idev.uniform_points(M, device=device)
    f = idev.uniform_values(M, device=device)
    return x, f


def shard_inputs(cfg, dist_kind, device, rank, ws, partition="equal_size", exchange="grid_slab", n0=512):
    """This rank's x-slab subcell of the seeded workload, generated in place: the
    counter-based generator is streamed over the M points in chunks and only the rank's points
    are kept (no full copy of the M points on any rank).  Equal-size slabs, equal-count slabs, or
    the cell-aligned slabs of the grid_slab exchange (option G; equal-cost edges from the summed
    plane histogram, every rank computes the same)."""
    import torch

    import inputs.device as idev
    from paper_2001_01583_b200.dist import equal_count_edges, grid_slab_edges_hist, grid_slab_mask, slab_mask

    M = cfg["M"]
    chunk = 1 << 25

    def gen(start, cnt):
        if dist_kind == "clustered":
            xx = idev.clustered_points(cnt, s=0.05, start=start, device=device)
        else:
            xx = idev.uniform_points(cnt, start=start, device=device)
        return xx, idev.uniform_values(cnt, start=start, device=device)

    edges = None
    if partition == "equal_count":   # a first pass over the chunks: the histogram / quantiles of all M points
        if exchange == "grid_slab":
            hist = torch.zeros(n0, dtype=torch.int64, device=device)
            for s0 in range(0, M, chunk):
                xx, _ = gen(s0, min(chunk, M - s0))
                c0 = torch.floor(xx[:, 0] * float(n0)).to(torch.int64) % n0   # memory plane
                hist += torch.bincount(c0, minlength=n0)
            edges = grid_slab_edges_hist(hist, ws, n0, m=M_WINDOW)
        else:
            xs = [gen(s0, min(chunk, M - s0))[0][:, 0].clone() for s0 in range(0, M, chunk)]
            edges = equal_count_edges(torch.cat(xs).unsqueeze(1), ws)
    xs, fs = [], []
    for s0 in range(0, M, chunk):
        xx, ff = gen(s0, min(chunk, M - s0))
        if exchange == "grid_slab":
            mask = grid_slab_mask(xx, rank, ws, n0, edges)
        else:
            mask = slab_mask(xx, rank, ws, edges)
        xs.append(xx[mask].contiguous())
        fs.append(ff[mask].contiguous())
        del xx, ff, mask
    x = torch.cat(xs) if len(xs) > 1 else xs[0]
    f = torch.cat(fs) if len(fs) > 1 else fs[0]
    del xs, fs
    torch.cuda.empty_cache()
    return x, f, (edges if exchange == "grid_slab" else None)


def run_ours(args):
    import torch
    import torch.distributed as tdist

    import paper_2001_01583_b200 as hp

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = CONFIGS[args.config]
    N = cfg["N"]
    M_total = cfg["M"]
    if ws == 1:
        x, f = make_inputs(cfg, args.dist, dev)
        slab_edges = None
    else:
        x, f, slab_edges = shard_inputs(cfg, args.dist, dev, rank, ws, args.partition, args.exchange,
                                        int(SIGMA * N[0]))
    M_local = x.shape[0]
    torch.cuda.synchronize()

    if ws > 1:   # the library's multi-GPU plan: the exchange runs inside libhpnfft.so (NCCL)
        from paper_2001_01583_b200.dist import DistPlan

        dplan = DistPlan(N, M_local, m=M_WINDOW, sigma=SIGMA, window="kb", mode=args.exchange, device=dev,
                         slab_edges=slab_edges)
        plan = dplan.plan
    else:
        plan = hp.Plan(N, M_local, m=M_WINDOW, sigma=SIGMA, window="kb", device=dev)
    plan.set_spread_method(args.method)
    out = torch.empty(plan.out_shape, dtype=torch.complex128, device=dev)

    inverse = args.direction == "inverse"
    if inverse:   # Eq. 6: input the full spectrum, output this rank's points (Alg. 4)
        gen = torch.Generator(device=dev)
        gen.manual_seed(2006)
        fhat_in = torch.randn(N, dtype=torch.complex128, device=dev, generator=gen)
        f_out = torch.empty(M_local, dtype=torch.complex128, device=dev)

    def step():
        plan.set_points(x)
        if inverse:
            plan.inverse(fhat_in, out=f_out)
        else:
            plan.adjoint(f, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = plan.launch_count()

    # ---- timed region: K steps, CUDA events on the plan's (current) stream ----
    plan.enable_timing(True)
    plan.stage_times()   # reset
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if ws > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    clocks = sampler.stop()
    ms_local = e0.elapsed_time(e1)
    stages = plan.stage_times()
    plan.enable_timing(False)
    if os.environ.get("HPNFFT_BENCH_RANK_STAGES"):   # diagnostics: every rank's own stage times
        print(json.dumps({"rank": rank, "M_local": M_local, "ms": ms_local / args.steps, "info": plan.info()["planes"],
                          "stages": {k: round(v, 4) for k, v in stages.items()}}), file=sys.stderr, flush=True)
    ms = ms_local
    if ws > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = M_total / (ms_per_step * 1e-3)

    # ---- e2e: the public API with HOST buffers (pinned), H2D + transform + D2H each step ----
    if inverse:
        return _finish_inverse(args, plan, stages, ms_per_step, value, ws, rank, launches_per_step, clocks, N,
                               M_total, M_local)
    xh = x.cpu().pin_memory()
    fh = f.cpu().pin_memory()
    oh = [torch.empty(plan.out_shape, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    # the device-resident inputs are not needed any more; two device buffer sets when they fit
    del x, f, out
    torch.cuda.empty_cache()
    need = M_local * (24 + 16) + 16 * plan.out_shape[0] * plan.out_shape[1] * plan.out_shape[2]
    depth = 2 if torch.cuda.mem_get_info(dev)[0] > 2 * need + (1 << 30) else 1
    pipe = hp.HostPipeline(plan, M_local, depth=depth)

    def e2e_step(i):
        pipe.submit(xh, fh, oh[i & 1])

    for i in range(max(2, min(args.warmup, 3))):
        e2e_step(i)
    pipe.flush()
    torch.cuda.synchronize()
    k_e2e = max(2, min(args.steps, 8))
    if ws > 1:
        tdist.barrier()
    # device-side timing on the compute stream, bracketing K submitted transforms and the drain
    # of the last D2H copy (the copy streams are joined back into the compute stream)
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record()
    for i in range(k_e2e):
        e2e_step(i)
    cs = torch.cuda.current_stream()
    cs.wait_stream(pipe.d2h)
    cs.wait_stream(pipe.h2d)
    a1.record()
    torch.cuda.synchronize()
    e2e_ms = a0.elapsed_time(a1) / k_e2e
    if ws > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = int(xh.numel() * 8 + fh.numel() * 16)
    d2h = int(oh[0].numel() * 16)

    # ---- roofline of the dominant kernel (largest stage) ----
    # the spread stage = point-record kernel + sweep kernel; the sweep is timed as the difference
    info = plan.info()
    kern = {k: v for k, v in stages.items() if k in ("fft_z", "fft_y", "fft_x_deconv")}
    if "spread" in stages:
        kern["sweep"] = stages["spread"] - stages.get("records", 0.0)
        kern["records"] = stages.get("records", 0.0)
    dom = max(kern, key=kern.get) if kern else "sweep"
    peaks = measured_peaks()
    traffic, traffic_src = None, None
    if ws == 1:   # the committed ncu capture is of the 1-GPU line of this config only
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
            traffic = tr.get(f"config{args.config}_{args.dist}_{dom}", tr.get(f"config{args.config}_{dom}"))
            traffic_src = tr.get("_source")
        except Exception:
            pass
    if dom in ("sweep", "records"):
        fl = M_local * spread_flops_per_point(M_WINDOW)
        achieved = fl / (kern["sweep"] * 1e-3) / 1e12
        roof = {"kernel": "k_spread_sweep", "bound": "tensor", "achieved": achieved, "peak": FP64_TC_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_TC_PEAK_TFLOPS, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_source": "measured FP64 DMMA m8n8k4 (tools/ubench_dmma.cu, profiles/ubench_dmma.txt)",
                "algorithmic": f"{spread_flops_per_point(M_WINDOW):.0f} flop/point x {M_local} points (this rank)",
                "timed_as": "spread stage - records stage (CUDA events on the plan stream)"}
    else:
        byts = info["pass_bytes"][dom]
        hbm = peaks.get("hbm_gbs", 6650.0)
        achieved = byts / (stages[dom] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650"}
    fft_ms = sum(stages.get(k, 0.0) for k in ("fft_z", "fft_y", "fft_x_deconv"))
    fbytes = sum(info["pass_bytes"].values())   # this rank's passes (its planes / k1 rows)
    extra = {
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "fft_hbm": {"achieved_gbs": fbytes / (fft_ms * 1e-3) / 1e9 if fft_ms else None,
                    "frac": (fbytes / (fft_ms * 1e-3) / 1e9) / peaks.get("hbm_gbs", 6650.0) if fft_ms else None,
                    "bytes": fbytes, "per_pass_bytes": info["pass_bytes"],
                    "how": "hpnfft_plan_info algorithmic bytes of this rank's three passes / their CUDA-event time"},
        "M_local": M_local,
        "record_group": info["record_group"],
        "workspace_bytes": info["workspace_bytes"],
    }

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.dist)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "points/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": f"synthetic seeded {args.dist} points (inputs/), counter-based generator",
            "config": {"workload": f"BASELINE config {args.config}: d=3, N={N[0]}^3, M={M_total}, "
                                   f"KB m={M_WINDOW}, sigma={SIGMA}, {args.dist}",
                       "N": list(N), "M": M_total, "m": M_WINDOW, "sigma": SIGMA, "window": "kaiser_bessel",
                       "points": args.dist, "partition": ((f"cell-aligned equal-cost x-slabs x{ws} (dist.grid_slab_edges)" if args.partition == "equal_count"
                                      else f"cell-aligned equal-size x-slabs x{ws}") if args.exchange == "grid_slab"
                                     else f"{args.partition} x-slabs x{ws}"),
                       "exchange": EXCHANGE_TEXT[info["exchange_path"]].format(mode=args.exchange),
                       "fhat_layout": ("full on every rank" if ws == 1 or args.exchange == "allreduce"
                                       else f"distributed: block {list(plan.out_shape)} per rank"),
                       "spread_method": args.method,
                       "l2": "inputs larger than L2 (x 240 MB, f 160 MB, grid 2.1 GB); no flush"},
            "e2e": {"value": M_total / (e2e_ms * 1e-3), "unit": "points/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "how": f"HostPipeline.submit per step (pinned host x, f -> device, set_points + adjoint, "
                           f"fhat -> pinned host), {depth} buffer set(s), copies on their own streams overlapping "
                           f"the neighbouring steps' kernels; CUDA events around K steps + final drain"},
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "detail": extra,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def _finish_inverse(args, plan, stages, ms_per_step, value, ws, rank, launches_per_step, clocks, N, M_total, M_local):
    """JSON line of the inverse direction (Eq. 6), a separate run."""
    import torch.distributed as tdist

    fl = M_local * 2.0 * (2 * M_WINDOW) ** 3 * 2.0          # 2 (2m)^3 FMA per point
    t_interp = stages.get("interp", 0.0)
    achieved = fl / (t_interp * 1e-3) / 1e12 if t_interp else None
    if rank == 0:
        line = {
            "metric": "inverse NFFT (Eq. 6) nonuniform points/s at N=256³ float64",
            "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": f"synthetic seeded {args.dist} points (inputs/), seeded random spectrum",
            "config": {"workload": f"config {args.config} inverse direction: d=3, N={N[0]}^3, M={M_total}, "
                                   f"KB m={M_WINDOW}, sigma={SIGMA}, {args.dist}",
                       "step": "set_points + inverse (subdivide + inverse FFT + interpolation); f left on the "
                               "rank that owns the point"},
            "e2e": None,
            "gpu_launches": int(launches_per_step * args.steps),
            "roofline": {"kernel": "k_spread_sweep<INV> (DMMA gather sweep)", "bound": "tensor", "achieved": achieved,
                         "peak": FP64_TC_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_TC_PEAK_TFLOPS if achieved else None, "traffic": None,
                         "peak_source": "measured FP64 DMMA m8n8k4 (tools/ubench_dmma.cu, profiles/ubench_dmma.txt)",
                         "algorithmic": "2 (2m)^3 FMA per point",
                         "timed_as": "interp stage (point records + gather sweep), CUDA events on the plan stream"},
            "cpu_baseline": None,
            "clocks": clocks,
            "detail": {"stages_ms": {k: round(v, 4) for k, v in stages.items()}, "M_local": M_local},
        }
        print(json.dumps(line), flush=True)
    plan.close()
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def run_f32(args):
    """--precision f32: the FP32 plan (float coordinates, complex64
    values, grid, FFT and fhat; shared-memory box spread) on config 4's points at --m (default 3,
    the survey's low-m FP32 regime).  One step = set_points_f32 + adjoint_f32; its own JSON line."""
    import torch

    import paper_2001_01583_b200 as hp

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = CONFIGS[args.config]
    N, M = cfg["N"], cfg["M"]
    m = args.m if args.m else 3
    x64, f64 = make_inputs(cfg, args.dist, dev)
    x, f = x64.to(torch.float32), f64.to(torch.complex64)
    del x64, f64
    plan = hp.Plan(N, M, m=m, sigma=SIGMA, window="kb", device=dev, precision="f32")
    out = torch.empty(plan.out_shape, dtype=torch.complex64, device=dev)

    def step():
        plan.set_points(x)
        plan.adjoint(f, out=out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = plan.launch_count()
    plan.enable_timing(True)
    plan.stage_times()
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    stages = plan.stage_times()
    ms = e0.elapsed_time(e1) / args.steps
    info = plan.info()
    n = [int(SIGMA * v) for v in N]
    cells = n[0] * n[1] * n[2]
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    # the spread's algorithmic bytes: sorted coordinates (the plan's float64 copy, 24 B) + permutation
    # (4 B) + complex64 value (8 B) per point, the complex64 grid zeroed and written once (2 x 8 B/cell)
    sp_bytes = M * (24 + 4 + 8) + 2 * 8 * cells
    fft_ms = sum(stages.get(k, 0.0) for k in ("fft_z", "fft_y", "fft_x_deconv"))
    fft_b = sum(info["pass_bytes"].values()) // 2   # complex64: half the float64 pass bytes
    dom = "spread" if stages.get("spread", 0.0) >= fft_ms else "fft"
    if dom == "spread":
        ach = sp_bytes / (stages["spread"] * 1e-3) / 1e9
        roof = {"kernel": "k_spread_red_f32 (+ grid zero fill)", "bound": "hbm", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                "algorithmic": "36 B/point (float64 sorted x, perm, complex64 f) + 16 B/cell (zero + write)",
                "limiter": f"L2 vector float2 reductions, (2m)^3 = {(2 * m) ** 3} per point: "
                           f"{M * (2 * m) ** 3 / (stages['spread'] * 1e-3):.3g} reductions/s (DESIGN.md §9e)"}
    else:
        ach = fft_b / (fft_ms * 1e-3) / 1e9
        roof = {"kernel": "k_fft_pass<complex64> z, y, x", "bound": "hbm", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": None, "algorithmic": "pruned pass bytes (complex64)"}
    line = {
        "metric": f"adjoint NFFT (FP32 variant, NEXT #4) nonuniform points/s at N={N[0]}^3, KB m={m}",
        "value": M / (ms * 1e-3), "unit": "points/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": f"synthetic seeded {args.dist} points (inputs/), rounded to float32",
        "config": {"workload": f"config {args.config} points, FP32 plan: d=3, N={N[0]}^3, M={M}, KB m={m}, "
                               f"sigma={SIGMA}, {args.dist}", "precision": "f32",
                   "l2": "inputs larger than L2; no flush"},
        "e2e": None, "gpu_launches": int(launches * args.steps), "roofline": roof, "cpu_baseline": None,
        "clocks": clocks,
        "detail": {"stages_ms": {k: round(v, 4) for k, v in stages.items()},
                   "fft_hbm_frac": (fft_b / (fft_ms * 1e-3) / 1e9) / hbm if fft_ms else None},
    }
    print(json.dumps(line), flush=True)
    plan.close()


# ----------------------------------------------------------------------------- CPU oracle --
def _host_cpu():
    """Host facts for the CPU-baseline record: usable cores and the CPU model."""
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cores, model


def _oracle_run(cfg, dist_kind, M_s):
    """The CPU oracle (oracle.nfft_adjoint's three steps, unmodified: O2 spread on all host cores
    by plane ownership, scipy FFT on all cores, deconvolve + crop) on the first M_s points of the
    workload's seeded point set.  Returns (seconds total, seconds spread, seconds FFT+deconvolve);
    input generation is outside the timed region."""
    import inputs
    import oracle

    N = cfg["N"]
    n = oracle.grid_size(N, SIGMA)
    x = inputs.clustered_points(M_s, s=0.05) if dist_kind == "clustered" else inputs.uniform_points(M_s)
    f = inputs.uniform_values(M_s)
    t0 = time.perf_counter()
    g = oracle.spread(x, f, n, M_WINDOW, SIGMA)
    t1 = time.perf_counter()
    oracle.deconvolve_crop(oracle.fft_grid(g), N, M_WINDOW, SIGMA)
    t2 = time.perf_counter()
    return t2 - t0, t1 - t0, t2 - t1


def cpu_baseline(cfg, dist_kind):
    """The whole oracle transform of the workload (all M points, full grid) once on the host's
    cores (config 4: ~10-20 s of CPU work); no extrapolation."""
    cores, model = _host_cpu()
    t, ts, tf = _oracle_run(cfg, dist_kind, cfg["M"])
    return {"value": cfg["M"] / t, "unit": "points/s", "cores": cores, "kind": "oracle",
            "sample": f"the full workload once: oracle/ CPU NFFT of all {cfg['M']} points (O2 spread "
                      f"{ts:.2f} s by grid-plane ownership on {cores} threads, scipy FFT + deconvolve/crop of "
                      f"the full grid {tf:.2f} s on {cores} workers) = {t:.2f} s",
            "cpu_model": model, "threads": cores}


REF_SAMPLE = 10 ** 6   # points per reference step (bounded sample of config 4's 1e7)


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on the host cores.  One step = the oracle
    transform of a bounded sample of the workload: the first min(M, 1e6) points of the seeded
    point set, spread onto the FULL oversampled grid, full-grid FFT, deconvolve + crop (every
    step is a complete transform of those points; value = points transformed / step time)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    M_s = min(cfg["M"], REF_SAMPLE)
    cores, model = _host_cpu()
    for _ in range(args.warmup):
        _oracle_run(cfg, args.dist, M_s)
    per, sp, ff = [], [], []
    for _ in range(args.steps):
        t, ts, tf = _oracle_run(cfg, args.dist, M_s)
        per.append(t)
        sp.append(ts)
        ff.append(tf)
    t_step = sum(per) / len(per)
    value = M_s / t_step
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "points/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_step * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": f"synthetic seeded {args.dist} points (inputs/)",
        "config": {"workload": f"BASELINE config {args.config}: d=3, N={cfg['N'][0]}^3, M={cfg['M']}, "
                               f"KB m={M_WINDOW}, sigma={SIGMA}, {args.dist}; each step transforms a bounded "
                               f"sample of {M_s} of its points on the full grid"},
        "cpu_baseline": {"value": value, "unit": "points/s", "kind": "oracle", "cores": cores, "threads": cores,
                         "cpu_model": model,
                         "sample": f"each step: oracle/ CPU NFFT of the first {M_s} points (O2 spread by plane "
                                   f"ownership, median {statistics.median(sp):.2f} s; scipy FFT + deconvolve/crop "
                                   f"of the full {int(SIGMA * cfg['N'][0])}^3 grid, median "
                                   f"{statistics.median(ff):.2f} s) on {cores} host threads; mean of {args.steps} "
                                   f"timed steps (median {statistics.median(per):.2f} s)"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dist", default="uniform", choices=["uniform", "clustered"])
    ap.add_argument("--config", default="4", choices=sorted(CONFIGS))
    ap.add_argument("--method", default="auto", choices=["auto", "atomic", "sweep"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partition", default="equal_size", choices=["equal_size", "equal_count"])
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="f32 = the FP32 plan (NEXT #4), its own JSON line")
    ap.add_argument("--m", type=int, default=0, help="window cut-off of the --precision f32 line (default 3)")
    ap.add_argument("--direction", default="adjoint", choices=["adjoint", "inverse"],
                    help="adjoint = Eq. 5 (the BASELINE metric); inverse = Eq. 6 (NEXT #1)")
    ap.add_argument("--exchange", default="grid_slab", choices=["allreduce", "reduce", "reduce_scatter", "grid_slab"],
                    help="multi-GPU exchange (SURVEY.md §8(e)); grid_slab = option G")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.precision == "f32":
        run_f32(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
