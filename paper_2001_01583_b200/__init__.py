"""B200-native adjoint NFFT (the HP-NFFT hot path of arXiv 2001.01583).

Thin Python binding over the C ABI in include/hpnfft.h (libhpnfft.so, sm_100a).  This module
only marshals arguments: torch supplies device memory and the current CUDA stream; every step
of the transform runs in the library's kernels.  There is no CPU fallback: if the library is
missing or no GPU is present, the calls raise.

    plan = Plan(N=(256, 256, 256), M=10**7, m=6, sigma=2.0, window="kb")
    plan.set_points(x)          # x: cuda float64 [M, 3], coordinates in [-0.5, 0.5]
    fhat = plan.adjoint(f)      # f: cuda complex128 [M]  ->  complex128 [N0, N1, N2]

fhat[k0 + N0/2, k1 + N1/2, k2 + N2/2] = sum_j f_j exp(-2 pi i k.x_j)   (Eq. 5)
up to the NFFT approximation error (E2 ~ 1e-11 at m = 6, sigma = 2, Kaiser-Bessel).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPNFFT_LIB", os.path.join(_HERE, "libhpnfft.so"))

WINDOWS = {"kb": 0, "kaiser_bessel": 0, "gaussian": 1, "gauss": 1, "b_spline": 2, "bspline": 2,
           "sinc_power": 3, "sinc": 3}
SPREAD_METHODS = {"auto": 0, "atomic": 1, "sweep": 2}
STAGES = ("keys", "scan", "scatter", "spread", "fft_z", "fft_y", "fft_x_deconv", "records", "exchange", "alltoall",
          "inv_fft", "interp")
DIST_MODES = {"allreduce": 0, "reduce": 1, "reduce_scatter": 2, "grid_slab": 3}

HPNFFT_OK = 0
_ERRORS = {
    -1: ValueError,
    -2: NotImplementedError,
    -3: ValueError,
    -4: MemoryError,
    -5: RuntimeError,
    -6: RuntimeError,
    -7: RuntimeError,
    -8: ValueError,
}
_ERROR_NAMES = {-1: "E_INVALID", -2: "E_UNSUPPORTED", -3: "E_RANGE", -4: "E_NOMEM", -5: "E_CUDA",
                -6: "E_NCCL", -7: "E_STATE", -8: "E_DEGENERATE_WINDOW"}

_lib = None


class HpnfftError(RuntimeError):
    pass


def load_library(path: str = LIB_PATH):
    """Load libhpnfft.so and declare the C signatures (raises if the library is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    vp, i64, i64p, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p
    lib.hpnfft_plan.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, i64, ctypes.c_int, ctypes.c_double,
                                ctypes.c_int, vp]
    lib.hpnfft_plan.restype = ctypes.c_int
    lib.hpnfft_set_points_async.argtypes = [vp, dp]
    lib.hpnfft_set_points_async.restype = ctypes.c_int
    lib.hpnfft_check_points.argtypes = [vp]
    lib.hpnfft_check_points.restype = ctypes.c_int
    lib.hpnfft_set_points.argtypes = [vp, dp]
    lib.hpnfft_set_points.restype = ctypes.c_int
    lib.hpnfft_adjoint.argtypes = [vp, dp, dp]
    lib.hpnfft_adjoint.restype = ctypes.c_int
    lib.hpnfft_destroy.argtypes = [vp]
    lib.hpnfft_destroy.restype = ctypes.c_int
    lib.hpnfft_last_error.argtypes = []
    lib.hpnfft_last_error.restype = ctypes.c_char_p
    lib.hpnfft_workspace_bytes.argtypes = [vp]
    lib.hpnfft_workspace_bytes.restype = ctypes.c_size_t
    lib.hpnfft_set_stream.argtypes = [vp, vp]
    lib.hpnfft_set_stream.restype = ctypes.c_int
    lib.hpnfft_set_spread_method.argtypes = [vp, ctypes.c_int]
    lib.hpnfft_set_spread_method.restype = ctypes.c_int
    lib.hpnfft_launch_count.argtypes = [vp]
    lib.hpnfft_launch_count.restype = ctypes.c_int64
    lib.hpnfft_enable_timing.argtypes = [vp, ctypes.c_int]
    lib.hpnfft_enable_timing.restype = ctypes.c_int
    lib.hpnfft_stage_times.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    lib.hpnfft_stage_times.restype = ctypes.c_int
    lib.hpnfft_version.argtypes = []
    lib.hpnfft_version.restype = ctypes.c_char_p
    lib.hpnfft_inverse.argtypes = [vp, dp, dp]
    lib.hpnfft_inverse.restype = ctypes.c_int
    lib.hpnfft_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.hpnfft_get_unique_id.restype = ctypes.c_int
    lib.hpnfft_plan_dist.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, i64, ctypes.c_int, ctypes.c_double,
                                     ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
    lib.hpnfft_plan_dist.restype = ctypes.c_int
    lib.hpnfft_ewald_reciprocal.argtypes = [vp, dp, ctypes.c_double, ctypes.c_double, dp]
    lib.hpnfft_ewald_reciprocal.restype = ctypes.c_int
    lib.hpnfft_set_slabs.argtypes = [vp, i64p]
    lib.hpnfft_set_slabs.restype = ctypes.c_int
    lib.hpnfft_plan_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, i64p, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_int, vp, ctypes.c_int, ctypes.c_int]
    lib.hpnfft_plan_group.restype = ctypes.c_int
    lib.hpnfft_adjoint_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    lib.hpnfft_adjoint_group.restype = ctypes.c_int
    lib.hpnfft_plan_f32.argtypes = lib.hpnfft_plan.argtypes
    lib.hpnfft_plan_f32.restype = ctypes.c_int
    lib.hpnfft_set_points_f32.argtypes = [vp, dp]
    lib.hpnfft_set_points_f32.restype = ctypes.c_int
    lib.hpnfft_adjoint_f32.argtypes = [vp, dp, dp]
    lib.hpnfft_adjoint_f32.restype = ctypes.c_int
    lib.hpnfft_plan_info.argtypes = [vp, i64p, ctypes.c_int]
    lib.hpnfft_plan_info.restype = ctypes.c_int
    lib.hpnfft_output_shape.argtypes = [vp, i64p]
    lib.hpnfft_output_shape.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int):
    if rc != HPNFFT_OK:
        msg = load_library().hpnfft_last_error().decode()
        exc = _ERRORS.get(rc, HpnfftError)
        raise exc(f"hpnfft {_ERROR_NAMES.get(rc, rc)}: {msg}")


def _stream_ptr(stream):
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def get_unique_id() -> bytes:
    """128-byte NCCL unique id for hpnfft_plan_dist (create on one rank, share with all)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().hpnfft_get_unique_id(buf))
    return buf.raw


class Plan:
    """One adjoint NFFT plan (hpnfft_plan): fixed N, M, m, sigma and window.

    dist=(nranks, rank, unique_id, mode) makes it rank `rank` of a multi-GPU plan
    (hpnfft_plan_dist; mode one of DIST_MODES or its integer); M is then this rank's point count
    and adjoint() returns this rank's block of fhat (out_shape).
    """

    def __init__(self, N, M: int, m: int = 6, sigma: float = 2.0, window="kb", stream=None, device=None, dist=None,
                 _handle=None, precision: str = "f64"):
        import torch

        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("hpnfft needs a CUDA device (there is no CPU path)")
        self.N = tuple(int(v) for v in N)
        self.M = int(M)
        self.m = int(m)
        self.sigma = float(sigma)
        self.window = WINDOWS[window] if isinstance(window, str) else int(window)
        if precision not in ("f64", "f32"):
            raise ValueError("precision must be 'f64' or 'f32'")
        self.precision = precision   # f32: hpnfft_plan_f32 (float x, complex64 f and fhat; NEXT #4)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._stream = stream
        arr = (ctypes.c_int64 * len(self.N))(*self.N)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            if _handle is not None:   # a member of a PlanGroup (created by hpnfft_plan_group)
                h = ctypes.c_void_p(_handle)
            elif dist is None:
                fn = lib.hpnfft_plan_f32 if precision == "f32" else lib.hpnfft_plan
                _check(fn(ctypes.byref(h), len(self.N), arr, self.M, self.m, self.sigma, self.window, _stream_ptr(stream)))
            else:
                nranks, rank, uid, mode = dist
                mode = DIST_MODES[mode] if isinstance(mode, str) else int(mode)
                if len(uid) != 128:
                    raise ValueError("unique id must be 128 bytes")
                _check(lib.hpnfft_plan_dist(ctypes.byref(h), len(self.N), arr, self.M, self.m, self.sigma,
                                            self.window, _stream_ptr(stream), int(nranks), int(rank), uid, mode))
        self._h = h
        shp = (ctypes.c_int64 * 3)()
        _check(lib.hpnfft_output_shape(h, shp))
        self.out_shape = tuple(int(v) for v in shp)[3 - len(self.N):]   # d < 3: drop the trivial leading 1s

    def ewald_reciprocal(self, q, L: float, alpha: float, out=None):
        """hpnfft_ewald_reciprocal: Eq. 12's reciprocal-space energy of the real charges q
        (CUDA float64 [M]) at the points of the last set_points (x = r / L - 1/2).  Returns a
        CUDA float64 tensor of one element (stream-ordered; .item() synchronises)."""
        import torch

        if not (q.is_cuda and q.dtype == torch.float64 and q.numel() == self.M):
            raise TypeError("q must be a CUDA float64 tensor with M elements")
        q = q.contiguous()
        if out is None:
            out = torch.empty((1,), dtype=torch.float64, device=q.device)
        self._sync_stream()
        _check(load_library().hpnfft_ewald_reciprocal(self._h, ctypes.c_void_p(q.data_ptr()), float(L), float(alpha),
                                                      ctypes.c_void_p(out.data_ptr())))
        return out

    def set_slabs(self, edges):
        """hpnfft_set_slabs: grid_slab plans only; `edges` = nranks + 1 cyclic x-ordered cell
        planes (e.g. dist.grid_slab_edges); every rank passes the same edges, then set_points."""
        arr = (ctypes.c_int64 * len(edges))(*[int(e) for e in edges])
        _check(load_library().hpnfft_set_slabs(self._h, arr))

    # -- stream plumbing: every call runs on the caller's current torch stream (or the fixed one)
    def _sync_stream(self):
        _check(load_library().hpnfft_set_stream(self._h, _stream_ptr(self._stream)))

    def set_points(self, x, sync: bool = True):
        """hpnfft_set_points; sync=False: hpnfft_set_points_async (no host wait, all grid planes,
        a range error is raised by the next set_points / check_points)."""
        import torch

        d = len(self.N)
        xt = torch.float32 if self.precision == "f32" else torch.float64
        if not (x.is_cuda and x.dtype == xt and x.dim() == 2 and x.shape[1] == d):
            raise TypeError(f"x must be a CUDA {xt} tensor of shape [M, {d}]")
        if x.shape[0] != self.M:
            raise ValueError(f"x has {x.shape[0]} points, the plan was built for M = {self.M}")
        x = x.contiguous()
        self._sync_stream()
        if self.precision == "f32":
            _check(load_library().hpnfft_set_points_f32(self._h, ctypes.c_void_p(x.data_ptr())))
            return
        fn = load_library().hpnfft_set_points if sync else load_library().hpnfft_set_points_async
        _check(fn(self._h, ctypes.c_void_p(x.data_ptr())))

    def check_points(self):
        """hpnfft_check_points: raise the deferred error of the last set_points(sync=False)."""
        _check(load_library().hpnfft_check_points(self._h))

    def adjoint(self, f, out=None):
        import torch

        ct = torch.complex64 if self.precision == "f32" else torch.complex128
        if not (f.is_cuda and f.dtype == ct and f.numel() == self.M):
            raise TypeError(f"f must be a CUDA {ct} tensor with M elements")
        f = f.contiguous()
        if out is None:
            out = torch.empty(self.out_shape, dtype=ct, device=f.device)
        elif not (out.is_cuda and out.dtype == ct and tuple(out.shape) == self.out_shape and out.is_contiguous()):
            raise TypeError(f"out must be a contiguous CUDA {ct} tensor of shape {self.out_shape}")
        self._sync_stream()
        fn = load_library().hpnfft_adjoint_f32 if self.precision == "f32" else load_library().hpnfft_adjoint
        _check(fn(self._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(out.data_ptr())))
        return out

    def inverse(self, fhat, out=None):
        """Eq. 6 (hpnfft_inverse): f(x_j) = sum_k fhat(k) exp(+2 pi i k.x_j) for the points of the
        last set_points, in their original order.  fhat: CUDA complex128 of shape N."""
        import torch

        if not (fhat.is_cuda and fhat.dtype == torch.complex128 and tuple(fhat.shape) == self.N):
            raise TypeError(f"fhat must be a CUDA complex128 tensor of shape {self.N}")
        fhat = fhat.contiguous()
        if out is None:
            out = torch.empty((self.M,), dtype=torch.complex128, device=fhat.device)
        elif not (out.is_cuda and out.dtype == torch.complex128 and out.numel() == self.M and out.is_contiguous()):
            raise TypeError("out must be a contiguous CUDA complex128 tensor with M elements")
        self._sync_stream()
        _check(load_library().hpnfft_inverse(self._h, ctypes.c_void_p(fhat.data_ptr()), ctypes.c_void_p(out.data_ptr())))
        return out

    def __call__(self, x, f):
        self.set_points(x)
        return self.adjoint(f)

    def transform_host(self, x_host, f_host, out_host=None):
        """End-to-end call with HOST inputs/outputs (pinned torch CPU tensors): H2D copy of x and
        f, set_points + adjoint, D2H copy of fhat, all on the current stream."""
        import torch

        x = x_host.to(self.device, non_blocking=True)
        f = f_host.to(self.device, non_blocking=True)
        self.set_points(x)
        fh = self.adjoint(f)
        if out_host is None:
            out_host = torch.empty(self.out_shape, dtype=torch.complex128, pin_memory=True)
        out_host.copy_(fh, non_blocking=True)
        return out_host

    def set_spread_method(self, method):
        m = SPREAD_METHODS[method] if isinstance(method, str) else int(method)
        _check(load_library().hpnfft_set_spread_method(self._h, m))

    @property
    def workspace_bytes(self) -> int:
        return int(load_library().hpnfft_workspace_bytes(self._h))

    EXCHANGE_PATHS = ("none", "nccl_collective", "grid_slab_nvlink_p2p", "grid_slab_nccl_sendrecv", "one_gpu_group")

    def info(self) -> dict:
        """hpnfft_plan_info: algorithmic FFT-pass bytes of the current geometry, exchange path, ..."""
        buf = (ctypes.c_int64 * 8)()
        w = load_library().hpnfft_plan_info(self._h, buf, 8)
        if w < 0:
            _check(w)
        v = [int(buf[i]) for i in range(w)]
        return {"pass_bytes": {"fft_z": v[0], "fft_y": v[1], "fft_x_deconv": v[2]},
                "exchange_path": self.EXCHANGE_PATHS[v[3]], "planes": v[4], "record_group": v[5],
                "spread_kernel": {1: "atomic", 2: "sweep"}[v[6]], "workspace_bytes": v[7]}

    def launch_count(self) -> int:
        return int(load_library().hpnfft_launch_count(self._h))

    def enable_timing(self, on: bool = True):
        _check(load_library().hpnfft_enable_timing(self._h, 1 if on else 0))

    def stage_times(self) -> dict:
        buf = (ctypes.c_float * len(STAGES))()
        w = load_library().hpnfft_stage_times(self._h, buf, len(STAGES))
        if w < 0:
            _check(w)
        return {STAGES[i]: float(buf[i]) for i in range(w)}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load_library().hpnfft_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PlanGroup:
    """hpnfft_plan_group: the `nranks` ranks of a multi-GPU plan (mode as DIST_MODES) emulated as
    plans on ONE GPU, for validating the exchange code with fewer GPUs than ranks.  members[r]
    is a Plan (set_slabs, set_points, out_shape as rank r); adjoint(fs) runs every exchange phase
    for all members before the next (hpnfft_adjoint_group) and returns the members' output
    blocks.  Ms: the members' point counts."""

    def __init__(self, N, Ms, m: int = 6, sigma: float = 2.0, window="kb", mode="grid_slab", device=None):
        import torch

        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("hpnfft needs a CUDA device (there is no CPU path)")
        self.N = tuple(int(v) for v in N)
        self.P = len(Ms)
        self.mode = DIST_MODES[mode] if isinstance(mode, str) else int(mode)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        win = WINDOWS[window] if isinstance(window, str) else int(window)
        arr = (ctypes.c_int64 * len(self.N))(*self.N)
        marr = (ctypes.c_int64 * self.P)(*[int(v) for v in Ms])
        hs = (ctypes.c_void_p * self.P)()
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream(self.device)
            _check(lib.hpnfft_plan_group(hs, len(self.N), arr, marr, int(m), float(sigma), win,
                                         ctypes.c_void_p(self.stream.cuda_stream), self.P, self.mode))
        self.members = [Plan(self.N, int(Ms[r]), m=m, sigma=sigma, window=window, stream=self.stream,
                             device=self.device, _handle=hs[r]) for r in range(self.P)]

    def set_slabs(self, edges):
        for p in self.members:
            p.set_slabs(edges)

    def set_points(self, xs):
        for p, x in zip(self.members, xs):
            p.set_points(x)

    def adjoint(self, fs):
        import torch

        outs, fp, op, hs = [], (ctypes.c_void_p * self.P)(), (ctypes.c_void_p * self.P)(), (ctypes.c_void_p * self.P)()
        keep = []
        for r, (p, f) in enumerate(zip(self.members, fs)):
            if not (f.is_cuda and f.dtype == torch.complex128 and f.numel() == p.M):
                raise TypeError("f must be a CUDA complex128 tensor with M elements")
            f = f.contiguous()
            keep.append(f)
            o = torch.empty(p.out_shape, dtype=torch.complex128, device=self.device)
            outs.append(o)
            fp[r], op[r], hs[r] = f.data_ptr(), o.data_ptr(), p._h.value
        with torch.cuda.stream(self.stream):
            _check(load_library().hpnfft_adjoint_group(hs, self.P, fp, op))
        return outs

    def close(self):
        for p in self.members:
            p.close()


class HostPipeline:
    """Streamed end-to-end transforms from and to pinned HOST memory.

    submit(x_host, f_host, out_host) enqueues one transform: the H2D copies of x and f on a copy
    stream, set_points + adjoint on the compute stream, the D2H copy of fhat on a second copy
    stream, with `depth` (default two) device buffer sets so that the copies of one transform
    overlap the kernels of its neighbours (PCIe in both directions and the GPU busy at once).
    out_host is complete after flush() (or after the next-but-one submit).  Every submitted
    transform still moves all of its own inputs and its result across PCIe.
    """

    def __init__(self, plan: "Plan", M: int, depth: int = 2):
        import torch

        self.plan = plan
        dev = plan.device
        self.depth = depth
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        self.compute = torch.cuda.current_stream(dev)
        self.x = [torch.empty((M, 3), dtype=torch.float64, device=dev) for _ in range(depth)]
        self.f = [torch.empty((M,), dtype=torch.complex128, device=dev) for _ in range(depth)]
        self.o = [torch.empty(plan.out_shape, dtype=torch.complex128, device=dev) for _ in range(depth)]
        self.in_ready = [torch.cuda.Event() for _ in range(depth)]
        self.used = [None] * depth      # compute finished reading buffer set s
        self.drained = [None] * depth   # D2H finished reading output buffer s
        self.pending = None             # D2H of the previous transform, enqueued after the next H2D
        self.i = 0

    def _drain_pending(self):
        # enqueued after the next transform's H2D: a D2H that waits for its kernels must not sit
        # in front of that H2D in a shared hardware queue
        import torch

        if self.pending is None:
            return
        s, out_host, done = self.pending
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(done)
            out_host.copy_(self.o[s], non_blocking=True)
            drained = torch.cuda.Event()
            drained.record(self.d2h)
        self.drained[s] = drained
        self.pending = None

    def submit(self, x_host, f_host, out_host):
        import torch

        s = self.i % self.depth
        with torch.cuda.stream(self.h2d):
            if self.used[s] is not None:
                self.h2d.wait_event(self.used[s])
            self.x[s].copy_(x_host, non_blocking=True)
            self.in_ready[s].record(self.h2d)
            self.f[s].copy_(f_host, non_blocking=True)
            f_ready = torch.cuda.Event()
            f_ready.record(self.h2d)
        self._drain_pending()
        self.compute.wait_event(self.in_ready[s])
        if self.drained[s] is not None:
            self.compute.wait_event(self.drained[s])
        with torch.cuda.stream(self.compute):
            # needs x only (f is still copying); no host wait: the host stays a transform ahead,
            # a range error surfaces at the next submit or at flush
            self.plan.set_points(self.x[s], sync=False)
            self.compute.wait_event(f_ready)
            self.plan.adjoint(self.f[s], out=self.o[s])
            done = torch.cuda.Event()
            done.record(self.compute)
        self.used[s] = done
        self.pending = (s, out_host, done)
        self.i += 1
        return out_host

    def flush(self):
        self._drain_pending()
        self.h2d.synchronize()
        self.compute.synchronize()
        self.d2h.synchronize()
        self.plan.check_points()


def version() -> str:
    return load_library().hpnfft_version().decode()
