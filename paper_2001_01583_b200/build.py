"""Build libhpnfft.so (sm_100a) in-tree with nvcc.  Product build; no oracle code involved."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhpnfft.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "hpnfft.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile every csrc/*.cu for sm_100a and link libhpnfft.so (or `out`, with extra -D flags,
    for measurement variants)."""
    lib = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    objdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    logs = []
    ok = True
    for src, pr in procs:
        out, _ = pr.communicate()
        logs.append(f"== {os.path.basename(src)}\n{out}")
        if pr.returncode != 0:
            ok = False
    log = "\n".join(logs)
    with open(os.path.join(objdir, "ptxas.log"), "w") as fh:
        fh.write(log)
    if not ok:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed")
    if verbose:
        print(log)
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-ldl"])
    return lib


CHECKED_LIB = os.path.join(HERE, "libhpnfft_checked.so")


def build_checked(force: bool = False) -> str:
    """libhpnfft_checked.so: the same sources with HPNFFT_CHECKED=1 (device-side bounds/protocol
    assertions and mbarrier deadlock timeouts; tests/test_gpu_parity.py runs the small cases of
    tools/sanitize_case.py on it, as compute-sanitizer is closed on the GPU pool)."""
    if not force and os.path.exists(CHECKED_LIB) and os.path.getmtime(CHECKED_LIB) >= max(
            os.path.getmtime(d) for d in deps()):
        return CHECKED_LIB
    return build(force=True, defines=("HPNFFT_CHECKED=1",), out=CHECKED_LIB)


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, out=outs[0] if outs else None))
