"""Build inputs/libhpnfft_inputs.so (device twin of the seeded generator; not product code)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libhpnfft_inputs.so")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "gen.cu")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-o", LIB, src])
    return LIB
