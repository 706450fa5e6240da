"""Build baseline_cufft/libcufftbase.so (the cuFFT comparison pipeline, not part of libgrace).

Links cuFFT and libgrace (for the fp64 tensor octant of the setup only).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PKG = os.path.join(ROOT, "paper_1411_2565_b200")
LIB = os.path.join(HERE, "libcufftbase.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    src = os.path.join(HERE, "cufft_step.cu")
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) > os.path.getmtime(src):
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
           "-fPIC", "-shared", src, "-o", LIB, "-L", PKG, "-lgrace", "-L/usr/local/cuda/lib64", "-lcufft",
           "-Xlinker", "-rpath,$ORIGIN/../paper_1411_2565_b200", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
