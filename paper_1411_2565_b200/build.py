"""Build libgrace.so in-tree with nvcc for sm_100a (called by __graft_entry__.build()).

tensor_setup.cu is compiled with -fmad=false (bit-exact fp64 tensor, DESIGN.md
reading Q8); the per-step kernels keep FMA contraction.  No fast-math anywhere.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.environ.get("GRACE_LIB_OUT") or os.path.join(HERE, "libgrace.so")  # GRACE_LIB_OUT: sweep variants
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
COMMON += os.environ.get("GRACE_NVCC_FLAGS", "").split()  # tuning experiments only
UNITS = {
    "grace_api.cu": [],
    # --split-compile halves the build time but measured slower code (K3 1.08 -> 1.21 ms): dev only
    "step_kernels.cu": (["--split-compile=0"] if os.environ.get("GRACE_SPLIT_COMPILE") else [])
    + (["-Xptxas", "-v"] if os.environ.get("GRACE_PTXAS_V") else []),
    "tensor_setup.cu": ["-fmad=false"],
    "small_step.cu": [],
}
HEADERS = ["fft_engine.cuh", "internal.h", "pencil.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(force=False, verbose=False):
    deps = [os.path.join(CSRC, f) for f in list(UNITS) + HEADERS] + [os.path.join(ROOT, "include", "grace.h")]
    newest = max(_mtime(p) for p in deps)
    if not force and _mtime(LIB) > newest:
        return LIB
    objs = []
    procs = []
    for src, extra in UNITS.items():
        obj = os.path.join(CSRC, src.replace(".cu", "") + "_" + os.path.basename(LIB).replace(".so", ".o"))
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs]
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
