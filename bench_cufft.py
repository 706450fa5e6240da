"""cuFFT comparison baseline beside the hand-written path (BASELINE.json north_star:
"cuFFT is timed only as a comparison baseline").

    python bench_cufft.py [--workload slab_1024x1024x32] [--steps K] [--warmup W]

Runs, on the same GPU and the same synthetic input (workloads.random_m), the
naive library pipeline of baseline_cufft/cufft_step.cu (pad, cufftExecR2C x3, full
complex k-space multiply, cufftExecC2R x3, unpad + the same LLG/Euler arithmetic)
and libgrace's graph-replayed step, each timed with CUDA events around K steps
after W warm-up steps.  Prints one JSON line with both ms/step, the ratio, the
algorithmic bytes per cell of each pipeline and their relative difference after
K steps (the two compute the same method in fp32: a sanity check, the parity
test is tests/test_gpu_cufft_baseline.py).  cuFFT never enters libgrace.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import WORKLOADS, random_m  # noqa: E402


def load_baseline():
    import paper_1411_2565_b200 as pb

    pb.load()  # libgrace first (the baseline takes its fp64 tensor octant for the setup)
    from baseline_cufft.build import LIB, build

    if not os.path.exists(LIB):
        build()
    lib = ctypes.CDLL(LIB)
    D, I, P = ctypes.c_double, ctypes.c_int, ctypes.c_void_p
    lib.cufft_baseline_run.restype = I
    lib.cufft_baseline_run.argtypes = [I, I, I, D, D, D, D, D, D, D, D, P, D, P, I, I, P, P, P, ctypes.c_char_p]
    return lib


def cufft_run(w, M0, steps, warmup, want_m=True, want_hd=False):
    """(ms/step, final M [3,nz,ny,nx] f32 or None, H_demag of M0 or None)."""
    lib = load_baseline()
    m0 = np.ascontiguousarray(M0, dtype=np.float32)
    hext = np.ascontiguousarray(w.hext, dtype=np.float64)
    ms = ctypes.c_double(0.0)
    mout = np.empty_like(m0) if want_m else None
    hd = np.empty_like(m0) if want_hd else None
    err = ctypes.create_string_buffer(256)
    rc = lib.cufft_baseline_run(*w.n, *w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0, hext.ctypes.data, w.dt,
                                m0.ctypes.data, warmup, steps, ctypes.byref(ms),
                                mout.ctypes.data if want_m else None, hd.ctypes.data if want_hd else None, err)
    if rc != 0:
        raise RuntimeError(f"cufft_baseline_run: {rc} {err.value.decode()}")
    return ms.value, mout, hd


def naive_bytes_per_cell(w):
    """Compulsory bytes of the library pipeline per cell per step (fp32): pad (read M
    12 B/cell, write 3 padded reals), R2C (read 3 padded reals, write 3 half spectra),
    multiply (read 3 + 6, write 3 half spectra), C2R (read 3 half spectra, write 3
    padded reals), LLG (read 3 padded reals at the cells + M 12, write M 12).  cuFFT's
    own multi-pass traffic for large transforms comes on top."""
    nx, ny, nz = w.n
    pad = lambda n: 1 if n == 1 else 1 << (2 * n - 2).bit_length()  # noqa: E731
    P = pad(nx) * pad(ny) * pad(nz)
    Ph = (pad(nx) // 2 + 1) * pad(ny) * pad(nz)
    N = nx * ny * nz
    b = (12 * N + 12 * P) + (12 * P + 24 * Ph) + (24 * Ph + 48 * Ph + 24 * Ph) + (24 * Ph + 12 * P) + (12 * N + 24 * N)
    return b / N


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="slab_1024x1024x32", choices=sorted(WORKLOADS))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    import torch

    import paper_1411_2565_b200 as pb

    M0 = random_m(w.n, w.Ms)
    ms_cufft, Mc, _ = cufft_run(w, M0, args.steps, args.warmup)
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0)
    stream = torch.cuda.Stream()
    pb.grace_set_stream(g.h, stream.cuda_stream)
    g.set_m(M0.astype(np.float32).astype(np.float64))
    g.set_hext(w.hext)
    g.step(args.warmup, w.dt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    g.step(args.steps, w.dt)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_grace = e0.elapsed_time(e1) / args.steps
    Mg = g.get_m()
    geo = g.geometry
    g.close()
    from bench import design_step_bytes

    N = w.cells
    rel = float(np.linalg.norm(Mg - Mc) / np.linalg.norm(Mg))
    out = {"workload": w.name, "steps": args.steps, "warmup": args.warmup,
           "cufft_ms_per_step": ms_cufft, "grace_ms_per_step": ms_grace, "speedup": ms_cufft / ms_grace,
           "cufft_cell_updates_per_s": N / (ms_cufft / 1e3), "grace_cell_updates_per_s": N / (ms_grace / 1e3),
           "bytes_per_cell": {"cufft_pipeline_compulsory": naive_bytes_per_cell(w),
                              "grace_design": design_step_bytes(geo) / N},
           "rel_diff_after_steps": rel,
           "note": "both timed with CUDA events around K steps after W warm-up; cuFFT pipeline in "
                   "baseline_cufft/cufft_step.cu (not part of libgrace)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
