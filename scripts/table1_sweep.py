"""Paper Table 1 workload sweep and small-grid latency.

The paper's only numeric result is Table 1: per-step time of an
N x N x N cube (A = 1e-11 J/m, Ms = 1e6 A/m, H_anis = 1e5 A/m, Euler) for
N = 8..128 on an AMD HD 7970 (Grace, C++ AMP) and OOMMF on an i7-930.  This
script times the same workload through libgrace on one B200 (CUDA-graph step
loop, steps timed with CUDA events after warm-up) and, for small N, the fp64
oracle on this host, and prints one JSON object plus a markdown table.  Also
times the SP4 grids (BASELINE configs 1-2), whose steps are launch-bound.

python scripts/table1_sweep.py [--out profiles/r02_table1] [--oracle-max 128]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import WORKLOADS, random_m, table1_cube  # noqa: E402

PAPER = {  # P:L74-78, ms per step: (CPU OOMMF i7-930, GPU Grace HD 7970)
    8: (0.8492, 1.95), 16: (4.066, 2.723), 32: (36.14, 3.151), 64: (489.6, 6.558), 128: (4487.0, 26.34)}


def gpu_ms_per_step(w, steps):
    import torch

    import paper_1411_2565_b200 as pb

    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0)
    s = torch.cuda.Stream()
    pb.grace_set_stream(g.h, s.cuda_stream)
    g.set_m(random_m(w.n, w.Ms))
    g.set_hext(w.hext)
    g.step(32, w.dt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    g.step(steps, w.dt)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    g.close()
    return ms


def oracle_ms_per_step(w, steps=3):
    """fp64 oracle on this host: (single-thread ms/step, all-core ms/step, setup s).
    Single thread: numpy.fft; all cores: scipy.fft workers = affinity size
    (BASELINE.md Sec. 4); setup = tensor octant + kernel spectrum, once."""
    from oracle.demag import DemagFFT
    from oracle.llg import Sim
    from oracle.tensor import tensor_octant

    ncores = len(os.sched_getaffinity(0))
    t = time.perf_counter()
    oct_ = tensor_octant(*w.n, *w.d)
    op = DemagFFT(oct_)
    setup = time.perf_counter() - t
    res = []
    for o in (op, DemagFFT(oct_, workers=ncores)):
        sim = Sim(random_m(w.n, w.Ms), o, w.Ms, w.A, w.Ku, w.alpha, w.gamma0, w.d)
        sim.euler_step(w.dt)
        t = time.perf_counter()
        sim.run(steps, w.dt)
        res.append((time.perf_counter() - t) / steps * 1e3)
    return res[0], res[1], setup


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--oracle-max", type=int, default=128)
    args = ap.parse_args()
    rows = []
    for N in (8, 16, 32, 64, 128, 256, 512):
        w = table1_cube(N)
        steps = 2000 if N <= 64 else (400 if N <= 128 else 50)
        gms = gpu_ms_per_step(w, steps)
        oms, omk, osetup = oracle_ms_per_step(w) if N <= args.oracle_max else (None, None, None)
        cpu_p, gpu_p = PAPER.get(N, (None, None))
        rows.append({"N": N, "cells": N ** 3, "b200_ms": gms, "b200_Mcell_s": N ** 3 / gms / 1e3,
                     "oracle_ms_this_host": oms, "oracle_ms_all_cores": omk, "oracle_setup_s": osetup,
                     "paper_hd7970_ms": gpu_p, "paper_oommf_i7_ms": cpu_p})
    sp4 = []
    for name in ("sp4_field1", "sp4_field2_refined"):
        w = WORKLOADS[name]
        gms = gpu_ms_per_step(w, 20000)
        sp4.append({"workload": name, "grid": list(w.n), "b200_us_per_step": gms * 1e3,
                    "ns_simulated_per_s": w.dt * 1e9 / (gms * 1e-3)})
    out = {"table1": rows, "sp4": sp4, "note": "B200 numbers: CUDA events around grace_step(K) after 32 warm-up "
           "steps (graph replay); paper numbers are other hardware (HD 7970 / OOMMF on i7-930), context only"}
    ncores = len(os.sched_getaffinity(0))
    lines = ["| N | cells | B200 ms/step | B200 Mcell-updates/s | fp64 oracle ms/step, 1 thread | "
             f"fp64 oracle ms/step, {ncores} threads | oracle setup s | B200 speed-up vs oracle (1 thr / all) | "
             "paper HD 7970 ms | paper OOMMF i7-930 ms | paper GPU/CPU |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        f = lambda v: "-" if v is None else f"{v:.4g}"  # noqa: E731
        sp = "-" if r["oracle_ms_this_host"] is None else \
            f"{r['oracle_ms_this_host'] / r['b200_ms']:.0f} / {r['oracle_ms_all_cores'] / r['b200_ms']:.0f}"
        pr = "-" if r["paper_hd7970_ms"] is None else f"{r['paper_oommf_i7_ms'] / r['paper_hd7970_ms']:.3g}"
        lines.append(f"| {r['N']} | {r['cells']} | {r['b200_ms']:.4f} | {r['b200_Mcell_s']:.1f} | "
                     f"{f(r['oracle_ms_this_host'])} | {f(r['oracle_ms_all_cores'])} | {f(r['oracle_setup_s'])} | {sp} | "
                     f"{f(r['paper_hd7970_ms'])} | {f(r['paper_oommf_i7_ms'])} | {pr} |")
    lines += ["", "| SP4 workload | grid | B200 us/step | simulated ns per wall-clock s |", "|---|---|---|---|"]
    for r in sp4:
        lines.append(f"| {r['workload']} | {r['grid']} | {r['b200_us_per_step']:.2f} | {r['ns_simulated_per_s']:.3f} |")
    print(json.dumps(out))
    print("\n".join(lines))
    if args.out:
        json.dump(out, open(args.out + ".json", "w"), indent=1)
        open(args.out + ".md", "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
