"""Per-kernel times (libgrace profiling mode) and graph-mode ms/step for a workload
or a Table-1 cube.   python scripts/kernel_split.py [slab_1024x1024x32 | cube:128 ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1411_2565_b200 as pb  # noqa: E402
from workloads import WORKLOADS, random_m, table1_cube  # noqa: E402


def run(spec, steps=40):
    w = table1_cube(int(spec.split(":")[1])) if spec.startswith("cube:") else WORKLOADS[spec]
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0)
    s = torch.cuda.Stream()
    pb.grace_set_stream(g.h, s.cuda_stream)
    g.set_m(random_m(w.n, w.Ms))
    g.set_hext(w.hext)
    g.step(8, w.dt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    g.step(steps, w.dt)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    pb.grace_set_profiling(g.h, True)
    g.step(2, w.dt)
    pb.grace_kernel_times(g.h, reset=True)
    g.step(steps, w.dt)
    torch.cuda.synchronize()
    kms, kl = pb.grace_kernel_times(g.h, reset=True)
    geo = g.geometry
    g.close()
    per = " ".join(f"{t / max(n, 1):.4f}" for t, n in zip(kms, kl))
    print(f"{spec:22s} n={list(w.n)} P={[geo['Px'], geo['Py'], geo['Pz']]} graph {ms:.4f} ms/step "
          f"{w.n[0] * w.n[1] * w.n[2] / ms / 1e6:.2f} Gcell/s | kernels ms: {per}", flush=True)


for spec in (sys.argv[1:] or ["slab_1024x1024x32"]):
    run(spec)
