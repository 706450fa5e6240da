"""Per-kernel event times (libgrace profiling mode) and graph step time for small Table-1 cubes.

python scripts/small_cube_kernels.py [N ...]   (GPU; prints one line per N)
"""
import sys
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1411_2565_b200 as pb  # noqa: E402
from workloads import GAMMA0, random_m, table1_cube  # noqa: E402

for N in [int(a) for a in sys.argv[1:]] or [8, 16, 32, 64]:
    w = table1_cube(N)
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    g.set_m(random_m(w.n, w.Ms))
    g.step(50, w.dt)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    g.step(500, w.dt)
    e.record()
    torch.cuda.synchronize()
    graph_us = s.elapsed_time(e) / 500 * 1e3
    pb.grace_set_profiling(g.h, 1)
    g.step(20, w.dt)
    pb.grace_kernel_times(g.h, reset=True)
    g.step(200, w.dt)
    ms, ln = pb.grace_kernel_times(g.h)
    per = " ".join(f"{m / max(l, 1) * 1e3:.1f}" for m, l in zip(ms, ln))
    print(f"N={N} graph {graph_us:.1f} us/step; per-kernel us (profiling mode, K1..): {per}", flush=True)
    g.close()
