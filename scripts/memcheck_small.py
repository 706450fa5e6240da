"""A few steps of the film (BASELINE config 3) and of small cubes, for
compute-sanitizer memcheck runs (K3 / K2' KS-slice reads at the row
end).  Usage: compute-sanitizer --tool memcheck python scripts/memcheck_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1411_2565_b200 as pb  # noqa: E402
from workloads import GAMMA0, WORKLOADS, random_m  # noqa: E402

cases = [WORKLOADS["film_512x512x8"], WORKLOADS["sp4_field1"]]
for w in cases:
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    g.set_m(random_m(w.n, w.Ms))
    g.step(3, w.dt)
    g.heff()
    g.close()
    print("ok", w.name, flush=True)
for N in (4, 8, 16):
    n = (N, N, N)
    g = pb.Grace(n, (1e-9,) * 3, 1e6, 1e-11, 6.28e4, 0.5, GAMMA0)
    g.set_m(random_m(n, 1e6))
    g.step(3, 1e-15)
    g.heff()
    g.close()
    print("ok cube", N, flush=True)
