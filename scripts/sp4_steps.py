"""Run n graph-replayed Euler steps of an SP4 workload (for ncu launch lists).

    python scripts/sp4_steps.py [n] [workload | cube:N]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1411_2565_b200 as pb  # noqa: E402
from workloads import GAMMA0, WORKLOADS, random_m, table1_cube  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
name = sys.argv[2] if len(sys.argv) > 2 else "sp4_field1"
w = table1_cube(int(name[5:])) if name.startswith("cube:") else WORKLOADS[name]
g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
g.set_m(random_m(w.n, w.Ms))
g.step(n, w.dt)
print("mavg", g.mavg())
g.close()
