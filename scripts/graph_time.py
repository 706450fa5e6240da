"""Time graph-mode steps (the product path, no per-kernel events) for A/B runs.

python scripts/graph_time.py [workload] [steps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1411_2565_b200 as pb  # noqa: E402
from workloads import WORKLOADS, random_m  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "slab_1024x1024x32"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0)
integ = os.environ.get("GRACE_INTEGRATOR", "euler")
g.set_integrator(integ)
s = torch.cuda.Stream()
pb.grace_set_stream(g.h, s.cuda_stream)
g.set_m(random_m(w.n, w.Ms))
g.set_hext(w.hext)
g.step(16, w.dt)
res = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    g.step(steps, w.dt)
    e1.record(s)
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / steps)
print(f"{w.name} graph-mode ms/step {min(res):.4f} (runs {', '.join('%.4f' % r for r in res)}) "
      f"PDL={'off' if os.environ.get('GRACE_NO_PDL') else 'on'} integrator={integ}")
