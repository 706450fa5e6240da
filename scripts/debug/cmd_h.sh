cat > /tmp/t2.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1411_2565_b200 as pb
from workloads import GAMMA0, random_m
n, P, d = (64, 48, 16), 2, (1e-9,)*3
M = random_m(n, 1e6, seed=61)
ref = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
ref.set_m(M); ref.set_hext((1e4, 0, 0)); ref.step(19, 1e-15); Hr = ref.heff(); Mr = ref.get_m(); ref.close()
for env in ({}, {"GRACE_NO_PIPE": "1"}, {"GRACE_DIST_EAGER": "1"}, {"GRACE_NO_PIPE": "1", "GRACE_DIST_EAGER": "1"}):
    for k in ("GRACE_NO_PIPE", "GRACE_DIST_EAGER"):
        os.environ.pop(k, None)
    os.environ.update(env)
    for rep in range(2):
        g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
        g.set_m(M); g.set_hext((1e4, 0, 0))
        g.step(19, 1e-15)
        H = g.heff(); Mo = g.get_m()
        g.close()
        dz = [float(np.abs(H[:, z] - Hr[:, z]).max()) for z in range(16)]
        print(env, rep, "M", float(np.abs(Mo - Mr).max()), "H per comp", [float(np.abs(H[c] - Hr[c]).max()) for c in range(3)], "H per z", [f"{v:.3g}" for v in dz], flush=True)
PY
python /tmp/t2.py > gpurun_out/dbg_h.log 2>&1
python -m pytest tests/test_gpu_dist.py -q 2>&1 | tail -3 >> gpurun_out/dbg_h.log
