python -m pytest tests/test_gpu_dist.py -q -x -k "pipelined_graph" 2>&1 | grep -E "assert|Error|^E " | head -30 > gpurun_out/dbg_g.log
cat > /tmp/t.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1411_2565_b200 as pb
from workloads import GAMMA0, random_m
n, P, d = (64, 48, 16), 2, (1e-9,)*3
M = random_m(n, 1e6, seed=61)
def run(env, steps):
    for k in ("GRACE_NO_PIPE", "GRACE_DIST_EAGER", "GRACE_NO_PDL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
    g.set_m(M); g.set_hext((1e4, 0, 0))
    H0 = g.heff()
    g.step(steps, 1e-15)
    r = (H0, g.get_m(), pb.grace_partition(g.h))
    g.close()
    return r
ref = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
ref.set_m(M); ref.set_hext((1e4, 0, 0)); Hr = ref.heff(); ref.step(19, 1e-15); Mr = ref.get_m(); ref.close()
for env in ({}, {"GRACE_NO_PIPE": "1"}, {"GRACE_DIST_EAGER": "1"}, {"GRACE_NO_PIPE": "1", "GRACE_DIST_EAGER": "1"}):
    for steps in (1, 19):
        H0, Mo, part = run(env, steps)
        print(env, steps, part["pipelined"], part["graphs"], "H0 diff", float(np.abs(H0 - Hr).max()), 
              "M diff per comp", [float(np.abs(Mo[c] - (Mr[c] if steps == 19 else Mo[c])).max()) for c in range(3)], flush=True)
PY
python /tmp/t.py >> gpurun_out/dbg_g.log 2>&1
