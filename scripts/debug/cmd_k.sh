cat > /tmp/t4.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1411_2565_b200 as pb
from workloads import GAMMA0, random_m
n, P, d = (128, 64, 16), 4, (1e-9,)*3
M = random_m(n, 1e6, seed=61)
mode = sys.argv[1]
g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
g.set_m(M); g.set_hext((1e4, 0, 0))
Hs = []
H0 = g.heff(); Hs.append(H0)
if mode == "a":
    g.step(19, 1e-15)
    Hs.append(g.heff()); Hs.append(g.heff())
Mo = g.get_m()
g.close()
ref = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
ref.set_m(M); ref.set_hext((1e4, 0, 0)); R = [ref.heff()]
if mode == "a":
    ref.step(19, 1e-15); R.append(ref.heff()); R.append(ref.heff())
Mr = ref.get_m(); ref.close()
print(mode, "M", float(np.abs(Mo-Mr).max()))
for H, Hr in zip(Hs, R):
    print("  H per comp", [float(np.abs(H[c]-Hr[c]).max()) for c in range(3)], "per z", [f"{float(np.abs(H[:, z]-Hr[:, z]).max()):.2g}" for z in range(n[2])], flush=True)
PY
python /tmp/t4.py a > gpurun_out/dbg_k.log 2>&1
python /tmp/t4.py b >> gpurun_out/dbg_k.log 2>&1
GRACE_NO_PDL=1 python /tmp/t4.py a >> gpurun_out/dbg_k.log 2>&1
