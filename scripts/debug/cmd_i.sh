cat > /tmp/t3.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1411_2565_b200 as pb
from workloads import GAMMA0, random_m
for n in ((64, 48, 16), (128, 64, 16), (100, 25, 1), (1024, 1024, 32)):
    d = (1e-9,)*3
    M = random_m(n, 1e6, seed=61)
    g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
    g.set_m(M); g.set_hext((1e4, 0, 0)); g.step(19, 1e-15)
    H1 = g.heff(); H1b = g.heff(); Mo = g.get_m(); H2 = g.heff()
    print(n, "heff twice", float(np.abs(H1 - H1b).max()), "after get_m", float(np.abs(H1 - H2).max()),
          [float(np.abs(H1[c] - H2[c]).max()) for c in range(3)], flush=True)
    if n[2] > 1:
        bad = np.argwhere(np.abs(H1 - H2) > 0)
        print("   first bad", bad[:5].tolist(), len(bad))
    g.close()
PY
python /tmp/t3.py > gpurun_out/dbg_i.log 2>&1
