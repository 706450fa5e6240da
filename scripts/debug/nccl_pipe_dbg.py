import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
if len(sys.argv) > 1:
    os.environ["GRACE_FORCE_NCCL"] = "1"
    import paper_1411_2565_b200 as pb
    from workloads import GAMMA0, random_m
    n, d, Ms = (48, 20, 6), (2e-9, 2e-9, 3e-9), 8e5
    M = random_m(n, Ms, seed=53)
    h = pb.grace_create_dist(*n, *d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, 0, 1, pb.grace_nccl_unique_id())
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    out = []
    for hh in (h, ref.h):
        pb.grace_set_m(hh, M.ravel().copy())
        pb.grace_set_hext(hh, 1e4, -3e3, 2e3)
        H = np.empty(3 * M[0].size)
        pb.grace_heff(hh, H)
        H2 = np.empty(3 * M[0].size)
        pb.grace_heff(hh, H2)
        out.append((H.reshape(3, -1), H2.reshape(3, -1)))
    a, b = out
    print(sys.argv[1], pb.grace_partition(h), [float(np.abs(a[0][c] - b[0][c]).max()) for c in range(3)],
          [float(np.abs(a[1][c] - b[1][c]).max()) for c in range(3)], flush=True)
else:
    for env in ({}, {"GRACE_NO_PIPE": "1"}, {"GRACE_DIST_EAGER": "1"}, {"GRACE_NO_HALO_COMM": "1"},
                {"GRACE_NO_PIPE": "1", "GRACE_DIST_EAGER": "1"}):
        e = dict(os.environ); e.update(env)
        subprocess.run([sys.executable, __file__, json.dumps(env)], env=e)
