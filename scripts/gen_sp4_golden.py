"""Write the oracle's muMAG SP4 trajectories to tests/golden/ (calls only oracle/).

Usage: python scripts/gen_sp4_golden.py [sp4_field1_coarse|sp4_field2_refined ...]

For each config (oracle/sp4.py CONFIGS; readings Q13-Q15, Q20): relax from
uniform (1,1,1)/sqrt(3) at alpha = 1, H = 0; store the relaxed S-state M
(npy) and its <m>; then reverse at alpha = 0.02 under the field and store
<m>(t) every 10 ps.  These files are oracle output, not paper numbers: the
paper's Figs. 2-5 print none.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import sp4  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def main(names):
    os.makedirs(GOLD, exist_ok=True)
    for name in names:
        t0 = time.time()
        sim = sp4.make_sim(name)
        sp4.relax(sim, name)
        np.save(os.path.join(GOLD, f"{name}_sstate.npy"), sim.M)
        m0 = sim.mavg()
        ts, ms = sp4.reverse(sim, name)
        tc = sp4.first_crossing(ts, ms[:, 0])
        path = os.path.join(GOLD, f"{name}_oracle.csv")
        with open(path, "w") as f:
            f.write(f"# oracle/sp4.py {name}: fp64 oracle trajectory written by scripts/gen_sp4_golden.py\n")
            f.write(f"# config: {sp4.CONFIGS[name]}\n")
            f.write(f"# relaxed S-state <m> = {m0[0]:.9f} {m0[1]:.9f} {m0[2]:.9f}\n")
            f.write(f"# first <mx>=0 crossing (linear interpolation) t = {tc!r} s\n")
            f.write("# t_s mx my mz\n")
            for t, m in zip(ts, ms):
                f.write(f"{t:.6e} {m[0]:.12f} {m[1]:.12f} {m[2]:.12f}\n")
        print(name, "S-state", m0, "crossing", tc, f"{time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(sp4.CONFIGS))
