"""muMAG standard problem #4 harness, fp64 (BASELINE.json configs 1-2).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L90: permalloy film 500 x 125 x 3 nm, A = 1.3e-11 J/m, Ms = 8.0e5 A/m, no
anisotropy; "relaxed to S-state by setting a large damping constant"; then
field 1 (-24.6, 4.3, 0) mT or field 2 (-35.5, -6.3, 0) mT with alpha = 0.02.
Discretisation per BASELINE.json (reading Q14): 100x25x1 cells of 5x5x3 nm
(config 1) and 200x50x1 cells of 2.5x2.5x3 nm (config 2).  Initial state,
relaxation length and time steps per readings Q13/Q15; fields in A/m = B/mu0
(reading Q12).  <m> is recorded every 10 ps (reading Q20).
"""
import numpy as np

from . import MU0
from .demag import DemagFFT
from .llg import Sim
from .tensor import tensor_octant

GAMMA0 = 2.211e5  # gamma*mu0, m/(A s) (reading Q1)
MS = 8.0e5
A_EX = 1.3e-11
FIELD1_MT = (-24.6, 4.3, 0.0)
FIELD2_MT = (-35.5, -6.3, 0.0)

CONFIGS = {
    # name: grid, cell, field (mT), relax (steps, dt), run (steps, dt), record every
    "sp4_field1_coarse": dict(n=(100, 25, 1), d=(5e-9, 5e-9, 3e-9), field=FIELD1_MT,
                              relax=(30000, 1e-13), run=(40000, 2.5e-14), every=400),
    "sp4_field2_refined": dict(n=(200, 50, 1), d=(2.5e-9, 2.5e-9, 3e-9), field=FIELD2_MT,
                               relax=(40000, 5e-14), run=(160000, 6.25e-15), every=1600),
}


def field_Am(mT):
    return tuple(b * 1e-3 / MU0 for b in mT)


def make_sim(name, demag_op=None):
    cfg = CONFIGS[name]
    nx, ny, nz = cfg["n"]
    d = cfg["d"]
    if demag_op is None:
        demag_op = DemagFFT(tensor_octant(nx, ny, nz, *d))
    M = np.empty((3, nz, ny, nx))
    M[:] = (MS / np.sqrt(3.0))  # uniform (1,1,1)/sqrt(3) saturation (reading Q15)
    return Sim(M, demag_op, MS, A_EX, 0.0, 1.0, GAMMA0, d)


def relax(sim, name):
    steps, dt = CONFIGS[name]["relax"]
    sim.alpha = 1.0
    sim.hext = (0.0, 0.0, 0.0)
    sim.run(steps, dt)
    return sim


def reverse(sim, name, steps=None, record=True):
    """alpha -> 0.02, H -> field; returns (t [s], <m> [k,3]) sampled every ``every`` steps."""
    cfg = CONFIGS[name]
    nsteps, dt = cfg["run"]
    if steps is not None:
        nsteps = steps
    sim.alpha = 0.02
    sim.hext = field_Am(cfg["field"])
    ts, ms = [0.0], [sim.mavg()]
    for s in range(1, nsteps + 1):
        sim.euler_step(dt)
        if record and s % cfg["every"] == 0:
            ts.append(s * dt)
            ms.append(sim.mavg())
    return np.array(ts), np.array(ms)


def first_crossing(t, mx):
    """First sample with <mx> <= 0 after one > 0, linearly interpolated (reading Q20)."""
    for i in range(1, len(t)):
        if mx[i - 1] > 0.0 and mx[i] <= 0.0:
            return t[i - 1] + (t[i] - t[i - 1]) * mx[i - 1] / (mx[i - 1] - mx[i])
    return None
