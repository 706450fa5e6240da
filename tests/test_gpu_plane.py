"""KP, the plane-fused y.z.y pass (thin films: 2 <= nz, Pz <= 16; SURVEY §8(f) #3;
opt-in with GRACE_PLANE=1), against the fp64 oracle and against the K2/K3/K4
pencil path it replaces.

Grids span the plane lengths (Py = 256 .. 2048) and z padding
(Pz = 4, 8, 16), with ragged y (ny not a power of two, ny just past Py/4),
z rows below Pz/2 (nz = 3, 5, 6: zero columns in the plane), odd nx and the
full film of BASELINE configs[2].  Bars: H_eff relative L2 <= 1e-5 (north_star)
against the oracle, and the pencil path's H_eff to fp32 rounding (the two
compute the same sums in a different order).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def plane_on(monkeypatch):
    """KP is opt-in (GRACE_PLANE=1, read at context creation)."""
    monkeypatch.setenv("GRACE_PLANE", "1")

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.fields import heff as oracle_heff  # noqa: E402
from oracle.llg import Sim  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, WORKLOADS, random_m  # noqa: E402

PLANE_CASES = [
    # n, d
    ((16, 130, 8), (5e-9, 5e-9, 3e-9)),   # Pz = 16, Py = 256
    ((24, 200, 5), (5e-9, 5e-9, 3e-9)),   # Pz = 16 with nz = 5 (three zero z columns), Py = 512
    ((20, 150, 3), (2e-9, 2e-9, 3e-9)),   # Pz = 8, nz = 3
    ((10, 129, 4), (1e-9, 1e-9, 1e-9)),   # Pz = 8, ny = Py/2 + 1
    ((12, 300, 2), (1e-9, 1e-9, 1e-9)),   # Pz = 4, Py = 1024
    ((9, 257, 6), (3e-9, 2e-9, 1e-9)),    # odd nx, Pz = 16, Py = 1024
    ((6, 700, 2), (1e-9, 1e-9, 1e-9)),    # Pz = 4, Py = 2048, ny > 2 TMA boxes
]


def relL2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make(n, d, Ms=8e5, A=1.3e-11, Ku=0.0, alpha=0.5):
    return pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)


@pytest.mark.parametrize("n,d", PLANE_CASES)
def test_plane_heff_vs_oracle_and_pencil_path(n, d, monkeypatch):
    Ms, A, Ku, hext = 8e5, 1.3e-11, 2e4, (3e3, -1e3, 2e3)
    M = random_m(n, Ms, seed=sum(n))
    g = make(n, d, Ms, A, Ku)
    assert g.geometry["kernels"] == 4 and g.geometry["Pz"] > 1  # K1, KP, K5, K6
    g.set_m(M)
    g.set_hext(hext)
    Hg = g.heff()
    g.close()
    op = DemagFFT(tensor_octant(*n, *d))
    assert relL2(Hg, oracle_heff(M, op, A, Ms, Ku, d, hext)) <= 1e-5
    g0 = make(n, d, Ms, 0.0, 0.0)
    g0.set_m(M)
    Hd = g0.heff()
    g0.close()
    Hdo = op(M)
    assert relL2(Hd, Hdo) <= 1e-5
    assert np.abs(Hd - Hdo).max() <= 2e-5 * Ms
    monkeypatch.delenv("GRACE_PLANE")
    gp = make(n, d, Ms, 0.0, 0.0)
    assert gp.geometry["kernels"] == 6
    gp.set_m(M)
    Hp = gp.heff()
    gp.close()
    assert relL2(Hd, Hp) <= 2e-6


def test_plane_euler_steps_match_oracle_and_pencil_path(monkeypatch):
    n, d = (16, 130, 8), (5e-9, 5e-9, 3e-9)
    Ms, A, alpha, dt = 8e5, 1.3e-11, 0.5, 1e-14
    M = random_m(n, Ms, seed=7)
    g = make(n, d, Ms, A, 0.0, alpha)
    g.set_m(M)
    M0 = g.get_m()
    g.step(1, dt)
    M1 = g.get_m()
    g.step(19, dt)
    Mg = g.get_m()
    g.close()
    sim = Sim(M0, DemagFFT(tensor_octant(*n, *d)), Ms, A, 0.0, alpha, GAMMA0, d)
    sim.euler_step(dt)
    assert np.abs(M1 - sim.M).max() <= 2e-5 * Ms
    monkeypatch.delenv("GRACE_PLANE")
    gp = make(n, d, Ms, A, 0.0, alpha)
    gp.set_m(M)
    gp.step(20, dt)
    Mp = gp.get_m()
    gp.close()
    assert np.abs(Mg - Mp).max() <= 2e-5 * Ms


def test_plane_heun_and_adaptive_match_pencil_path(monkeypatch):
    n, d = (12, 300, 2), (1e-9, 1e-9, 1e-9)
    Ms, A, alpha = 1e6, 1e-11, 0.5
    M = random_m(n, Ms, seed=11)

    def run():
        g = make(n, d, Ms, A, 6.2832e4, alpha)
        g.set_m(M)
        g.set_integrator("heun")
        g.step(4, 2e-15)
        a = g.get_m()
        g.set_integrator("euler")
        g.set_m(M)
        g.step_adaptive(2e-14, 1e-15, 1e-4)
        b = g.get_m()
        k = g.geometry["kernels"]
        g.close()
        return k, a, b

    k1, a1, b1 = run()
    monkeypatch.delenv("GRACE_PLANE")
    k2, a2, b2 = run()
    assert (k1, k2) == (4, 6)
    assert np.abs(a1 - a2).max() <= 1e-5 * Ms
    assert np.abs(b1 - b2).max() <= 1e-4 * Ms


def test_film_runs_plane_path_graph_equals_eager():
    """BASELINE configs[2] on KP: the graph + PDL replay equals the eager launches bit for bit."""
    w = WORKLOADS["film_512x512x8"]
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    assert g.geometry["kernels"] == 4
    M = random_m(w.n, w.Ms, seed=9)
    g.set_m(M)
    g.step(20, w.dt)
    a = g.get_m()
    g.set_m(M)
    pb.grace_set_profiling(g.h, True)
    g.step(20, w.dt)
    pb.grace_set_profiling(g.h, False)
    b = g.get_m()
    g.close()
    assert np.array_equal(a, b)
