"""Adaptive time steps on the GPU (grace_step_adaptive, P:L129 future work) against
the oracle's Sim.adaptive_run: the same controller, so the same accepted and
rejected counts and the same final state within fp32 rounding; the single-cell
precession closed form (each accepted step rotates by the exact Heun angle)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.llg import Sim  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, random_m  # noqa: E402


def test_adaptive_single_cell_precession():
    g0, Hm, Ms = GAMMA0, 1e5, 8e5
    g = pb.Grace((1, 1, 1), (2e-9,) * 3, Ms, 0.0, 0.0, 0.0, g0)
    M = np.zeros((3, 1, 1, 1))
    M[0] = Ms
    g.set_m(M)
    g.set_hext((0, 0, Hm))
    sim = Sim(M, DemagFFT(tensor_octant(1, 1, 1, 2e-9, 2e-9, 2e-9)), Ms, 0.0, 0.0, 0.0, g0, (2e-9,) * 3,
              hext=(0, 0, Hm))
    log, dto = sim.adaptive_run(3e-11, 1e-15, 1e-5)
    dt, acc, rej = g.step_adaptive(3e-11, 1e-15, 1e-5)
    assert acc == sum(1 for x in log if x[3]) and rej == sum(1 for x in log if not x[3])
    assert abs(dt / dto - 1) <= 1e-3
    assert np.abs(g.get_m()[:, 0, 0, 0] - sim.M[:, 0, 0, 0]).max() <= 2e-5 * Ms
    assert g.steps == acc
    g.close()


@pytest.mark.parametrize("n,d,vr", [((24, 10, 3), (2e-9, 2e-9, 3e-9), None), ((100, 25, 1), (5e-9, 5e-9, 3e-9), None),
                                    ((32, 16, 8), (2e-9, 2e-9, 2e-9), 2)])
def test_adaptive_matches_oracle(n, d, vr):
    Ms, A, Ku, alpha = 8e5, 1.3e-11, 1e4, 0.1
    hext = (2e4, -1e4, 5e3)
    M = random_m(n, Ms, seed=23)
    g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0, virtual_ranks=vr)
    g.set_m(M)
    g.set_hext(hext)
    sim = Sim(g.get_m(), DemagFFT(tensor_octant(*n, *d)), Ms, A, Ku, alpha, GAMMA0, d, hext)
    T, tol = 2e-12, 2e-4
    log, dto = sim.adaptive_run(T, 1e-15, tol)
    dt, acc, rej = g.step_adaptive(T, 1e-15, tol)
    na, nr = sum(1 for x in log if x[3]), sum(1 for x in log if not x[3])
    # the same decisions except where an error estimate sits within fp32 noise of tol
    assert abs(acc - na) <= 1 and abs(rej - nr) <= 1, (acc, rej, na, nr)
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 1e-4 * Ms
    assert np.abs(np.sqrt((Mg ** 2).sum(0)) / Ms - 1).max() <= 1e-6
    # state and step counter continue normally after an adaptive run
    g.step(2, 1e-15)
    sim.run(2, 1e-15)
    assert np.abs(g.get_m() - sim.M).max() <= 1e-4 * Ms
    with pytest.raises(pb.GraceError):
        g.step_adaptive(1e-12, -1.0, tol)
    g.close()
