"""Small-grid latency path (opt-in GRACE_SMALL=1, measured
slower than the pencil path): grace_step(n) of the SP4 grids runs as one
thread-block-cluster kernel with every intermediate in distributed shared memory.  Same arithmetic as the pencil path (same FFT
plans, KS table, stencil and update expressions), so the two agree to fp32
rounding order (observed: bitwise); the oracle parity of the small path is the
SP4 trajectory test (tests/test_gpu_parity.py) and the steps below."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.llg import Sim  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, WORKLOADS, random_m  # noqa: E402


def _run(w, M, nsteps, small, sched=None):
    if small:
        os.environ["GRACE_SMALL"] = "1"
    else:
        os.environ.pop("GRACE_SMALL", None)
    try:
        g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
        g.set_m(M)
        g.set_hext(w.hext)
        if sched:
            g.set_field_schedule(*sched)
        for k in nsteps:
            g.step(k, w.dt)
        out = (g.get_m(), g.steps, g.mavg())
        g.close()
    finally:
        os.environ.pop("GRACE_SMALL", None)
    return out


@pytest.mark.parametrize("name", ["sp4_field1", "sp4_field2_refined"])
def test_small_path_matches_pencil_path(name):
    w = WORKLOADS[name]
    M = random_m(w.n, w.Ms, seed=71)
    a = _run(w, M, (1, 16, 20), True)
    b = _run(w, M, (1, 16, 20), False)
    assert a[1] == b[1] == 37
    assert np.abs(a[0] - b[0]).max() <= 1e-6 * w.Ms, np.abs(a[0] - b[0]).max()
    np.testing.assert_allclose(a[2], b[2], rtol=0, atol=1e-7)
    # with a field schedule (step-indexed applied field)
    sched = ((0.0, 3e4, -2e4), 3, 9, 20)
    a = _run(w, M, (5, 24), True, sched)
    b = _run(w, M, (5, 24), False, sched)
    assert np.abs(a[0] - b[0]).max() <= 1e-6 * w.Ms


def test_small_path_steps_match_oracle(monkeypatch):
    monkeypatch.setenv("GRACE_SMALL", "1")
    w = WORKLOADS["sp4_field1"]
    M = random_m(w.n, w.Ms, seed=72)
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    g.set_m(M)
    g.set_hext(w.hext)
    sim = Sim(g.get_m(), DemagFFT(tensor_octant(*w.n, *w.d)), w.Ms, w.A, w.Ku, w.alpha, GAMMA0, w.d, w.hext)
    g.step(1, w.dt)
    sim.euler_step(w.dt)
    assert np.abs(g.get_m() - sim.M).max() <= 2e-5 * w.Ms
    g.step(40, w.dt)
    sim.run(40, w.dt)
    assert np.abs(g.get_m() - sim.M).max() <= 1e-4 * w.Ms
    # the non-finite report carries the step and cell
    g.set_hext((3e38, 3e38, 3e38))
    with pytest.raises(pb.GraceError) as e:
        g.step(3, 1e-13)
    assert e.value.code == pb.GRACE_ENONFINITE
    assert pb.grace_last_nonfinite(g.h)[0] == 41
    g.close()
