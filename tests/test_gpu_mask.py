"""Geometry mask (reading Q26, "non-regular geometry")
through the C-ABI vs the fp64 oracle's masked fields and steps.

Shapes: an elliptical disc with an off-centre hole (irregular edges on every
row, so the masked stencil meets empty neighbours along x, y and through the
hole) on the 3-D K1..K6 path, the nz = 1 K1/K2'/K5/K6 path and the z-slab path
with virtual ranks (halo planes crossing the mask).  Tolerances as the unmasked
parity tests.  Also: the GPU's own box-embedding invariance and
the round trip to no mask.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.energy import energy as oracle_energy  # noqa: E402
from oracle.fields import heff as oracle_heff  # noqa: E402
from oracle.llg import Sim  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, box_mask, ellipse_mask, random_m  # noqa: E402

CASES = [
    ((64, 48, 4), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 5e3, 0.5, 1e-14, (1e4, -5e3, 2e3)),
    ((100, 25, 1), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, 0.3, 2e-14, (-2e4, 3e3, 0.0)),
    ((36, 20, 33), (2e-9, 2e-9, 2e-9), 1e6, 1e-11, 6.2832e4, 0.5, 1e-15, (0.0, 0.0, 0.0)),
]


def relL2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,d,Ms,A,Ku,alpha,dt,hext", CASES)
def test_masked_heff_steps_energy_match_oracle(n, d, Ms, A, Ku, alpha, dt, hext):
    mask = ellipse_mask(n)
    M = random_m(n, Ms, seed=21)
    g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)
    g.set_geometry(mask)
    g.set_m(M)
    g.set_hext(hext)
    Mg = g.get_m()
    assert np.all(Mg[:, mask == 0] == 0.0)
    op = DemagFFT(tensor_octant(*n, *d))
    sim = Sim(Mg, op, Ms, A, Ku, alpha, GAMMA0, d, hext, mask=mask)
    Hg = g.heff()
    Ho = sim.heff()
    assert np.all(Hg[:, mask == 0] == 0.0)
    assert relL2(Hg, Ho) <= 1e-5
    e_g = g.energy()
    e_o, t_o = oracle_energy(sim.M, op, A, Ms, Ku, d, hext, mask)
    scale = sum(abs(v) for v in t_o.values())
    for k, v in t_o.items():
        assert abs(e_g[k] - v) <= 1e-5 * scale, k
    g.step(1, dt)
    sim.euler_step(dt)
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 2e-5 * Ms
    g.step(9, dt)
    sim.run(9, dt)
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 1e-4 * Ms
    assert np.all(Mg[:, mask == 0] == 0.0)
    nrm = np.sqrt((Mg ** 2).sum(0))
    assert np.abs(nrm[mask == 1] / Ms - 1).max() <= 1e-6
    np.testing.assert_allclose(g.mavg(), sim.mavg(), rtol=0, atol=1e-4)
    g.close()


def test_masked_heun_matches_oracle():
    n, d = (48, 40, 4), (4e-9, 4e-9, 3e-9)
    mask = ellipse_mask(n)
    g = pb.Grace(n, d, 8e5, 1.3e-11, 0.0, 0.2, GAMMA0)
    g.set_geometry(mask)
    g.set_m(random_m(n, 8e5, seed=22))
    g.set_integrator(1)
    sim = Sim(g.get_m(), DemagFFT(tensor_octant(*n, *d)), 8e5, 1.3e-11, 0.0, 0.2, GAMMA0, d, mask=mask)
    g.step(5, 3e-14)
    sim.run(5, 3e-14, "heun")
    assert np.abs(g.get_m() - sim.M).max() <= 1e-4 * 8e5
    g.close()


def test_masked_virtual_ranks_match_single():
    n, d = (40, 24, 8), (3e-9, 3e-9, 3e-9)
    mask = ellipse_mask(n)
    mask[3] = 0  # an empty plane: halos across it
    M = random_m(n, 8e5, seed=23)
    out = []
    for kw in ({}, {"virtual_ranks": 2}, {"virtual_ranks": 4}):
        g = pb.Grace(n, d, 8e5, 1.3e-11, 1e4, 0.5, GAMMA0, **kw)
        g.set_geometry(mask)
        g.set_m(M)
        H = g.heff()
        g.step(5, 1e-14)
        out.append((H, g.get_m(), g.mavg(), g.energy()["total"]))
        g.close()
    for H, Mk, mv, e in out[1:]:
        assert relL2(H, out[0][0]) <= 1e-6
        assert np.abs(Mk - out[0][1]).max() <= 1e-5 * 8e5
        np.testing.assert_allclose(mv, out[0][2], rtol=0, atol=1e-7)
        assert abs(e - out[0][3]) <= 1e-6 * abs(out[0][3])


def test_box_embedding_and_unmask_round_trip():
    """A box magnet in a larger masked grid = the box on its own grid (GPU vs GPU,
    different FFT sizes: fp32 rounding); removing the mask restores the unmasked
    results bit for bit."""
    big, lo, box = (40, 24, 6), (7, 5, 1), (20, 12, 4)
    d = (3e-9, 3e-9, 3e-9)
    args = (8e5, 1.3e-11, 2e4, 0.5, GAMMA0)
    Mb = random_m(box, 8e5, seed=24)
    M = np.zeros((3, big[2], big[1], big[0]))
    sl = (slice(None), slice(lo[2], lo[2] + box[2]), slice(lo[1], lo[1] + box[1]), slice(lo[0], lo[0] + box[0]))
    M[sl] = Mb
    gb = pb.Grace(box, d, *args)
    gb.set_m(Mb)
    gg = pb.Grace(big, d, *args)
    gg.set_geometry(box_mask(big, lo, box))
    gg.set_m(M)
    assert relL2(gg.heff()[sl], gb.heff()) <= 1e-6
    gb.step(10, 1e-14)
    gg.step(10, 1e-14)
    assert np.abs(gg.get_m()[sl] - gb.get_m()).max() <= 1e-5 * 8e5
    np.testing.assert_allclose(gg.mavg(), gb.mavg(), rtol=0, atol=1e-6)
    # round trip: no mask again
    Mr = random_m(big, 8e5, seed=25)
    gg.set_geometry(None)
    gg.set_m(Mr)
    g0 = pb.Grace(big, d, *args)
    g0.set_m(Mr)
    assert np.array_equal(gg.heff(), g0.heff())
    gg.step(3, 1e-14)
    g0.step(3, 1e-14)
    assert np.array_equal(gg.get_m(), g0.get_m())
    for g in (gb, gg, g0):
        g.close()


def test_mask_errors():
    g = pb.Grace((8, 8, 2), (1e-9,) * 3, 8e5, 1e-11, 0, 0.5, GAMMA0)
    with pytest.raises(pb.GraceError) as e:
        g.set_geometry(np.zeros((2, 8, 8), np.uint8))
    assert e.value.code == pb.GRACE_EINVAL
    with pytest.raises(ValueError):
        g.set_geometry(np.ones((2, 8, 7), np.uint8))
    g.close()
