"""Pins of the oracle's geometry mask (reading Q26, the
paper's "non-regular geometry").

The pin is embedding invariance, fixed by the physics rather than by the code:
a magnet occupying a box of a larger masked grid is the same magnet as that box
simulated on its own grid.  The demag convolution sees M = 0 outside (the
tensor depends on the offset only), exchange bonds to empty cells vanish like
the outer Neumann boundary, and the update leaves empty cells at 0.  A dropped
bond mask, a bond kept to an empty cell, an unmasked renormalisation (0/0) or an
<m> over all cells each break one of these tests.  An all-ones mask must equal
the unmasked oracle exactly.
"""
import numpy as np
import pytest

from oracle.demag import DemagFFT
from oracle.energy import energy
from oracle.fields import heff
from oracle.llg import Sim
from oracle.tensor import tensor_octant
from workloads import GAMMA0, box_mask, ellipse_mask, random_m

MS, A, KU = 8e5, 1.3e-11, 5e3
D = (5e-9, 4e-9, 3e-9)
HEXT = (1.5e4, -7e3, 3e3)
BIG, LO, BOX = (16, 9, 4), (3, 2, 1), (10, 6, 2)


def _embed(Mb):
    M = np.zeros((3, BIG[2], BIG[1], BIG[0]))
    M[:, LO[2]:LO[2] + BOX[2], LO[1]:LO[1] + BOX[1], LO[0]:LO[0] + BOX[0]] = Mb
    return M


def _box(M):
    return M[:, LO[2]:LO[2] + BOX[2], LO[1]:LO[1] + BOX[1], LO[0]:LO[0] + BOX[0]]


@pytest.fixture(scope="module")
def ops():
    return DemagFFT(tensor_octant(*BIG, *D)), DemagFFT(tensor_octant(*BOX, *D))


def test_heff_box_embedding(ops):
    big, small = ops
    mask = box_mask(BIG, LO, BOX)
    Mb = random_m(BOX, MS, seed=11)
    Hb = heff(Mb, small, A, MS, KU, D, HEXT)
    H = heff(_embed(Mb), big, A, MS, KU, D, HEXT, mask)
    assert np.abs(_box(H) - Hb).max() <= 1e-10 * np.abs(Hb).max()
    out = H.copy()
    out[:, LO[2]:LO[2] + BOX[2], LO[1]:LO[1] + BOX[1], LO[0]:LO[0] + BOX[0]] = 0
    assert np.all(out == 0.0)
    # without the bond mask the box surface picks up -M_c/Delta^2 terms
    Hu = heff(_embed(Mb), big, A, MS, KU, D, HEXT) * mask
    assert np.abs(_box(Hu) - Hb).max() > 1e3 * np.abs(_box(H) - Hb).max() + 1.0


@pytest.mark.parametrize("method", ["euler", "heun"])
def test_steps_box_embedding(ops, method):
    big, small = ops
    Mb = random_m(BOX, MS, seed=12)
    sb = Sim(Mb, small, MS, A, KU, 0.3, GAMMA0, D, HEXT)
    sg = Sim(_embed(Mb), big, MS, A, KU, 0.3, GAMMA0, D, HEXT, mask=box_mask(BIG, LO, BOX))
    sb.run(4, 2e-14, method)
    sg.run(4, 2e-14, method)
    assert np.abs(_box(sg.M) - sb.M).max() <= 1e-10 * MS
    assert np.all(sg.M[:, box_mask(BIG, LO, BOX) == 0] == 0.0)
    assert np.allclose(sg.mavg(), sb.mavg(), rtol=0, atol=1e-12)


def test_energy_box_embedding(ops):
    big, small = ops
    Mb = random_m(BOX, MS, seed=13)
    eb, tb = energy(Mb, small, A, MS, KU, D, HEXT)
    eg, tg = energy(_embed(Mb), big, A, MS, KU, D, HEXT, box_mask(BIG, LO, BOX))
    for k in tb:
        assert abs(tg[k] - tb[k]) <= 1e-10 * abs(eb) + 1e-30, k


def test_all_ones_mask_is_unmasked(ops):
    big, _ = ops
    M = random_m(BIG, MS, seed=14)
    ones = np.ones((BIG[2], BIG[1], BIG[0]), dtype=np.uint8)
    assert np.array_equal(heff(M, big, A, MS, KU, D, HEXT, ones), heff(M, big, A, MS, KU, D, HEXT))
    s0 = Sim(M, big, MS, A, KU, 0.5, GAMMA0, D, HEXT)
    s1 = Sim(M, big, MS, A, KU, 0.5, GAMMA0, D, HEXT, mask=ones)
    s0.run(2, 1e-14)
    s1.run(2, 1e-14)
    assert np.array_equal(s0.M, s1.M)


def test_ellipse_mask_invariants(ops):
    """Irregular shape: |M| = Ms on the magnet, 0 elsewhere; the damped energy
    decreases with the masked fields."""
    big, _ = ops
    mask = ellipse_mask(BIG)
    assert 0 < mask.sum() < mask.size
    s = Sim(random_m(BIG, MS, seed=15), big, MS, A, KU, 1.0, GAMMA0, D, (0.0, 0.0, 0.0), mask=mask)
    e0 = energy(s.M, big, A, MS, KU, D, (0, 0, 0), mask)[0]
    s.run(20, 5e-14)
    e1 = energy(s.M, big, A, MS, KU, D, (0, 0, 0), mask)[0]
    n = np.sqrt((s.M * s.M).sum(axis=0))
    assert np.allclose(n[mask == 1], MS, rtol=1e-12) and np.all(n[mask == 0] == 0)
    assert e1 < e0
