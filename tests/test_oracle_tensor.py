"""Pins of the oracle's demag tensor (oracle/tensor.py) against things it does not compute itself.

* closed forms: cube self-term 1/3, Aharoni's prism factor for a
  single non-cubic cell and for the whole sample (tests/pins/aharoni.py);
* direct Gauss-Legendre quadrature of the dipole kernel over two cells
  (tests/pins/quadrature.py) -- pins f, g, the stencil weights, the
  permutations and the sign of every component;
* the point-dipole limit, zero trace off the origin, exact
  parity and zeros (reading Q7).
"""
import numpy as np
import pytest

from oracle.tensor import COMPONENTS, full_tensor, tensor_entry, tensor_octant
from tests.pins.aharoni import aharoni_factors
from tests.pins.quadrature import cell_tensor_quad


def test_cube_self_term_one_third():
    o = tensor_octant(1, 1, 1, 1e-9, 1e-9, 1e-9)
    for c in (0, 3, 5):
        assert abs(o[c, 0, 0, 0] - 1.0 / 3.0) < 1e-14
    for c in (1, 2, 4):
        assert o[c, 0, 0, 0] == 0.0


@pytest.mark.parametrize("d", [(5e-9, 5e-9, 3e-9), (2.5e-9, 2.5e-9, 3e-9), (1e-9, 2e-9, 3e-9), (4e-9, 1e-9, 1e-9)])
def test_single_cell_equals_aharoni(d):
    o = tensor_octant(1, 1, 1, *d)
    D = aharoni_factors(*d)
    np.testing.assert_allclose([o[0, 0, 0, 0], o[3, 0, 0, 0], o[5, 0, 0, 0]], D, rtol=0, atol=1e-14)
    assert abs(o[0, 0, 0, 0] + o[3, 0, 0, 0] + o[5, 0, 0, 0] - 1.0) < 1e-13


CASES = [
    ((1.0, 1.0, 1.0), [("xx", (2, 0, 0)), ("xy", (2, 1, 0)), ("xz", (2, 0, 1)), ("yz", (0, 2, 1)),
                       ("zz", (1, 2, 1)), ("yy", (3, 2, 1)), ("xy", (3, 2, 2))]),
    ((5.0, 5.0, 3.0), [("xx", (2, 0, 0)), ("yy", (0, 2, 0)), ("zz", (0, 0, 2)), ("xy", (2, 1, 0)),
                       ("xz", (2, 0, 1)), ("yz", (0, 2, 1)), ("xz", (1, 1, 2)), ("zz", (1, 2, 1))]),
    ((1.0, 2.0, 3.0), [("xx", (2, 1, 1)), ("xy", (1, 2, 1)), ("xz", (2, 1, 3)), ("yz", (1, 2, 1)),
                       ("yy", (1, 2, 0)), ("zz", (0, 1, 2))]),
]


@pytest.mark.parametrize("d,cases", CASES)
def test_newell_matches_direct_quadrature(d, cases):
    for comp, R in cases:
        q = cell_tensor_quad(comp, [R[a] * d[a] for a in range(3)], d, n=24)
        e = tensor_entry(comp, *R, *[x * 1e-9 for x in d])
        assert abs(e - q) <= 1e-10 * abs(q) + 1e-16, (comp, R, e, q)


def test_dipole_far_field_limit():
    # displacement (10,0,0) cubic cells -> dipole value within 0.1 %
    dip = -2.0 * 1.0 / (4.0 * np.pi * 10.0 ** 3)
    e = tensor_entry("xx", 10, 0, 0, 1.0, 1.0, 1.0)
    assert e < 0 and abs(e - dip) / abs(dip) < 1e-3
    # beyond the cutoff the tensor is exactly the dipole formula, continuous with Newell
    o = tensor_octant(60, 1, 1, 1e-9, 1e-9, 1e-9)
    last_near = int(np.floor(30.0 * np.sqrt(3.0)))  # 51
    rn, rf = last_near, last_near + 1
    dipf = -2.0 * 1e-27 / (4.0 * np.pi * (rf * 1e-9) ** 3)
    assert abs(o[0, 0, 0, rf] - dipf) / abs(dipf) < 1e-12
    # Newell at 51 vs dipole at 51: agreement to the Q6 envelope
    dipn = -2.0 * 1e-27 / (4.0 * np.pi * (rn * 1e-9) ** 3)
    assert abs(o[0, 0, 0, rn] - dipn) / abs(dipn) < 1e-5


def test_trace_zero_off_origin_and_parity():
    o = tensor_octant(9, 7, 4, 2e-9, 1e-9, 1.5e-9)
    tr = o[0] + o[3] + o[5]
    tr[0, 0, 0] -= 1.0
    assert np.abs(tr).max() < 1e-8
    # exact zeros (Q7)
    assert np.all(o[1][:, :, 0] == 0) and np.all(o[1][:, 0, :] == 0)
    assert np.all(o[2][:, :, 0] == 0) and np.all(o[2][0, :, :] == 0)
    assert np.all(o[4][:, 0, :] == 0) and np.all(o[4][0, :, :] == 0)
    # full tensor symmetric; N_xy odd in x and y, even in z
    N = full_tensor(o, 2, 3, 1)
    assert np.array_equal(N, N.T)
    assert full_tensor(o, -2, 3, 1)[0, 1] == -N[0, 1]
    assert full_tensor(o, 2, -3, 1)[0, 1] == -N[0, 1]
    assert full_tensor(o, 2, 3, -1)[0, 1] == N[0, 1]
    assert full_tensor(o, -2, -3, -1)[0, 0] == N[0, 0]


def test_octant_matches_entries():
    d = (5e-9, 5e-9, 3e-9)
    o = tensor_octant(70, 6, 2, *d)  # spans near and far field
    rng = np.random.default_rng(0)
    for _ in range(40):
        c, k, j, i = rng.integers(0, 6), rng.integers(0, 2), rng.integers(0, 6), rng.integers(0, 70)
        assert o[c, k, j, i] == tensor_entry(int(c), int(i), int(j), int(k), *d)
    assert COMPONENTS == ("xx", "xy", "xz", "yy", "yz", "zz")
