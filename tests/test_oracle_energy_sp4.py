"""Pins of oracle/energy.py (absolute values, not only its gradient) and of the
SP4 harness oracle/sp4.py, against what SPEC/the paper and closed forms fix.

energy (Eq. (1); SPEC total_energy examples S:L295-296):
* single cubic cell, uniform M along the easy axis x, no field:
  E_exch = 0, E_anis = 0, E_demag = 1/2 mu0 Ms^2 V / 3 (cube self-energy);
* uniform M perpendicular to the easy axis: E_anis = Ku V per cell;
* uniform M of a whole prism (several cells): E_demag = 1/2 mu0 Ms^2 V_tot D_a,
  D_a the Aharoni prism factor (tests/pins/aharoni.py, an independent closed form);
* Zeeman: -mu0 H_ext . M V per cell, summed;
* exchange of a planar spin spiral with angle step theta along one axis:
  A V (n-1) (2 - 2 cos theta) / Delta^2 per row (the per-bond form of S:L289-297).

sp4 (acceptance 6 S:L499):
* field_Am: B/mu0 for the paper's fields in mT (reading Q12), against the
  A/m values typed independently in SURVEY Sec. 9;
* the relaxed coarse S-state <m> = (0.97, 0.12, 0) +- 0.02 (published
  muMAG submissions);
* field 1 reversal: the first <mx> = 0 crossing within +-10 % of 0.14 ns (SPEC
  acceptance 6; the published muMAG SP4 field-1 curves cross near
  0.14 ns) and a single crossing up to 0.2 ns; |M| = Ms throughout;
* first_crossing on a hand-made series (reading Q20).
"""
import numpy as np
import pytest

from oracle import MU0
from oracle import sp4 as osp4
from oracle.demag import DemagFFT
from oracle.energy import energy
from oracle.tensor import tensor_octant
from tests.pins.aharoni import aharoni_factors
from workloads import uniform_m

MS, A, KU = 8e5, 1.3e-11, 5e4


def _op(n, d):
    return DemagFFT(tensor_octant(*n, *d))


def test_energy_single_cube_along_easy_axis():
    d = (3e-9, 3e-9, 3e-9)
    V = d[0] * d[1] * d[2]
    M = uniform_m((1, 1, 1), MS, (1, 0, 0))
    E, t = energy(M, _op((1, 1, 1), d), A, MS, KU, d, (0.0, 0.0, 0.0))
    assert t["exchange"] == 0.0
    assert t["anisotropy"] == 0.0
    want = 0.5 * MU0 * MS * MS * V / 3.0
    assert abs(t["demag"] - want) <= 1e-12 * want
    assert t["zeeman"] == 0.0
    assert abs(E - want) <= 1e-12 * want


@pytest.mark.parametrize("direction", [(0, 1, 0), (0, 0, 1), (0, 0.6, 0.8)])
def test_energy_anisotropy_perpendicular_is_ku_v_per_cell(direction):
    n, d = (3, 2, 2), (2e-9, 3e-9, 4e-9)
    V = d[0] * d[1] * d[2]
    M = uniform_m(n, MS, direction)
    _, t = energy(M, _op(n, d), A, MS, KU, d, (0.0, 0.0, 0.0))
    want = KU * V * 12
    assert abs(t["anisotropy"] - want) <= 1e-12 * want
    assert t["exchange"] == 0.0


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_energy_demag_whole_prism_aharoni(axis):
    """Uniform M along a of an all-near-field prism: E_d = 1/2 mu0 Ms^2 V_tot D_a."""
    n, d = (5, 4, 3), (2e-9, 3e-9, 5e-9)
    direction = [0, 0, 0]
    direction[axis] = 1
    M = uniform_m(n, MS, direction)
    _, t = energy(M, _op(n, d), A, MS, KU, d, (0.0, 0.0, 0.0))
    D = aharoni_factors(n[0] * d[0], n[1] * d[1], n[2] * d[2])[axis]
    Vtot = n[0] * n[1] * n[2] * d[0] * d[1] * d[2]
    want = 0.5 * MU0 * MS * MS * Vtot * D
    assert abs(t["demag"] - want) <= 1e-10 * want


def test_energy_zeeman_closed_form():
    n, d = (4, 3, 2), (2e-9, 2e-9, 2e-9)
    V = d[0] * d[1] * d[2]
    u = np.array([0.36, 0.48, 0.8])
    M = uniform_m(n, MS, u)
    h = (1e4, -2e4, 3e4)
    _, t = energy(M, _op(n, d), A, MS, 0.0, d, h)
    want = -MU0 * MS * float(np.dot(h, u)) * V * 24
    assert abs(t["zeeman"] - want) <= 1e-12 * abs(want)


@pytest.mark.parametrize("axis,theta", [(3, 0.3), (2, 0.7), (1, 1.1)])
def test_energy_exchange_spin_spiral(axis, theta):
    """m(i) = (cos i theta, sin i theta, 0) along one axis: every bond costs
    |m_{i+1} - m_i|^2 = 2 - 2 cos theta; (n - 1) bonds per line."""
    shape = (3, 3, 4, 5)  # [c][z][y][x]
    d = (2e-9, 3e-9, 5e-9)
    n_ax = shape[axis]
    delta = {3: d[0], 2: d[1], 1: d[2]}[axis]
    idx = np.arange(n_ax)
    bshape = [1, 1, 1]
    bshape[axis - 1] = n_ax
    ang = (idx * theta).reshape(bshape)
    M = np.zeros(shape)
    M[0] = MS * np.cos(ang)
    M[1] = MS * np.sin(ang)
    nlines = (shape[1] * shape[2] * shape[3]) // n_ax
    V = d[0] * d[1] * d[2]
    n = (shape[3], shape[2], shape[1])
    _, t = energy(M, _op(n, d), A, MS, 0.0, d, (0.0, 0.0, 0.0))
    want = A * V * nlines * (n_ax - 1) * (2.0 - 2.0 * np.cos(theta)) / (delta * delta)
    assert abs(t["exchange"] - want) <= 1e-12 * want


# ---------------------------------------------------------------- SP4 harness

def test_sp4_field_Am_values():
    """P:L90 fields in mT -> A/m (B/mu0, reading Q12); SURVEY Sec. 9 values typed
    independently: F1 = (-19576.058, 3421.831, 0), F2 = (-28250.002, -5013.381, 0)."""
    f1 = osp4.field_Am(osp4.FIELD1_MT)
    f2 = osp4.field_Am(osp4.FIELD2_MT)
    np.testing.assert_allclose(f1, (-19576.058, 3421.831, 0.0), rtol=0, atol=2e-3)
    np.testing.assert_allclose(f2, (-28250.002, -5013.381, 0.0), rtol=0, atol=2e-3)
    # the paper's values themselves: -24.6 / 4.3 mT and -35.5 / -6.3 mT
    assert osp4.FIELD1_MT == (-24.6, 4.3, 0.0) and osp4.FIELD2_MT == (-35.5, -6.3, 0.0)
    # material and discretisation (reading Q14)
    assert (osp4.MS, osp4.A_EX, osp4.GAMMA0) == (8.0e5, 1.3e-11, 2.211e5)
    c1 = osp4.CONFIGS["sp4_field1_coarse"]
    assert c1["n"] == (100, 25, 1) and np.allclose(np.array(c1["n"]) * np.array(c1["d"]), (500e-9, 125e-9, 3e-9))
    c2 = osp4.CONFIGS["sp4_field2_refined"]
    assert c2["n"] == (200, 50, 1) and np.allclose(np.array(c2["n"]) * np.array(c2["d"]), (500e-9, 125e-9, 3e-9))


def test_sp4_first_crossing_hand_series():
    t = np.array([0.0, 1.0, 2.0, 3.0, 4.0])
    assert osp4.first_crossing(t, np.array([1.0, 0.5, -0.5, -1.0, 0.2])) == 1.5
    assert osp4.first_crossing(t, np.array([1.0, 0.25, 0.0, -1.0, -1.0])) == 2.0
    assert osp4.first_crossing(t, np.array([-1.0, -0.5, 0.5, 1.0, 1.0])) is None
    assert osp4.first_crossing(t, np.array([-1.0, 0.5, 0.2, -0.6, 1.0])) == 2.25


@pytest.mark.slow
def test_sp4_coarse_sstate_and_field1_crossing():
    """SPEC S:L307 S-state and acceptance 6 crossing, on the oracle itself."""
    name = "sp4_field1_coarse"
    sim = osp4.make_sim(name)
    E0, _ = energy(sim.M, sim.demag, osp4.A_EX, osp4.MS, 0.0, osp4.CONFIGS[name]["d"], (0.0, 0.0, 0.0))
    osp4.relax(sim, name)
    m = sim.mavg()
    assert abs(m[0] - 0.97) <= 0.02 and abs(m[1] - 0.12) <= 0.02 and abs(m[2]) <= 0.02, m
    E1, _ = energy(sim.M, sim.demag, osp4.A_EX, osp4.MS, 0.0, osp4.CONFIGS[name]["d"], (0.0, 0.0, 0.0))
    assert E1 < E0  # damped relaxation lowers Eq. (1)
    # reversal under field 1 up to 0.2 ns (8000 steps of 2.5e-14 s)
    t, ms = osp4.reverse(sim, name, steps=8000)
    tc = osp4.first_crossing(t, ms[:, 0])
    assert tc is not None and abs(tc - 0.14e-9) <= 0.1 * 0.14e-9, tc
    assert np.sum((ms[:-1, 0] > 0) & (ms[1:, 0] <= 0)) == 1
    nrm = np.sqrt((sim.M ** 2).sum(0))
    assert np.abs(nrm / osp4.MS - 1).max() <= 1e-12
