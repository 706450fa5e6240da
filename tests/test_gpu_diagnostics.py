"""Energy, max torque and relax through the C-ABI vs the oracle.

grace_energy / grace_max_torque evaluate H_demag with the step's kernels and
reduce in fp64; the oracle's Eq. (1) energy (oracle/energy.py, pinned there by
finite differences against the fields) and its H_eff give the references.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle import MU0  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.energy import energy as oracle_energy  # noqa: E402
from oracle.fields import heff as oracle_heff  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, random_m, uniform_m  # noqa: E402

CASES = [
    ((16, 8, 4), (2e-9, 2e-9, 3e-9), 8e5, 1.3e-11, 2e4, (1e4, -2e4, 5e3)),
    ((100, 25, 1), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, (-19576.058, 3421.831, 0.0)),
    ((33, 17, 5), (1e-9, 1.5e-9, 2e-9), 1e6, 1e-11, 6.2832e4, (5e3, -5e3, 1e4)),
]


@pytest.mark.parametrize("n,d,Ms,A,Ku,hext", CASES)
def test_energy_terms_match_oracle(n, d, Ms, A, Ku, hext):
    g = pb.Grace(n, d, Ms, A, Ku, 0.5, GAMMA0)
    g.set_m(random_m(n, Ms, seed=17))
    g.set_hext(hext)
    M = g.get_m()  # the fp32 state the GPU holds
    tot, terms = oracle_energy(M, DemagFFT(tensor_octant(*n, *d)), A, Ms, Ku, d, hext)
    e = g.energy()
    for k in ("exchange", "anisotropy", "demag", "zeeman"):
        assert abs(e[k] - terms[k]) <= 1e-5 * max(abs(terms[k]), 1e-3 * abs(tot) + 1e-30), (k, e[k], terms[k])
    assert abs(e["total"] - tot) <= 1e-5 * (abs(terms["exchange"]) + abs(terms["demag"]) + abs(terms["zeeman"])
                                           + abs(terms["anisotropy"]))
    g.close()


def test_energy_single_cube_closed_form():
    """One cubic cell along z: E_demag = mu0 Ms^2 V / 6 (N_zz = 1/3), no exchange,
    anisotropy Ku V (m_x = 0), Zeeman -mu0 V H.M."""
    n, d, Ms, Ku = (1, 1, 1), (3e-9, 3e-9, 3e-9), 8e5, 5e4
    hext = (1e3, 2e3, 3e3)
    g = pb.Grace(n, d, Ms, 1.3e-11, Ku, 0.5, GAMMA0)
    g.set_m(uniform_m(n, Ms, (0, 0, 1)))
    g.set_hext(hext)
    e = g.energy()
    V = d[0] * d[1] * d[2]
    assert e["exchange"] == 0.0
    assert abs(e["demag"] - MU0 * Ms * Ms * V / 6) <= 1e-6 * MU0 * Ms * Ms * V / 6
    assert abs(e["anisotropy"] - Ku * V) <= 1e-7 * Ku * V
    assert abs(e["zeeman"] + MU0 * V * hext[2] * Ms) <= 1e-6 * MU0 * V * hext[2] * Ms
    g.close()


@pytest.mark.parametrize("n,d,Ms,A,Ku,hext", CASES)
def test_max_torque_matches_oracle(n, d, Ms, A, Ku, hext):
    g = pb.Grace(n, d, Ms, A, Ku, 0.5, GAMMA0)
    g.set_m(random_m(n, Ms, seed=23))
    g.set_hext(hext)
    M = g.get_m()
    H = oracle_heff(M, DemagFFT(tensor_octant(*n, *d)), A, Ms, Ku, d, hext)
    t = np.sqrt((np.cross(M, H, axis=0) ** 2).sum(0)) / (Ms * np.sqrt((H ** 2).sum(0)) + 1e-30)
    assert abs(g.max_torque() - t.max()) <= 1e-4 * t.max()
    g.close()


def test_relax_single_cell_easy_axis():
    """one cell with an easy x-axis, M at 45 deg, relaxes to +-x."""
    n, d, Ms = (1, 1, 1), (2e-9, 2e-9, 2e-9), 8e5
    g = pb.Grace(n, d, Ms, 1.3e-11, 5e5, 0.02, GAMMA0)
    g.set_m(uniform_m(n, Ms, (1, 1, 0)))
    steps, t = g.relax(alpha_relax=1.0, dt=1e-13, max_steps=200000, tol=1e-6, check_every=500)
    assert t < 1e-6 and 0 < steps < 200000
    m = g.get_m()[:, 0, 0, 0] / Ms
    assert abs(abs(m[0]) - 1) < 1e-6
    assert g.steps == steps
    # alpha restored: a further step from the relaxed state keeps it relaxed
    g.step(10, 1e-13)
    assert g.max_torque() < 1e-5
    g.close()


def test_energy_decreases_while_relaxing():
    """Damped dynamics at zero field lower the Eq. (1) energy (SPEC monotonicity)."""
    n, d, Ms = (32, 16, 2), (3e-9, 3e-9, 3e-9), 8e5
    g = pb.Grace(n, d, Ms, 1.3e-11, 0.0, 1.0, GAMMA0)
    g.set_m(random_m(n, Ms, seed=3))
    prev = g.energy()["total"]
    for _ in range(5):
        g.step(20, 1e-14)
        cur = g.energy()["total"]
        assert cur < prev
        prev = cur
    g.close()


def test_virtual_ranks_energy_matches_single():
    n, d, Ms = (16, 12, 8), (1e-9, 1e-9, 1e-9), 8e5
    M = random_m(n, Ms, seed=41)
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    dist = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, virtual_ranks=4)
    for g in (ref, dist):
        g.set_m(M)
        g.set_hext((1e4, 0, -5e3))
    a, b = ref.energy(), dist.energy()
    for k in a:
        assert abs(a[k] - b[k]) <= 1e-9 * abs(a["total"]) + 1e-12 * abs(a[k]), k
    assert abs(ref.max_torque() - dist.max_torque()) <= 1e-12
    ref.close()
    dist.close()
