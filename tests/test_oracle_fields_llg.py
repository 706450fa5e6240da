"""Pins of oracle/fields.py, oracle/llg.py and oracle/energy.py.

* exchange: exact zero for uniform M; SPEC's 3x1x1 hand stencil
  (S:L197); Neumann DCT-II modes are exact eigenvectors with eigenvalue
  -(2 - 2 cos(pi m/n))/Delta^2 (textbook discrete Laplacian); self-adjoint;
* anisotropy closed forms;
* fields = -1/(mu0 V) dE/dM of the separately written Eq. (1) energy, per term,
  by central differences (S:L225, S:L498 acceptance 5);
* Eq. (3) sign and magnitude examples;
* Euler + renormalisation: exact discrete precession map theta = atan(gamma0 H dt)
  for one cubic cell (its demag field is parallel to M); |M| = Ms, fixed
  points, damped energy decrease.
"""
import numpy as np
import pytest

from oracle import MU0
from oracle.demag import DemagFFT
from oracle.energy import energy
from oracle.fields import anisotropy, exchange, heff
from oracle.llg import NonFinite, Sim, llg_rhs
from oracle.tensor import tensor_octant
from workloads import GAMMA0, random_m

RNG = np.random.default_rng(7)
MS, A = 8e5, 1.3e-11


def test_exchange_uniform_is_exactly_zero():
    M = np.empty((3, 3, 4, 5))
    M[:] = np.array([0.3, -0.5, 0.81])[:, None, None, None] * MS
    assert np.all(exchange(M, A, MS, (1e-9, 2e-9, 3e-9)) == 0.0)


def test_exchange_hand_stencil_3x1x1():
    d = 2e-9
    M = np.zeros((3, 1, 1, 3))
    M[0, 0, 0, :] = MS
    M[:, 0, 0, 1] = (0.0, MS, 0.0)
    H = exchange(M, A, MS, (d, d, d))
    c = 2 * A / (MU0 * MS * MS * d * d)
    np.testing.assert_allclose(H[:, 0, 0, 1], c * np.array([2 * MS, -2 * MS, 0]), rtol=1e-14)
    np.testing.assert_allclose(H[:, 0, 0, 0], c * np.array([-MS, MS, 0]), rtol=1e-14)
    np.testing.assert_allclose(H[:, 0, 0, 2], c * np.array([-MS, MS, 0]), rtol=1e-14)


@pytest.mark.parametrize("axis,n,m", [(3, 16, 3), (2, 9, 4), (1, 5, 1)])
def test_exchange_neumann_dct_eigenmodes(axis, n, m):
    shape = [3, 2, 3, 4]
    shape[axis] = n
    d = (1e-9, 2e-9, 3e-9)
    delta = {3: d[0], 2: d[1], 1: d[2]}[axis]
    i = np.arange(n)
    mode = np.cos(np.pi * m * (i + 0.5) / n)
    sh = [1, 1, 1, 1]
    sh[axis] = n
    M = np.zeros(shape)
    M[1] = MS * mode.reshape(sh[1:])
    H = exchange(M, A, MS, d)
    lam = -(2.0 - 2.0 * np.cos(np.pi * m / n)) / (delta * delta)
    c = 2 * A / (MU0 * MS * MS)
    np.testing.assert_allclose(H[1], c * lam * M[1], rtol=1e-9, atol=1e-12 * abs(c * lam) * MS)
    assert np.all(H[0] == 0) and np.all(H[2] == 0)


def test_exchange_self_adjoint():
    d = (1e-9, 1.5e-9, 2e-9)
    M1 = RNG.standard_normal((3, 3, 4, 5))
    M2 = RNG.standard_normal((3, 3, 4, 5))
    a = (M1 * exchange(M2, A, 1.0, d)).sum()
    b = (M2 * exchange(M1, A, 1.0, d)).sum()
    assert abs(a - b) <= 1e-12 * abs(a)


def test_anisotropy_closed_forms():
    Ku = 6.2832e4
    Ms = 1e6
    Hk = 2 * Ku / (MU0 * Ms)
    M = np.zeros((3, 1, 1, 2))
    M[:, 0, 0, 0] = (Ms, 0, 0)
    M[:, 0, 0, 1] = (0, Ms / np.sqrt(2), Ms / np.sqrt(2))
    H = anisotropy(M, Ku, Ms)
    np.testing.assert_allclose(H[:, 0, 0, 0], (Hk, 0, 0), rtol=1e-14)
    assert np.all(H[:, 0, 0, 1] == 0)
    assert np.all(anisotropy(M, 0.0, Ms) == 0)


def test_fields_are_energy_gradient():
    nx, ny, nz = 4, 4, 4
    d = (2e-9, 3e-9, 2.5e-9)
    Ms, Aex, Ku = 8e5, 1.3e-11, 5e4
    hext = (1e4, -2e4, 3e4)
    op = DemagFFT(tensor_octant(nx, ny, nz, *d))
    M = RNG.standard_normal((3, nz, ny, nx))
    M = Ms * M / np.sqrt((M * M).sum(0))
    V = d[0] * d[1] * d[2]
    # per term: (A, Ku, demag on, hext)
    terms = {
        "exchange": dict(A=Aex, Ku=0.0, dem=False, h=(0, 0, 0)),
        "anisotropy": dict(A=0.0, Ku=Ku, dem=False, h=(0, 0, 0)),
        "demag": dict(A=0.0, Ku=0.0, dem=True, h=(0, 0, 0)),
        "zeeman": dict(A=0.0, Ku=0.0, dem=False, h=hext),
        "all": dict(A=Aex, Ku=Ku, dem=True, h=hext),
    }
    zero = lambda M_: np.zeros_like(M_)  # noqa: E731
    for name, t in terms.items():
        dem = op if t["dem"] else zero
        H = heff(M, dem, t["A"], Ms, t["Ku"], d, t["h"])
        for (a, k, j, i) in [(0, 1, 2, 3), (1, 0, 0, 0), (2, 3, 1, 2), (0, 3, 3, 3)]:
            hstep = 1e-3 * Ms
            Mp, Mm = M.copy(), M.copy()
            Mp[a, k, j, i] += hstep
            Mm[a, k, j, i] -= hstep
            Ep, _ = energy(Mp, dem, t["A"], Ms, t["Ku"], d, t["h"])
            Em, _ = energy(Mm, dem, t["A"], Ms, t["Ku"], d, t["h"])
            fd = -(Ep - Em) / (2 * hstep) / (MU0 * V)
            scale = np.abs(H).max()
            assert abs(fd - H[a, k, j, i]) <= 1e-6 * scale, (name, a, fd, H[a, k, j, i])


def test_llg_signs_and_magnitudes():
    g0, Hm, Ms = 2.211e5, 1e5, 8e5
    M = np.array([Ms, 0, 0])[:, None]
    H = np.array([0, 0, Hm])[:, None]
    np.testing.assert_allclose(llg_rhs(M, H, 0.0, g0, Ms)[:, 0], (0, g0 * Ms * Hm, 0), rtol=1e-15)
    assert np.all(llg_rhs(M, 3.0 * M, 0.3, g0, Ms) == 0)
    alpha = 0.1
    H = np.array([0, Hm, 0])[:, None]
    r = llg_rhs(M, H, alpha, g0, Ms)[:, 0]
    a = g0 / (1 + alpha ** 2)
    np.testing.assert_allclose(r, (0, alpha * a * Ms * Hm, -a * Ms * Hm), rtol=1e-14)
    Mr = RNG.standard_normal((3, 50))
    Hr = RNG.standard_normal((3, 50)) * 1e5
    r = llg_rhs(Mr, Hr, 0.3, g0, 1.0)
    assert np.abs((Mr * r).sum(0)).max() < 1e-9 * np.abs(r).max()


def _one_cube(Ms=8e5):
    return DemagFFT(tensor_octant(1, 1, 1, 2e-9, 2e-9, 2e-9))


@pytest.mark.parametrize("dt", [1e-13, 1e-14])
def test_euler_exact_precession_map(dt):
    g0, Hm, Ms = 2.211e5, 1e5, 8e5
    M0 = np.zeros((3, 1, 1, 1))
    M0[0] = Ms
    sim = Sim(M0, _one_cube(), Ms, 0.0, 0.0, 0.0, g0, (2e-9,) * 3, hext=(0, 0, Hm))
    theta = np.arctan(g0 * Hm * dt)
    for n in range(1, 501):
        sim.euler_step(dt)
        if n % 50 == 0:
            want = Ms * np.array([np.cos(n * theta), np.sin(n * theta), 0.0])
            np.testing.assert_allclose(sim.M[:, 0, 0, 0], want, rtol=0, atol=1e-12 * Ms)
    # Larmor period T = 2 pi (1+alpha^2)/(gamma0 H) is the dt -> 0 limit (reading Q1)
    T = 2 * np.pi / (g0 * Hm)
    Td = 2 * np.pi * dt / theta
    x = g0 * Hm * dt
    assert abs(Td - T) / T <= x * x / 3 * 1.01


def test_norm_fixed_point_and_damped_energy():
    nx, ny, nz = 6, 5, 2
    d = (3e-9, 3e-9, 3e-9)
    op = DemagFFT(tensor_octant(nx, ny, nz, *d))
    M = RNG.standard_normal((3, nz, ny, nx))
    M = MS * M / np.sqrt((M * M).sum(0))
    sim = Sim(M, op, MS, A, 1e4, 0.5, 2.211e5, d, hext=(1e4, 0, 0))
    E0, _ = energy(sim.M, op, A, MS, 1e4, d, sim.hext)
    for _ in range(30):
        sim.euler_step(2e-14)
        n = np.sqrt((sim.M ** 2).sum(0))
        assert np.abs(n / MS - 1).max() < 1e-12
        E1, _ = energy(sim.M, op, A, MS, 1e4, d, sim.hext)
        assert E1 <= E0 + 1e-12 * abs(E0)
        E0 = E1
    # fixed point: uniform M along x in a cube with H_ext along x
    M = np.zeros((3, 1, 1, 1))
    M[0] = MS
    s2 = Sim(M, _one_cube(), MS, A, 1e4, 0.5, 2.211e5, (2e-9,) * 3, hext=(5e4, 0, 0))
    s2.run(10, 1e-13)
    assert np.array_equal(s2.M, M)


def test_nonfinite_abort_reports_step_and_cell():
    M = np.zeros((3, 1, 1, 2))
    M[0] = MS
    op = DemagFFT(tensor_octant(2, 1, 1, 2e-9, 2e-9, 2e-9))
    sim = Sim(M, op, MS, A, 0.0, 0.1, 2.211e5, (2e-9,) * 3, hext=(0, np.inf, 0))
    with pytest.raises(NonFinite) as e:
        sim.euler_step(1e-13)
    assert e.value.step == 0 and e.value.cell == 0


# ---------------------------------------------------------------- field schedule

def test_schedule_amplitude_piecewise_definition():
    """0 before start, H0 in [start, decay), linear ramp to 0
    across [decay, stop), 0 at and after stop (values written out by hand)."""
    from oracle.fields import schedule_amplitude as amp
    s, d, e = 10, 20, 30
    assert [amp(k, s, d, e) for k in (0, 9)] == [0.0, 0.0]
    assert [amp(k, s, d, e) for k in (10, 15, 19)] == [1.0, 1.0, 1.0]
    assert amp(20, s, d, e) == 1.0 and amp(25, s, d, e) == 0.5 and amp(29, s, d, e) == pytest.approx(0.1)
    assert [amp(k, s, d, e) for k in (30, 31, 10 ** 9)] == [0.0, 0.0, 0.0]
    assert amp(5, 5, 5, 5) == 0.0               # empty window: never on
    assert amp(5, 5, 5, 6) == 1.0               # one-step ramp starts at full amplitude
    assert amp(7, 5, 9, 9) == 1.0 and amp(9, 5, 9, 9) == 0.0  # no ramp: a step switch-off
    with pytest.raises(ValueError):
        amp(0, 3, 2, 4)


def test_sim_schedule_enters_zeeman_only():
    """The scheduled field adds amplitude(k) H0 to H_ext at step k and nothing else:
    H_eff(step k) - H_eff(no schedule) is that uniform vector."""
    n, d = (4, 3, 2), (1e-9, 1e-9, 1e-9)
    M = random_m(n, 8e5, seed=2)
    op = DemagFFT(tensor_octant(*n, *d))
    base = Sim(M, op, 8e5, 1.3e-11, 1e4, 0.1, GAMMA0, d, (1e3, 0, 0))
    sch = Sim(M, op, 8e5, 1.3e-11, 1e4, 0.1, GAMMA0, d, (1e3, 0, 0), schedule=((0, 2e4, -4e4), 1, 2, 6))
    for k, a in ((0, 0.0), (1, 1.0), (2, 1.0), (4, 0.5), (6, 0.0)):
        sch.step_count = k
        diff = sch.heff() - base.heff()
        for q, h0 in enumerate((0, 2e4, -4e4)):
            np.testing.assert_allclose(diff[q], a * h0, rtol=0, atol=1e-9 * 4e4)


# ---------------------------------------------------------------- Heun (RK2)

def heun_precession_angle(phi):
    """Exact rotation per Heun + renormalisation step of a unit vector precessing
    (alpha = 0) about a perpendicular field, phi = gamma0 H dt: the predictor
    lands at theta = atan(phi); M + dt (f0 + f1)/2 = (1 - phi sin(theta)/2,
    phi (1 + cos(theta))/2) in the rotation plane (derived by hand)."""
    theta = np.arctan(phi)
    return np.arctan2(0.5 * phi * (1 + np.cos(theta)), 1 - 0.5 * phi * np.sin(theta))


@pytest.mark.parametrize("dt", [1e-13, 1e-14])
def test_heun_exact_precession_map(dt):
    g0, Hm, Ms = 2.211e5, 1e5, 8e5
    M0 = np.zeros((3, 1, 1, 1))
    M0[0] = Ms
    sim = Sim(M0, _one_cube(), Ms, 0.0, 0.0, 0.0, g0, (2e-9,) * 3, hext=(0, 0, Hm))
    psi = heun_precession_angle(g0 * Hm * dt)
    for n in range(1, 301):
        sim.heun_step(dt)
        if n % 50 == 0:
            want = Ms * np.array([np.cos(n * psi), np.sin(n * psi), 0.0])
            np.testing.assert_allclose(sim.M[:, 0, 0, 0], want, rtol=0, atol=1e-12 * Ms)


def test_heun_second_order_vs_euler_first_order():
    """Global error at fixed T vs the exact Larmor rotation: halving dt cuts it ~4x
    for Heun, ~2x for Euler (a random multi-cell case through the full H_eff)."""
    n, d, Ms = (4, 3, 2), (3e-9, 3e-9, 3e-9), 8e5
    M0 = RNG.standard_normal((3,) + n[::-1])
    M0 *= Ms / np.sqrt((M0 * M0).sum(0))  # on the sphere: the first renormalisation is not a jump
    op = DemagFFT(tensor_octant(*n, *d))

    def run(method, dt, steps):
        s = Sim(M0, op, Ms, 1.3e-11, 2e4, 0.05, 2.211e5, d, hext=(1e4, 0, 5e4))
        s.run(steps, dt, method)
        return s.M

    T, base = 2e-12, 400
    ref = run("heun", T / (base * 16), base * 16)
    err = {m: [np.abs(run(m, T / (base * k), base * k) - ref).max() for k in (1, 2)] for m in ("euler", "heun")}
    assert 3.5 < err["heun"][0] / err["heun"][1] < 4.5, err
    assert 1.7 < err["euler"][0] / err["euler"][1] < 2.3, err


# ---------------------------------------------------------------- adaptive steps

def test_adaptive_single_cell_precession_closed_forms():
    """One cube cell, alpha = 0, H perpendicular to M (its demag field is parallel to M):
    the Euler attempt rotates by atan(phi) and the Heun one by psi(phi) (the exact maps
    pinned above), phi = gamma0 H dt, so the error estimate of an attempt of step dt is
    exactly 2 sin(|psi - atan(phi)|/2), and the accepted steps rotate by the sum of psi."""
    g0, Hm, Ms = 2.211e5, 1e5, 8e5
    M0 = np.zeros((3, 1, 1, 1))
    M0[0] = Ms
    sim = Sim(M0, _one_cube(), Ms, 0.0, 0.0, 0.0, g0, (2e-9,) * 3, hext=(0, 0, Hm))
    tol, T = 1e-5, 3e-11
    log, dt_next = sim.adaptive_run(T, 1e-15, tol)
    ang = 0.0
    for t, h, err, ok in log:
        phi = g0 * Hm * h
        want = 2.0 * np.sin(abs(heun_precession_angle(phi) - np.arctan(phi)) / 2.0)
        assert abs(err - want) <= 1e-12, (h, err, want)
        assert ok == (err <= tol)
        if ok:
            ang += heun_precession_angle(phi)
    acc = [x for x in log if x[3]]
    assert abs(sum(x[1] for x in acc) - T) <= 1e-9 * T  # lands on T
    assert any(not x[3] for x in log) or len(acc) == len(log)
    np.testing.assert_allclose(sim.M[:, 0, 0, 0], Ms * np.array([np.cos(ang), np.sin(ang), 0.0]), rtol=0,
                               atol=1e-12 * Ms)
    # the controller grows a tiny first step and then runs near the tolerance
    assert acc[-2][2] > 0.1 * tol and max(x[2] for x in acc) <= tol
    assert dt_next > 0


def test_adaptive_tolerance_controls_the_global_error():
    """Multi-cell case through the full H_eff: the error at a fixed time against a
    fine fixed-step Heun reference falls with the tolerance, and a tighter
    tolerance takes more steps."""
    n, d, Ms = (4, 3, 2), (3e-9, 3e-9, 3e-9), 8e5
    M0 = RNG.standard_normal((3,) + n[::-1])
    M0 *= Ms / np.sqrt((M0 * M0).sum(0))
    op = DemagFFT(tensor_octant(*n, *d))
    T = 2e-12
    ref = Sim(M0, op, Ms, 1.3e-11, 2e4, 0.05, 2.211e5, d, hext=(1e4, 0, 5e4))
    ref.run(6400, T / 6400, "heun")
    res = []
    for tol in (1e-3, 1e-4, 1e-5):
        s = Sim(M0, op, Ms, 1.3e-11, 2e4, 0.05, 2.211e5, d, hext=(1e4, 0, 5e4))
        log, _ = s.adaptive_run(T, 1e-16, tol)
        res.append((np.abs(s.M - ref.M).max() / Ms, sum(1 for x in log if x[3])))
        assert np.abs(np.sqrt((s.M ** 2).sum(0)) / Ms - 1).max() <= 1e-12
    assert res[0][0] > res[1][0] > res[2][0], res
    assert res[0][1] < res[1][1] < res[2][1], res
    assert res[2][0] < 1e-4, res
