"""GPU (libgrace, through the C-ABI) vs the fp64 oracle, element by element.

Tolerances: real-space tensor bit-exact (BASELINE north_star);
spectral table within fp32 rounding of the oracle's rfftn at the same padding;
H_eff relative L2 <= 1e-5 per evaluation (north_star); one Euler step within
fp32 rounding of the oracle step; |M| = Ms to 1e-6; Euler precession closed
form to 1e-6.  Grids span several FFT tiles, ragged tails (non power-of-two
n, Kx not a multiple of the tile), degenerate axes (n = 1) and both step
variants (K1/K2'/K5 for nz = 1, K1..K5 otherwise).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from oracle import sp4 as osp4  # noqa: E402
from oracle.demag import DemagFFT, kernel_spectrum  # noqa: E402
from oracle.fields import heff as oracle_heff  # noqa: E402
from oracle.llg import Sim  # noqa: E402
from oracle.tensor import tensor_entry, tensor_octant  # noqa: E402
from workloads import GAMMA0, WORKLOADS, random_m, uniform_m  # noqa: E402


def relL2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---------------------------------------------------------------- tensor (setup)

OCT_CASES = [
    ((1, 1, 1), (1e-9, 1e-9, 1e-9)),
    ((1, 1, 1), (5e-9, 5e-9, 3e-9)),
    ((7, 5, 3), (1e-9, 2e-9, 3e-9)),
    ((100, 25, 1), (5e-9, 5e-9, 3e-9)),
    ((200, 50, 1), (2.5e-9, 2.5e-9, 3e-9)),
    ((70, 9, 4), (1e-9, 1e-9, 1e-9)),       # crosses the near/far cutoff (51.96 cells)
    ((16, 16, 16), (1e-9, 1e-9, 1e-9)),
]


@pytest.mark.parametrize("n,d", OCT_CASES)
def test_tensor_octant_bit_exact(n, d):
    gpu = pb.grace_tensor_octant(*n, *d)
    ora = tensor_octant(*n, *d)
    diff = np.flatnonzero(gpu.ravel() != ora.ravel())
    assert diff.size == 0, (diff[:10], gpu.ravel()[diff[:5]], ora.ravel()[diff[:5]])


@pytest.mark.parametrize("name", ["slab_1024x1024x32", "film_512x512x8"])
def test_tensor_octant_bit_exact_full_size_sampled(name):
    w = WORKLOADS[name]
    nx, ny, nz = w.n
    gpu = pb.grace_tensor_octant(nx, ny, nz, *w.d)
    rng = np.random.default_rng(5)
    pts = [(c, 0, 0, 0) for c in range(6)]
    pts += [(int(rng.integers(6)), int(rng.integers(nz)), int(rng.integers(60)), int(rng.integers(60))) for _ in range(40)]
    pts += [(int(rng.integers(6)), int(rng.integers(nz)), int(rng.integers(ny)), int(rng.integers(nx))) for _ in range(40)]
    for c, k, j, i in pts:
        assert gpu[c, k, j, i] == tensor_entry(c, i, j, k, *w.d), (c, k, j, i)


@pytest.mark.parametrize("n,d", [((7, 5, 3), (1e-9, 2e-9, 3e-9)), ((100, 25, 1), (5e-9, 5e-9, 3e-9)),
                                 ((12, 1, 9), (1e-9, 1e-9, 1e-9))])
def test_kernel_spectrum_matches_oracle_rfftn(n, d):
    g = pb.Grace(n, d, 8e5, 1.3e-11, 0.0, 0.5, GAMMA0)
    geo = g.geometry
    KS = pb.grace_kernel_spectrum(g.h)
    P = (geo["Pz"], geo["Py"], geo["Px"])
    spec = kernel_spectrum(tensor_octant(*n, *d), P)  # [6, Pz, Py, Px//2+1]
    assert np.abs(spec.imag).max() <= 1e-12 * np.abs(spec.real).max()
    want = -spec.real[:, : geo["Kzh"], : geo["Kyh"], :] / (P[0] * P[1] * P[2])
    got = KS[:, :, :, : geo["Kx"]].astype(np.float64)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 2e-7 * scale
    g.close()


@pytest.mark.parametrize("n,d", [((7, 5, 3), (1e-9, 2e-9, 3e-9)), ((100, 25, 1), (5e-9, 5e-9, 3e-9)),
                                 ((12, 1, 9), (1e-9, 1e-9, 1e-9)), ((33, 17, 20), (1e-9, 1.5e-9, 2e-9))])
def test_kernel_spectrum_fp64_matches_oracle_1e12(n, d):
    """the fp64 spectrum (before its fp32 rounding) against the oracle's
    rfftn of its own bit-identical octant at the GPU padding, within 1e-12 of the
    largest entry (different FFT algorithms: not bitwise)."""
    K64 = pb.grace_kernel_spectrum_f64(*n, *d)
    _, Kzh, Kyh, _ = K64.shape
    g = pb.Grace(n, d, 8e5, 1.3e-11, 0.0, 0.5, GAMMA0)
    geo = g.geometry
    KS = pb.grace_kernel_spectrum(g.h)
    g.close()
    P = (geo["Pz"], geo["Py"], geo["Px"])
    spec = kernel_spectrum(tensor_octant(*n, *d), P)
    want = -spec.real[:, :Kzh, :Kyh, :] / (P[0] * P[1] * P[2])
    got = K64[:, :, :, : geo["Kx"]]
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-12 * scale
    # the fp32 table is this fp64 table rounded once
    assert np.array_equal(KS[:, :, :, : geo["Kx"]], got.astype(np.float32))


# ---------------------------------------------------------------- H_eff

HEFF_CASES = [
    # n, d, Ms, A, Ku, hext
    ((1, 1, 1), (2e-9, 2e-9, 2e-9), 8e5, 1.3e-11, 5e4, (1e4, 2e4, -3e4)),
    ((7, 1, 1), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 6.2832e4, (0, 0, 0)),
    ((1, 6, 1), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),
    ((1, 1, 5), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),
    ((5, 1, 3), (2e-9, 1e-9, 1e-9), 8e5, 1.3e-11, 0.0, (1e3, 0, 0)),
    ((100, 25, 1), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, (-19576.058, 3421.831, 0)),
    ((200, 50, 1), (2.5e-9, 2.5e-9, 3e-9), 8e5, 1.3e-11, 0.0, (-28250.002, -5013.381, 0)),
    ((33, 17, 5), (1e-9, 1.5e-9, 2e-9), 1e6, 1e-11, 6.2832e4, (5e3, -5e3, 1e4)),
    ((16, 16, 16), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 6.2832e4, (0, 0, 0)),
    ((64, 48, 8), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, (0, 0, 0)),
    ((130, 3, 2), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),
    ((300, 7, 1), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),
    ((6, 5, 40), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),      # Pz = 128: unfused K3
    ((20, 300, 1), (2e-9, 1e-9, 1e-9), 8e5, 1.3e-11, 0.0, (0, 0, 0)),  # nz = 1, Py = 1024: K2/multiply/K4
    ((9, 31, 3), (1e-9, 1e-9, 1e-9), 8e5, 1.3e-11, 1e4, (0, 0, 0)),    # odd nx: scalar load/store paths
    ((4, 3, 100), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),     # Pz = 256: K3 4-column tiles
    ((3, 2, 200), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),     # Pz = 512: 8-column tiles
    ((2, 2, 300), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),     # Pz = 1024
    ((4, 2048, 2), (1e-9, 1e-9, 1e-9), 1e6, 1e-11, 0.0, (0, 0, 0)),    # Py = 4096: staged K2, partial tile
    ((16, 200, 1), (1e-9, 1e-9, 1e-9), 8e5, 1.3e-11, 0.0, (0, 0, 0)),  # nz = 1, Py = 512: K2' with smem twiddles
    ((24, 100, 1), (2e-9, 1e-9, 1e-9), 8e5, 1.3e-11, 0.0, (0, 0, 0)),  # nz = 1, Py = 256
]


@pytest.mark.parametrize("n,d,Ms,A,Ku,hext", HEFF_CASES)
def test_heff_relL2(n, d, Ms, A, Ku, hext):
    M = random_m(n, Ms, seed=hash(n) % 1000)
    g = pb.Grace(n, d, Ms, A, Ku, 0.5, GAMMA0)
    g.set_m(M)
    g.set_hext(hext)
    Hg = g.heff()
    op = DemagFFT(tensor_octant(*n, *d))
    Ho = oracle_heff(M, op, A, Ms, Ku, d, hext)
    assert relL2(Hg, Ho) <= 1e-5
    # demag alone (A = Ku = 0, no field) must also meet the bar
    g2 = pb.Grace(n, d, Ms, 0.0, 0.0, 0.5, GAMMA0)
    g2.set_m(M)
    assert relL2(g2.heff(), op(M)) <= 1e-5
    g.close()
    g2.close()


def test_heff_uniform_thin_film_aharoni_full_size():
    """Uniform z-magnetised film at BASELINE sizes: <H_z> = -Ms D_z(prism) (reading Q23)."""
    from tests.pins.aharoni import aharoni_factors

    for name in ("film_512x512x8", "slab_1024x1024x32"):
        w = WORKLOADS[name]
        g = pb.Grace(w.n, w.d, w.Ms, 0.0, 0.0, 0.5, GAMMA0)
        g.set_m(uniform_m(w.n, w.Ms, (0, 0, 1)))
        H = g.heff()
        D = aharoni_factors(w.n[0] * w.d[0], w.n[1] * w.d[1], w.n[2] * w.d[2])
        assert abs(H[2].mean() / w.Ms + D[2]) < 1e-5, (name, H[2].mean() / w.Ms, -D[2])
        assert abs(H[0].mean()) / w.Ms < 1e-6 and abs(H[1].mean()) / w.Ms < 1e-6
        g.close()


def test_heff_full_size_local_terms_sampled():
    """Slab at full size: H_eff - H_demag (exchange + anisotropy + Zeeman) at sampled cells."""
    w = WORKLOADS["slab_1024x1024x32"]
    M = random_m(w.n, w.Ms)
    hext = (1e3, -2e3, 3e3)
    g = pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    g.set_m(M)
    g.set_hext(hext)
    H = g.heff()
    g0 = pb.Grace(w.n, w.d, w.Ms, 0.0, 0.0, w.alpha, GAMMA0)
    g0.set_m(M)
    Hd = g0.heff()
    from oracle.fields import anisotropy, exchange

    rng = np.random.default_rng(3)
    nx, ny, nz = w.n
    cells = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (0, ny - 1, 5), (nx - 1, 0, nz - 1)]
    cells += [(int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))) for _ in range(26)]
    for i, j, k in cells:
        # the 3x3x3 window holds every existing neighbour of the centre cell, so the
        # Neumann stencil at the centre equals the full-grid value
        sl = (slice(None), slice(max(k - 1, 0), k + 2), slice(max(j - 1, 0), j + 2), slice(max(i - 1, 0), i + 2))
        sub = M[sl]
        ci, cj, ck = i - sl[3].start, j - sl[2].start, k - sl[1].start
        ex = exchange(sub, w.A, w.Ms, w.d)[:, ck, cj, ci]
        an = anisotropy(sub, w.Ku, w.Ms)[:, ck, cj, ci]
        want = ex + an + np.array(hext)
        got = H[:, k, j, i] - Hd[:, k, j, i]
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max() + 1e-3 * w.Ms * 1e-3, (i, j, k, got, want)
    g.close()
    g0.close()


# ---------------------------------------------------------------- Euler step

STEP_CASES = [
    ((100, 25, 1), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, 0.02, 2.5e-14, (-19576.058, 3421.831, 0)),
    ((33, 17, 5), (1e-9, 1.5e-9, 2e-9), 1e6, 1e-11, 6.2832e4, 0.5, 1e-15, (0, 0, 0)),
    ((64, 64, 8), (5e-9, 5e-9, 3e-9), 8e5, 1.3e-11, 0.0, 0.5, 1e-14, (0, 0, 0)),
    ((37, 50, 1), (2e-9, 2e-9, 3e-9), 8e5, 1.3e-11, 5e4, 0.1, 1e-14, (1e4, -2e4, 3e3)),  # nz = 1, odd nx
]


@pytest.mark.parametrize("n,d,Ms,A,Ku,alpha,dt,hext", STEP_CASES)
def test_euler_steps_match_oracle(n, d, Ms, A, Ku, alpha, dt, hext):
    M = random_m(n, Ms, seed=11)
    g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)
    g.set_m(M)
    g.set_hext(hext)
    sim = Sim(M, DemagFFT(tensor_octant(*n, *d)), Ms, A, Ku, alpha, GAMMA0, d, hext)
    # start both from the fp32-rounded state the GPU holds
    sim.M = g.get_m()
    g.step(1, dt)
    sim.euler_step(dt)
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 2e-5 * Ms
    assert relL2(Mg, sim.M) <= 1e-6
    g.step(9, dt)
    sim.run(9, dt)
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 1e-4 * Ms
    nrm = np.sqrt((Mg ** 2).sum(0))
    assert np.abs(nrm / Ms - 1).max() <= 1e-6
    np.testing.assert_allclose(g.mavg(), Mg.reshape(3, -1).mean(1) / Ms, rtol=0, atol=1e-12)
    assert g.steps == 10
    g.close()


def test_euler_precession_closed_form_single_cell():
    g0, Hm, Ms, dt = GAMMA0, 1e5, 8e5, 1e-13
    g = pb.Grace((1, 1, 1), (2e-9, 2e-9, 2e-9), Ms, 0.0, 0.0, 0.0, g0)
    M = np.zeros((3, 1, 1, 1))
    M[0] = Ms
    g.set_m(M)
    g.set_hext((0, 0, Hm))
    theta = np.arctan(g0 * Hm * dt)
    for n in (1, 10, 100, 1000):
        done = g.steps
        g.step(n - done, dt)
        want = Ms * np.array([np.cos(n * theta), np.sin(n * theta), 0.0])
        assert np.abs(g.get_m()[:, 0, 0, 0] - want).max() <= 2e-6 * Ms * max(1, n / 100)
    g.close()


def test_fixed_point_and_determinism():
    # one cell along x with the field along x: every transverse product is exactly 0
    g1 = pb.Grace((1, 1, 1), (2e-9,) * 3, 8e5, 1.3e-11, 1e4, 0.5, GAMMA0)
    M1 = uniform_m((1, 1, 1), 8e5, (1, 0, 0))
    g1.set_m(M1)
    g1.set_hext((1e5, 0, 0))
    g1.step(20, 1e-13)
    assert np.array_equal(g1.get_m(), M1.astype(np.float32).astype(np.float64))
    g1.close()
    n, d = (24, 10, 3), (2e-9, 2e-9, 2e-9)
    g = pb.Grace(n, d, 8e5, 1.3e-11, 1e4, 0.5, GAMMA0)
    M0 = random_m(n, 8e5, seed=9)
    outs = []
    for _ in range(2):
        g.set_m(M0)
        g.step(25, 1e-14)
        outs.append(g.get_m())
    assert np.array_equal(outs[0], outs[1])
    g.close()


# ---------------------------------------------------------------- errors / edge cases

def test_errors_and_nonfinite_report():
    with pytest.raises(pb.GraceError) as e:
        pb.grace_create(0, 1, 1, 1e-9, 1e-9, 1e-9, 8e5, 1e-11, 0, 0.5, GAMMA0)
    assert e.value.code == pb.GRACE_EINVAL
    with pytest.raises(pb.GraceError) as e:
        pb.grace_create(4, 4, 4, 1e-9, 1e-9, 1e-9, 8e5, 1e-11, 0, 0.5, 1.76e11)
    assert e.value.code == pb.GRACE_EINVAL
    n = (8, 4, 2)
    g = pb.Grace(n, (1e-9,) * 3, 8e5, 1e-11, 0.0, 0.5, GAMMA0)
    M = random_m(n, 8e5, seed=2)
    M[:, 1, 2, 5] = 0.0
    with pytest.raises(pb.GraceError) as e:
        g.set_m(M)
    assert e.value.code == pb.GRACE_EZEROCELL and "cell 53" in str(e.value)
    M[:, 1, 2, 5] = 1.0
    g.set_m(M)
    with pytest.raises(pb.GraceError) as e:
        g.step(1, -1e-15)
    assert e.value.code == pb.GRACE_EINVAL
    g.step(3, 1e-15)
    g.set_hext((3e38, 3e38, 3e38))
    with pytest.raises(pb.GraceError) as e:
        g.step(2, 1e-13)
    assert e.value.code == pb.GRACE_ENONFINITE
    assert pb.grace_last_nonfinite(g.h) == (3, 0)
    g.close()


def test_size_limits_unsupported_and_out_of_memory():
    """Padded lengths beyond the compiled FFT set -> GRACE_EUNSUPPORTED; a grid whose
    working set exceeds HBM (4096 x 2048 x 512: X2 alone ~207 GB) -> GRACE_ENOMEM
    with everything released, so a following create succeeds."""
    with pytest.raises(pb.GraceError) as e:
        pb.grace_create(5000, 4, 4, 1e-9, 1e-9, 1e-9, 8e5, 1e-11, 0, 0.5, GAMMA0)
    assert e.value.code == pb.GRACE_EUNSUPPORTED
    with pytest.raises(pb.GraceError) as e:
        pb.grace_create(4096, 2048, 512, 1e-9, 1e-9, 1e-9, 8e5, 1e-11, 0, 0.5, GAMMA0)
    assert e.value.code == pb.GRACE_ENOMEM
    g = pb.Grace((8, 8, 8), (1e-9,) * 3, 8e5, 1e-11, 0.0, 0.5, GAMMA0)
    g.step(2, 1e-14)
    g.close()


# ---------------------------------------------------------------- SP4 trajectories

def _golden(name):
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", f"{name}_oracle.csv")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (scripts/gen_sp4_golden.py)")
    return np.loadtxt(path)


@pytest.mark.parametrize("name,tmax", [("sp4_field1_coarse", 1.01e-9), ("sp4_field2_refined", 0.601e-9)])
def test_sp4_trajectory_within_1e3(name, tmax):
    gold = _golden(name)
    cfg = osp4.CONFIGS[name]
    nx, ny, nz = cfg["n"]
    g = pb.Grace(cfg["n"], cfg["d"], osp4.MS, osp4.A_EX, 0.0, 1.0, osp4.GAMMA0)
    g.set_m(uniform_m(cfg["n"], osp4.MS, (1, 1, 1)))
    steps, dt = cfg["relax"]
    g.step(steps, dt)
    g.set_alpha(0.02)
    g.set_hext(osp4.field_Am(cfg["field"]))
    nsteps, dt = cfg["run"]
    every = cfg["every"]
    rows = [g.mavg()]
    for _ in range(nsteps // every):
        g.step(every, dt)
        rows.append(g.mavg())
    rows = np.array(rows)
    t = np.arange(len(rows)) * every * dt
    assert np.allclose(t, gold[:, 0], rtol=1e-6)
    sel = t <= tmax
    dev = np.abs(rows[sel] - gold[sel, 1:]).max()
    assert dev <= 1e-3, dev
    g.close()


@pytest.mark.parametrize("name,nsample", [("film_512x512x8", 5), ("slab_1024x1024x32", 2)])
def test_heff_full_size_sampled_direct_sum(name, nsample):
    """BASELINE film 512x512x8 and slab 1024x1024x32 at full size (the bench's launch
    configuration): H_demag at sampled cells by the O(N) direct sum over every source
    cell (oracle tensor, one observer at a time) vs the GPU FFT path."""
    w = WORKLOADS[name]
    nx, ny, nz = w.n
    M = random_m(w.n, w.Ms, seed=77)
    g = pb.Grace(w.n, w.d, w.Ms, 0.0, 0.0, w.alpha, GAMMA0)
    g.set_m(M)
    H = g.heff()
    g.close()
    oct_ = tensor_octant(nx, ny, nz, *w.d)
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    Mf = M.reshape(3, -1)
    rng = np.random.default_rng(8)
    cells = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (nx // 2, ny // 2, nz // 2)]
    cells += [(int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))) for _ in range(nsample)]
    for i, j, k in cells:
        di, dj, dk = (i - I).ravel(), (j - J).ravel(), (k - K).ravel()
        v = oct_[:, np.abs(dk), np.abs(dj), np.abs(di)]
        sx, sy, sz = np.where(di < 0, -1.0, 1.0), np.where(dj < 0, -1.0, 1.0), np.where(dk < 0, -1.0, 1.0)
        nxy, nxz, nyz = v[1] * sx * sy, v[2] * sx * sz, v[4] * sy * sz
        want = -np.array([(v[0] * Mf[0] + nxy * Mf[1] + nxz * Mf[2]).sum(),
                          (nxy * Mf[0] + v[3] * Mf[1] + nyz * Mf[2]).sum(),
                          (nxz * Mf[0] + nyz * Mf[1] + v[5] * Mf[2]).sum()])
        got = H[:, k, j, i]
        # fp32 FFT of a 16.8M-point padded grid: error relative to the field scale Ms
        assert np.abs(got - want).max() <= 2e-5 * w.Ms, (i, j, k, got, want)


def test_field_schedule_steps_and_heff_match_oracle():
    """Paper Sec. 5 / SPEC S:L182-187 field schedule: the GPU steps and H_eff at a
    scheduled time against the oracle Sim with the same schedule."""
    n, d, Ms, A, Ku, alpha, dt = (24, 10, 3), (2e-9, 2e-9, 3e-9), 8e5, 1.3e-11, 1e4, 0.1, 5e-14
    hext, h0, sch = (2e3, 0.0, 0.0), (0.0, 3e5, -2e5), (2, 5, 9)
    M = random_m(n, Ms, seed=13)
    g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)
    g.set_m(M)
    g.set_hext(hext)
    g.set_field_schedule(h0, *sch)
    sim = Sim(g.get_m(), DemagFFT(tensor_octant(*n, *d)), Ms, A, Ku, alpha, GAMMA0, d, hext, schedule=(h0, *sch))
    for k in range(12):
        if k in (0, 3, 6, 9):
            Hg, Ho = g.heff(), sim.heff()
            assert relL2(Hg, Ho) <= 1e-5, k
        g.step(1, dt)
        sim.euler_step(dt)
        assert np.abs(g.get_m() - sim.M).max() <= 1e-4 * Ms, k
    with pytest.raises(pb.GraceError):
        g.set_field_schedule(h0, 5, 4, 9)
    g.close()


# ---------------------------------------------------------------- Heun (RK2)

def test_heun_precession_closed_form_single_cell():
    """Heun + renormalisation rotates by the exact angle of tests/test_oracle_fields_llg.py."""
    g0, Hm, Ms, dt = GAMMA0, 1e5, 8e5, 1e-13
    phi = g0 * Hm * dt
    th = np.arctan(phi)
    psi = np.arctan2(0.5 * phi * (1 + np.cos(th)), 1 - 0.5 * phi * np.sin(th))
    g = pb.Grace((1, 1, 1), (2e-9, 2e-9, 2e-9), Ms, 0.0, 0.0, 0.0, g0)
    g.set_integrator("heun")
    M = np.zeros((3, 1, 1, 1))
    M[0] = Ms
    g.set_m(M)
    g.set_hext((0, 0, Hm))
    for n in (1, 10, 100, 1000):
        g.step(n - g.steps, dt)
        want = Ms * np.array([np.cos(n * psi), np.sin(n * psi), 0.0])
        assert np.abs(g.get_m()[:, 0, 0, 0] - want).max() <= 2e-6 * Ms * max(1, n / 100)
    g.close()


@pytest.mark.parametrize("n,d", [((24, 10, 3), (2e-9, 2e-9, 3e-9)), ((100, 25, 1), (5e-9, 5e-9, 3e-9))])
def test_heun_steps_match_oracle(n, d):
    Ms, A, Ku, alpha, dt = 8e5, 1.3e-11, 1e4, 0.1, 5e-14
    hext, h0, sch = (2e3, 0.0, 0.0), (0.0, 3e5, -2e5), (2, 4, 8)
    g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)
    g.set_integrator("heun")
    g.set_m(random_m(n, Ms, seed=19))
    g.set_hext(hext)
    g.set_field_schedule(h0, *sch)
    sim = Sim(g.get_m(), DemagFFT(tensor_octant(*n, *d)), Ms, A, Ku, alpha, GAMMA0, d, hext, schedule=(h0, *sch))
    g.step(1, dt)
    sim.heun_step(dt)
    assert np.abs(g.get_m() - sim.M).max() <= 2e-5 * Ms
    g.step(9, dt)
    sim.run(9, dt, "heun")
    Mg = g.get_m()
    assert np.abs(Mg - sim.M).max() <= 1e-4 * Ms
    assert relL2(Mg, sim.M) <= 1e-5
    assert g.steps == 10
    # switching back to Euler continues from the same state
    g.set_integrator("euler")
    g.step(2, dt)
    sim.run(2, dt)
    assert np.abs(g.get_m() - sim.M).max() <= 1e-4 * Ms
    with pytest.raises(pb.GraceError):
        g.set_integrator(7)
    g.close()


def test_host_fp32_set_get_m():
    """grace_set_m_f32 / grace_get_m_f32 (12 B/cell each way) = the fp64 calls."""
    n = (33, 17, 5)
    M = random_m(n, 8e5, seed=81)
    g = pb.Grace(n, (1e-9,) * 3, 8e5, 1.3e-11, 0.0, 0.5, GAMMA0)
    g.set_m(M)
    a = g.get_m()
    pb.grace_set_m_f32(g.h, np.ascontiguousarray(M, dtype=np.float32))
    b = np.empty((3,) + n[::-1], dtype=np.float32)
    pb.grace_get_m_f32(g.h, b)
    assert np.abs(a - b).max() <= 4e-7 * 8e5  # fp32 vs fp64 normalisation: a few ulps
    M32 = np.ascontiguousarray(M, dtype=np.float32)
    M32[:, 1, 2, 3] = 0.0
    with pytest.raises(pb.GraceError) as e:
        pb.grace_set_m_f32(g.h, M32)
    assert e.value.code == pb.GRACE_EZEROCELL
    g.close()
