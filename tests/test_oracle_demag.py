"""Pins of oracle/demag.py: FFT convolution == O(N^2) sum, plus physics identities.

* S:L139, S:L494 (acceptance 1): FFT path equals the direct sum on small grids;
* BASELINE north_star: "O(N^2) brute-force demag summation equals the FFT
  convolution on <=8^3 grids";
* padding independence (reading Q9): 2n and power-of-two padding agree;
* Aharoni whole-prism identity: mean over cells of H for uniform M along a is
  -Ms D_a(prism) (closed form in tests/pins/aharoni.py) -- the north_star's
  "uniformly z-magnetised thin film gives H_demag ~ -Ms z" made exact (Q23);
* linearity, reciprocity, non-negative self energy.
"""
import numpy as np
import pytest

from oracle.demag import DemagFFT, demag_brute, demag_fft
from oracle.tensor import tensor_octant
from tests.pins.aharoni import aharoni_factors

RNG = np.random.default_rng(20240601)


@pytest.mark.parametrize("n,d", [((2, 2, 2), (1e-9, 1e-9, 1e-9)), ((4, 4, 4), (1e-9, 1e-9, 1e-9)),
                                 ((5, 3, 2), (2e-9, 1e-9, 3e-9)), ((8, 8, 8), (5e-9, 5e-9, 3e-9)),
                                 ((7, 1, 1), (1e-9, 1e-9, 1e-9)), ((6, 5, 1), (5e-9, 5e-9, 3e-9))])
def test_fft_equals_brute_force(n, d):
    nx, ny, nz = n
    o = tensor_octant(nx, ny, nz, *d)
    for _ in range(3):
        M = RNG.standard_normal((3, nz, ny, nx))
        Hb = demag_brute(M, o)
        Hf = demag_fft(M, o)
        assert np.linalg.norm(Hf - Hb) <= 1e-10 * np.linalg.norm(Hb)


def test_padding_independence():
    nx, ny, nz = 6, 5, 3
    o = tensor_octant(nx, ny, nz, 1e-9, 1e-9, 1e-9)
    M = RNG.standard_normal((3, nz, ny, nx))
    H1 = demag_fft(M, o)                     # 2n: (6, 10, 12)
    H2 = demag_fft(M, o, P=(8, 16, 16))      # power of two >= 2n - 1
    H3 = demag_fft(M, o, P=(5, 9, 11))       # minimal 2n - 1
    assert np.linalg.norm(H2 - H1) <= 1e-12 * np.linalg.norm(H1)
    assert np.linalg.norm(H3 - H1) <= 1e-12 * np.linalg.norm(H1)


def test_single_cell_self_demag():
    o = tensor_octant(1, 1, 1, 1e-9, 1e-9, 1e-9)
    for a in range(3):
        M = np.zeros((3, 1, 1, 1))
        M[a] = 8e5
        H = demag_fft(M, o)
        want = np.zeros(3)
        want[a] = -8e5 / 3.0
        np.testing.assert_allclose(H[:, 0, 0, 0], want, rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("n,d,tol", [((8, 4, 2), (2e-9, 3e-9, 1e-9), 1e-12),
                                     ((100, 25, 1), (5e-9, 5e-9, 3e-9), 1e-6),
                                     ((64, 64, 4), (5e-9, 5e-9, 3e-9), 1e-6)])
def test_whole_prism_mean_field_aharoni(n, d, tol):
    nx, ny, nz = n
    o = tensor_octant(nx, ny, nz, *d)
    op = DemagFFT(o)
    D = aharoni_factors(nx * d[0], ny * d[1], nz * d[2])
    Ms = 8e5
    for a in range(3):
        M = np.zeros((3, nz, ny, nx))
        M[a] = Ms
        H = op(M)
        assert abs(H[a].mean() / Ms + D[a]) < tol, (a, H[a].mean() / Ms, -D[a])
        others = [b for b in range(3) if b != a]
        for b in others:
            assert abs(H[b].mean()) / Ms < 1e-10


def test_linearity_reciprocity_energy():
    nx, ny, nz = 7, 6, 3
    o = tensor_octant(nx, ny, nz, 3e-9, 2e-9, 1e-9)
    op = DemagFFT(o)
    M1 = RNG.standard_normal((3, nz, ny, nx))
    M2 = RNG.standard_normal((3, nz, ny, nx))
    H1, H2 = op(M1), op(M2)
    H12 = op(2.0 * M1 - 3.0 * M2)
    assert np.linalg.norm(H12 - (2.0 * H1 - 3.0 * H2)) <= 1e-10 * np.linalg.norm(H12)
    r1, r2 = (M1 * H2).sum(), (M2 * H1).sum()
    assert abs(r1 - r2) <= 1e-9 * abs(r1)
    for _ in range(5):
        M = RNG.standard_normal((3, nz, ny, nx))
        assert -0.5 * (M * op(M)).sum() >= 0.0


def test_demagfft_workers_same_result():
    """The all-core CPU baseline (scipy.fft, workers=k) computes the same convolution."""
    import numpy as np

    from oracle.demag import DemagFFT
    from oracle.tensor import tensor_octant
    from workloads import random_m

    n, d = (12, 10, 6), (1e-9, 2e-9, 3e-9)
    oct_ = tensor_octant(*n, *d)
    M = random_m(n, 8e5, seed=4)
    a = DemagFFT(oct_)(M)
    b = DemagFFT(oct_, workers=4)(M)
    assert np.abs(a - b).max() <= 1e-9 * np.abs(a).max()
