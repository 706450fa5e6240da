"""Demagnetising field H_demag = -N * M, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L55 (Sec. 3): "the demagnetization field is actually the convolution of
magnetizations and demagnetization tensor ... the computation time can be
reduced to O(N log N) by applying the discrete convolution theorem and FFT.
Non-periodic boundary conditions can be used by adapting the zero-padding
method".  Both routes are here: the O(N^2) direct sum the paper contrasts with
 and the zero-padded FFT convolution (padding 2n per
axis and singleton axes unpadded; 1/(padded size) applied once on the
inverse).

Arrays are SoA ``M[3, nz, ny, nx]`` in A/m, x fastest.
"""
import numpy as np



def demag_brute(M, oct_):
    """H_a(r) = -sum_{r'} sum_b N_ab(r - r') M_b(r'), the O(N^2) direct sum.

    One observer at a time; the sum over sources is a plain dot product over
    the tensor fetched from the octant by parity.
    """
    _, nz, ny, nx = M.shape
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    K, J, I = K.ravel(), J.ravel(), I.ravel()
    Mf = M.reshape(3, -1)
    H = np.zeros((3, K.size), dtype=np.float64)
    for o in range(K.size):
        di, dj, dk = I[o] - I, J[o] - J, K[o] - K
        v = oct_[:, np.abs(dk), np.abs(dj), np.abs(di)]
        sx = np.where(di < 0, -1.0, 1.0)
        sy = np.where(dj < 0, -1.0, 1.0)
        sz = np.where(dk < 0, -1.0, 1.0)
        nxx, nxy, nxz, nyy, nyz, nzz = v[0], v[1] * sx * sy, v[2] * sx * sz, v[3], v[4] * sy * sz, v[5]
        H[0, o] = -(nxx * Mf[0] + nxy * Mf[1] + nxz * Mf[2]).sum()
        H[1, o] = -(nxy * Mf[0] + nyy * Mf[1] + nyz * Mf[2]).sum()
        H[2, o] = -(nxz * Mf[0] + nyz * Mf[1] + nzz * Mf[2]).sum()
    return H.reshape(M.shape)


def _pad(n, P=None):
    return (2 * n if n > 1 else 1) if P is None else P


def circulant(oct_, comp, P):
    """Circulant embedding A[d mod P] = N_comp(d) for |d| < n, zeros elsewhere.

    P = (Pz, Py, Px) with P_a >= 2 n_a - 1 (or 1 when n_a = 1).  Signs of the
    odd components by parity.
    """
    _, nz, ny, nx = oct_.shape
    Pz, Py, Px = P
    A = np.zeros((Pz, Py, Px), dtype=np.float64)
    odd = {0: (), 1: (0, 1), 2: (0, 2), 3: (), 4: (1, 2), 5: ()}[comp]
    for sk in ((1, -1) if nz > 1 else (1,)):
        for sj in ((1, -1) if ny > 1 else (1,)):
            for si in ((1, -1) if nx > 1 else (1,)):
                sgn = 1.0
                for ax, s in zip((0, 1, 2), (si, sj, sk)):
                    if ax in odd:
                        sgn *= s
                ii = (si * np.arange(nx)) % Px
                jj = (sj * np.arange(ny)) % Py
                kk = (sk * np.arange(nz)) % Pz
                A[np.ix_(kk, jj, ii)] = sgn * oct_[comp]
    return A


def kernel_spectrum(oct_, P):
    """rfftn of the six circulant components at padding P (complex, [6,Pz,Py,Px//2+1])."""
    return np.stack([np.fft.rfftn(circulant(oct_, c, P)) for c in range(6)])


_PAIRS = ((0, 1, 2), (1, 3, 4), (2, 4, 5))  # row a of N: components (a,x), (a,y), (a,z)


def demag_fft(M, oct_, P=None):
    """Zero-padded FFT convolution: H_a = irfftn(-sum_b rfftn(A_ab) rfftn(M_b))[:nz,:ny,:nx].

    Default padding is exactly (2nz, 2ny, 2nx) with singleton axes unpadded
    (S:L112).  numpy's irfftn applies the 1/(PxPyPz) once.
    """
    _, nz, ny, nx = M.shape
    if P is None:
        P = (_pad(nz), _pad(ny), _pad(nx))
    Ns = kernel_spectrum(oct_, P)
    Mh = [np.fft.rfftn(M[b], s=P, axes=(0, 1, 2)) for b in range(3)]
    H = np.empty((3, nz, ny, nx), dtype=np.float64)
    for a in range(3):
        acc = np.zeros_like(Mh[0])
        for b in range(3):
            acc = acc + Ns[_PAIRS[a][b]] * Mh[b]
        H[a] = np.fft.irfftn(-acc, s=P, axes=(0, 1, 2))[:nz, :ny, :nx]
    return H


class DemagFFT:
    """The same FFT convolution with the kernel spectrum computed once (P:L55 precompute).

    workers: None = numpy.fft (single thread); an int = scipy.fft with that many
    threads (the all-core CPU baseline).  The same rfftn /
    irfftn either way.
    """

    def __init__(self, oct_, P=None, workers=None):
        _, nz, ny, nx = oct_.shape
        self.shape = (nz, ny, nx)
        self.P = P if P is not None else (_pad(nz), _pad(ny), _pad(nx))
        self.Ns = kernel_spectrum(oct_, self.P)
        if workers is None:
            self._rfftn, self._irfftn = np.fft.rfftn, np.fft.irfftn
        else:
            import scipy.fft as sf

            self._rfftn = lambda a, s, axes: sf.rfftn(a, s=s, axes=axes, workers=workers)
            self._irfftn = lambda a, s, axes: sf.irfftn(a, s=s, axes=axes, workers=workers)

    def __call__(self, M):
        nz, ny, nx = self.shape
        Mh = [self._rfftn(M[b], s=self.P, axes=(0, 1, 2)) for b in range(3)]
        H = np.empty((3, nz, ny, nx), dtype=np.float64)
        for a in range(3):
            acc = np.zeros_like(Mh[0])
            for b in range(3):
                acc = acc + self.Ns[_PAIRS[a][b]] * Mh[b]
            H[a] = self._irfftn(-acc, s=self.P, axes=(0, 1, 2))[:nz, :ny, :nx]
        return H
