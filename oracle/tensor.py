"""Cell-averaged demagnetising tensor, real-space octant, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper uses "the convolution of magnetizations and demagnetization tensor in
a regular discretization" (Sec. 3) and defers the tensor formula to its
refs [3],[11].  Reading Q5: Newell's cell-averaged
tensor (f, g and the 27-point second difference) for near offsets, the point
dipole beyond C = 30 cell diagonals, exact zeros and parity
(reading Q7), and the fixed fp64 evaluation order of reading Q8 so the
GPU setup can be compared bit for bit.

Component order everywhere: 0 xx, 1 xy, 2 xz, 3 yy, 4 yz, 5 zz.
Octant layout: ``oct[c, k, j, i]`` = N_c at the cell offset (i*dx, j*dy, k*dz),
0 <= i < nx, 0 <= j < ny, 0 <= k < nz.  Sign convention: H = -N * M, so the
self-term of a cube is +1/3 on the diagonal.
"""
import functools
import math

import numpy as np

from . import PI
from .crmath import cratan, crlog

COMPONENTS = ("xx", "xy", "xz", "yy", "yz", "zz")
CUTOFF = 30.0  # far field beyond 30 cell diagonals (reading Q6)

# For each component: which function, and how the lattice indices (I,J,K) along
# (x,y,z) map onto its three arguments (0 -> I*dx, 1 -> J*dy, 2 -> K*dz).
#   N_xx: f(X,Y,Z)  N_yy: f(Y,X,Z)  N_zz: f(Z,Y,X)
#   N_xy: g(X,Y,Z)  N_xz: g(X,Z,Y)  N_yz: g(Y,Z,X)
_PERM = {
    "xx": ("f", (0, 1, 2)),
    "xy": ("g", (0, 1, 2)),
    "xz": ("g", (0, 2, 1)),
    "yy": ("f", (1, 0, 2)),
    "yz": ("g", (1, 2, 0)),
    "zz": ("f", (2, 1, 0)),
}
# Axes in which each component is odd: the sign of the node argument.
_ODD = {"xx": (), "xy": (0, 1), "xz": (0, 2), "yy": (), "yz": (1, 2), "zz": ()}
_W = {-1: -1.0, 0: 2.0, 1: -1.0}


@functools.lru_cache(maxsize=None)
def newell_f(x: float, y: float, z: float) -> float:
    """Newell's f at x, y, z >= 0 (f is even in each argument).

    f = 1/2 y (z^2-x^2) asinh(y/sqrt(x^2+z^2)) + 1/2 z (y^2-x^2) asinh(z/sqrt(x^2+y^2))
        - x y z atan(y z / (x R)) + (2x^2 - y^2 - z^2) R / 6,
    with asinh(u/sqrt(v^2+w^2)) = log((u+R)/sqrt(v^2+w^2)).  A term whose
    prefactor vanishes or whose log/atan argument is undefined is dropped (its
    analytic limit is 0).  Evaluated exactly as parenthesised (reading Q8).
    """
    x2 = x * x
    y2 = y * y
    z2 = z * z
    R = math.sqrt((x2 + y2) + z2)
    t = 0.0
    if y > 0.0 and (x2 + z2) > 0.0:
        t = t + ((0.5 * y) * (z2 - x2)) * crlog((y + R) / math.sqrt(x2 + z2))
    if z > 0.0 and (x2 + y2) > 0.0:
        t = t + ((0.5 * z) * (y2 - x2)) * crlog((z + R) / math.sqrt(x2 + y2))
    if x > 0.0 and y > 0.0 and z > 0.0:
        t = t - ((x * y) * z) * cratan((y * z) / (x * R))
    t = t + ((((2.0 * x2) - y2) - z2) * R) / 6.0
    return t


@functools.lru_cache(maxsize=None)
def newell_g(x: float, y: float, z: float) -> float:
    """Newell's g at x, y, z >= 0 (g is odd in x and y; the caller applies the sign).

    g = x y z asinh(z/sqrt(x^2+y^2)) + y/6 (3z^2-y^2) asinh(x/sqrt(y^2+z^2))
        + x/6 (3z^2-x^2) asinh(y/sqrt(x^2+z^2)) - z^3/6 atan(x y/(z R))
        - z y^2/2 atan(x z/(y R)) - z x^2/2 atan(y z/(x R)) - x y R/3.
    """
    x2 = x * x
    y2 = y * y
    z2 = z * z
    R = math.sqrt((x2 + y2) + z2)
    t = 0.0
    if x > 0.0 and y > 0.0 and z > 0.0:
        t = t + ((x * y) * z) * crlog((z + R) / math.sqrt(x2 + y2))
    if x > 0.0 and (y2 + z2) > 0.0:
        t = t + ((y / 6.0) * ((3.0 * z2) - y2)) * crlog((x + R) / math.sqrt(y2 + z2))
    if y > 0.0 and (x2 + z2) > 0.0:
        t = t + ((x / 6.0) * ((3.0 * z2) - x2)) * crlog((y + R) / math.sqrt(x2 + z2))
    if x > 0.0 and y > 0.0 and z > 0.0:
        t = t - ((z2 * z) / 6.0) * cratan((x * y) / (z * R))
        t = t - ((z * y2) / 2.0) * cratan((x * z) / (y * R))
        t = t - ((z * x2) / 2.0) * cratan((y * z) / (x * R))
    t = t - ((x * y) * R) / 3.0
    return t


def _node(comp, I, J, K, d):
    """Unsigned lattice value of component ``comp`` at non-negative node (I,J,K)."""
    fn, perm = _PERM[comp]
    coords = (float(I) * d[0], float(J) * d[1], float(K) * d[2])  # integer first, then * d (Q8)
    args = tuple(coords[p] for p in perm)
    return newell_f(*args) if fn == "f" else newell_g(*args)


def _sign(v):
    return (v > 0) - (v < 0)


def near_mask(nx, ny, nz, dx, dy, dz, cutoff=CUTOFF):
    """Boolean [nz,ny,nx]: offsets with r^2 <= (C*C)*diag^2 use Newell."""
    i = np.arange(nx, dtype=np.float64)
    j = np.arange(ny, dtype=np.float64)
    k = np.arange(nz, dtype=np.float64)
    X = (i * dx)[None, None, :]
    Y = (j * dy)[None, :, None]
    Z = (k * dz)[:, None, None]
    r2 = (X * X + Y * Y) + Z * Z
    diag2 = (dx * dx + dy * dy) + dz * dz
    return r2 <= (cutoff * cutoff) * diag2


def _dipole(X, Y, Z, dx, dy, dz):
    """Point-dipole tensor N_ab = -(V/4pi)(3 r_a r_b - delta_ab r^2)/r^5."""
    r2 = (X * X + Y * Y) + Z * Z
    r = np.sqrt(r2)
    r5 = (r2 * r2) * r
    V = (dx * dy) * dz
    c = V / (4.0 * PI)
    out = {
        "xx": -((c * ((3.0 * (X * X)) - r2)) / r5),
        "yy": -((c * ((3.0 * (Y * Y)) - r2)) / r5),
        "zz": -((c * ((3.0 * (Z * Z)) - r2)) / r5),
        "xy": -((c * (3.0 * (X * Y))) / r5),
        "xz": -((c * (3.0 * (X * Z))) / r5),
        "yz": -((c * (3.0 * (Y * Z))) / r5),
    }
    return out


def _near_values(comp, ii, jj, kk, d):
    """Newell 27-point second difference at the integer offsets (ii,jj,kk) (arrays).

    N = inv * sum_{a,b,c in (-1,0,1)} w_a w_b w_c F(i+a, j+b, k+c), w_0 = 2,
    w_+-1 = -1, accumulated a (x) outer, b (y), c (z) inner, then multiplied once
    by inv = 1/((((4 pi) dx) dy) dz)  (reading Q8).
    """
    dx, dy, dz = d
    imax = int(ii.max()) + 1 if ii.size else 0
    jmax = int(jj.max()) + 1 if jj.size else 0
    kmax = int(kk.max()) + 1 if kk.size else 0
    lat = np.empty((kmax + 1, jmax + 1, imax + 1), dtype=np.float64)
    # Only the nodes touched by some near offset are needed; evaluating the whole
    # box is simpler and the extra nodes are never read.
    need = np.zeros_like(lat, dtype=bool)
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                need[np.abs(kk + c), np.abs(jj + b), np.abs(ii + a)] = True
    for K, J, I in zip(*np.nonzero(need)):
        lat[K, J, I] = _node(comp, int(I), int(J), int(K), d)
    odd = _ODD[comp]
    s = np.zeros(ii.shape, dtype=np.float64)
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                w = (_W[a] * _W[b]) * _W[c]
                F = lat[np.abs(kk + c), np.abs(jj + b), np.abs(ii + a)]
                if odd:
                    sg = np.ones(ii.shape, dtype=np.float64)
                    for ax in odd:
                        v = (ii + a, jj + b, kk + c)[ax]
                        sg = sg * np.sign(v).astype(np.float64)
                    F = sg * F
                s = s + w * F
    inv = 1.0 / ((((4.0 * PI) * dx) * dy) * dz)
    return s * inv


def _exact_zeros(oct_):
    """N_xy = 0 on i=0 or j=0, N_xz on i=0 or k=0, N_yz on j=0 or k=0 (Q7)."""
    oct_[1][:, :, 0] = 0.0
    oct_[1][:, 0, :] = 0.0
    oct_[2][:, :, 0] = 0.0
    oct_[2][0, :, :] = 0.0
    oct_[4][:, 0, :] = 0.0
    oct_[4][0, :, :] = 0.0
    return oct_


def tensor_octant(nx, ny, nz, dx, dy, dz, cutoff=CUTOFF):
    """Real-space octant [6, nz, ny, nx] fp64 of the six unique N_ab.

    Near offsets (reading Q6): Newell; far offsets: point dipole; then exact zeros.
    """
    d = (float(dx), float(dy), float(dz))
    near = near_mask(nx, ny, nz, *d, cutoff=cutoff)
    kk, jj, ii = np.nonzero(near)
    fk, fj, fi = np.nonzero(~near)
    out = np.zeros((6, nz, ny, nx), dtype=np.float64)
    if fk.size:
        X = fi.astype(np.float64) * d[0]
        Y = fj.astype(np.float64) * d[1]
        Z = fk.astype(np.float64) * d[2]
        dip = _dipole(X, Y, Z, *d)
        for c, name in enumerate(COMPONENTS):
            out[c][fk, fj, fi] = dip[name]
    for c, name in enumerate(COMPONENTS):
        out[c][kk, jj, ii] = _near_values(name, ii, jj, kk, d)
    out = _exact_zeros(out)
    out[out == 0.0] = 0.0  # canonicalise -0.0
    return out


def tensor_entry(comp, i, j, k, dx, dy, dz, cutoff=CUTOFF):
    """One octant entry N_comp(i,j,k), i,j,k >= 0: the same arithmetic as tensor_octant.

    Used to check full-size GPU tensors at sampled offsets without building the
    whole octant.
    """
    name = COMPONENTS[comp] if isinstance(comp, int) else comp
    odd = _ODD[name]
    if any((i, j, k)[ax] == 0 for ax in odd):
        return 0.0
    d = (float(dx), float(dy), float(dz))
    X = float(i) * d[0]
    Y = float(j) * d[1]
    Z = float(k) * d[2]
    r2 = (X * X + Y * Y) + Z * Z
    diag2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]
    if r2 <= (cutoff * cutoff) * diag2:
        v = _near_values(name, np.array([i]), np.array([j]), np.array([k]), d)[0]
    else:
        v = _dipole(np.array([X]), np.array([Y]), np.array([Z]), *d)[name][0]
    return 0.0 if v == 0.0 else float(v)


def full_tensor(oct_, di, dj, dk):
    """3x3 N at a signed cell offset from the octant by parity.

    N_aa is even in every axis; N_ab is odd in axes a and b, even in the third.
    Returns a (3,3) array.
    """
    ai, aj, ak = abs(di), abs(dj), abs(dk)
    v = oct_[:, ak, aj, ai]
    sx, sy, sz = _sign(di) or 1, _sign(dj) or 1, _sign(dk) or 1
    xx, xy, xz, yy, yz, zz = v
    xy = xy * sx * sy
    xz = xz * sx * sz
    yz = yz * sy * sz
    return np.array([[xx, xy, xz], [xy, yy, yz], [xz, yz, zz]])
