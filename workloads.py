"""Seeded synthetic inputs and the BASELINE.json configurations.

Shared by the tests, ``bench.py`` and ``__graft_entry__``; imported by neither
the oracle nor the product library, and holds none of the method's arithmetic:
only grid/material constants and seeded random magnetisation fields.

Input recipe: a random M is i.i.d. standard-normal triplets per
cell, scaled to |M| = Ms, drawn from numpy PCG64(seed) in [3][nz][ny][nx]
(x fastest) order; the default seed 14112565 is the arXiv id.
"""
from dataclasses import dataclass, field

import numpy as np

SEED = 14112565
MU0 = 4.0 * 3.141592653589793 * 1e-7
GAMMA0 = 2.211e5  # gamma*mu0 in m/(A s) (reading Q1)


@dataclass(frozen=True)
class Workload:
    name: str
    n: tuple            # (nx, ny, nz)
    d: tuple            # (dx, dy, dz) metres
    Ms: float
    A: float
    Ku: float
    alpha: float
    dt: float
    hext: tuple = (0.0, 0.0, 0.0)
    gamma0: float = GAMMA0
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def cells(self):
        return self.n[0] * self.n[1] * self.n[2]


def _mT(b):
    return tuple(x * 1e-3 / MU0 for x in b)


# Paper Sec. 4 benchmark material: A = 1e-11 J/m, Ms = 1000 kA/m,
# H_anis = 100 kA/m along x -> Ku = mu0 Ms H_k / 2.
BENCH_MS = 1.0e6
BENCH_A = 1.0e-11
BENCH_KU = MU0 * BENCH_MS * 1.0e5 / 2.0
# muMAG SP4 permalloy
PY_MS = 8.0e5
PY_A = 1.3e-11

WORKLOADS = {
    "sp4_field1": Workload("sp4_field1", (100, 25, 1), (5e-9, 5e-9, 3e-9), PY_MS, PY_A, 0.0,
                           0.02, 2.5e-14, _mT((-24.6, 4.3, 0.0)),
                           note="BASELINE configs[0]: muMAG SP4 field 1, 5x5x3 nm cells"),
    "sp4_field2_refined": Workload("sp4_field2_refined", (200, 50, 1), (2.5e-9, 2.5e-9, 3e-9),
                                   PY_MS, PY_A, 0.0, 0.02, 6.25e-15, _mT((-35.5, -6.3, 0.0)),
                                   note="BASELINE configs[1]: SP4 refined mesh, field 2"),
    "film_512x512x8": Workload("film_512x512x8", (512, 512, 8), (5e-9, 5e-9, 3e-9), PY_MS, PY_A,
                               0.0, 0.5, 1e-14, note="BASELINE configs[2]: thin-film relaxation"),
    "slab_1024x1024x32": Workload("slab_1024x1024x32", (1024, 1024, 32), (1e-9, 1e-9, 1e-9),
                                  BENCH_MS, BENCH_A, BENCH_KU, 0.5, 1e-15,
                                  note="BASELINE configs[3]: 3-D slab, paper Sec. 4 material"),
    "block_2048x2048x64": Workload("block_2048x2048x64", (2048, 2048, 64), (1e-9, 1e-9, 1e-9),
                                   BENCH_MS, BENCH_A, BENCH_KU, 0.5, 1e-15,
                                   note="BASELINE configs[4]: large block"),
}


for _N in (128, 256):  # Table-1 sizes as bench workloads (table1_cube below)
    WORKLOADS[f"cube_{_N}"] = Workload(f"cube_{_N}", (_N, _N, _N), (1e-9, 1e-9, 1e-9), BENCH_MS, BENCH_A, BENCH_KU,
                                       0.5, 1e-15, note="paper Table 1 size")


def table1_cube(N):
    """Paper Table 1 workload: N^3 cube, Sec. 4 material, 1 nm cells."""
    return Workload(f"cube_{N}", (N, N, N), (1e-9, 1e-9, 1e-9), BENCH_MS, BENCH_A, BENCH_KU,
                    0.5, 1e-15, note="paper Table 1 size")


def random_m(n, Ms, seed=SEED):
    """Random magnetisation [3, nz, ny, nx] float64 with |M| = Ms per cell."""
    nx, ny, nz = n
    rng = np.random.Generator(np.random.PCG64(seed))
    v = rng.standard_normal((3, nz, ny, nx))
    v /= np.sqrt((v * v).sum(axis=0, keepdims=True))
    return Ms * v


def uniform_m(n, Ms, direction):
    nx, ny, nz = n
    u = np.asarray(direction, dtype=np.float64)
    u = u / np.sqrt((u * u).sum())
    M = np.empty((3, nz, ny, nx))
    for a in range(3):
        M[a] = Ms * u[a]
    return M


def ellipse_mask(n, hole=True):
    """Non-regular geometry: an elliptical disc
    inscribed in the nx x ny plane, extruded through z, optionally with an
    off-centre circular hole (antidot).  uint8 [nz, ny, nx]."""
    nx, ny, nz = n
    y, x = np.mgrid[0:ny, 0:nx]
    u = (x + 0.5 - nx / 2) / (nx / 2)
    v = (y + 0.5 - ny / 2) / (ny / 2)
    m = (u * u + v * v) <= 1.0
    if hole:
        hu = (x + 0.5 - 0.6 * nx) / (0.12 * nx)
        hv = (y + 0.5 - 0.45 * ny) / (0.12 * nx)
        m &= (hu * hu + hv * hv) > 1.0
    return np.broadcast_to(m, (nz, ny, nx)).astype(np.uint8).copy()


def box_mask(n, lo, size):
    """uint8 [nz, ny, nx] mask of the box of `size` (sx, sy, sz) cells at corner `lo`."""
    nx, ny, nz = n
    m = np.zeros((nz, ny, nx), dtype=np.uint8)
    m[lo[2]:lo[2] + size[2], lo[1]:lo[1] + size[1], lo[0]:lo[0] + size[0]] = 1
    return m
