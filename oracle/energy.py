"""Discrete Eq. (1) energy, fp64 (used to pin the fields by finite differences).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. (1): E = A [(grad Mx/Ms)^2 + (grad My/Ms)^2 + (grad Mz/Ms)^2]
                   + Ku (My^2 + Mz^2)/Ms^2 - 1/2 mu0 H_demag.M - mu0 H_ext.M,
discretised per bond / per cell:
  E = V sum_cells [ A sum_axis sum_{+neighbour} |m_nb - m_c|^2 / Delta^2
                    + Ku (1 - m_x^2) - 1/2 mu0 H_d.M - mu0 H_ext.M ],  m = M/Ms.
Ku (My^2+Mz^2)/Ms^2 = Ku (1 - m_x^2) on |M| = Ms; the latter is the form whose
unconstrained derivative is the SPEC field (reading Q4).
Returns (total, dict of terms) in joules.
"""
import numpy as np

from . import MU0


def energy(M, demag_op, A, Ms, Ku, d, hext, mask=None):
    """mask (reading Q26): sums over magnetic cells and bonds between two of them
    (M = 0 in empty cells; a bond to an empty cell is dropped)."""
    V = (d[0] * d[1]) * d[2]
    m = M / Ms
    w = np.ones(M.shape[1:]) if mask is None else (np.asarray(mask) != 0).astype(np.float64)
    e_ex = 0.0
    for arr_axis, delta in ((3, d[0]), (2, d[1]), (1, d[2])):
        n = M.shape[arr_axis]
        if n < 2:
            continue
        diff = np.diff(m, axis=arr_axis)
        bond = w.take(range(1, n), axis=arr_axis - 1) * w.take(range(0, n - 1), axis=arr_axis - 1)
        e_ex += A * ((diff * diff) * bond).sum() / (delta * delta)
    e_an = Ku * ((1.0 - m[0] * m[0]) * w).sum()
    Hd = demag_op(M)
    e_d = -0.5 * MU0 * (Hd * M).sum()
    e_z = -MU0 * sum(hext[a] * M[a].sum() for a in range(3))
    terms = {"exchange": V * e_ex, "anisotropy": V * e_an, "demag": V * e_d, "zeeman": V * e_z}
    return sum(terms.values()), terms
