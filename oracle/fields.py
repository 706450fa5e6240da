"""Local field terms and the effective field, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Exchange: "the exchange field calculation is done with a six-neighbor scheme"
  (ref [13]); H_ex = (2A/(mu0 Ms^2)) sum_axis sum_+- (M(r+-e) - M(r))/Delta^2
  with Neumann boundaries (a missing neighbour contributes 0; S:L193, S:L228,
  reading Q11).  This is -1/mu0 dE/dM of the exchange term of Eq. (1).
* Anisotropy: Eq. (1) term Ku (My^2+Mz^2)/Ms^2, "anisotropy is on the x
  direction"; field H_an = (2Ku/(mu0 Ms^2)) Mx x (reading Q4).
* Zeeman: uniform H_ext (reading Q19).
* H_eff = H_exch + H_anis + H_demag + H_extern, Eq. (2) (1/mu0 per Q3).
* Geometry mask (the paper's future work "non-regular
  geometry"; reading Q26): ``mask`` [nz,ny,nx] of 0/1, M = 0 in empty
  cells.  An exchange bond exists only between two magnetic cells (an empty
  neighbour is a free surface, like the outer boundary); H_eff is reported as 0
  in empty cells.
"""
import numpy as np

from . import MU0


def exchange(M, A, Ms, d, mask=None):
    """Six-neighbour exchange field with Neumann boundaries. M: [3,nz,ny,nx].
    mask: bonds only between two cells with mask 1 (Q26)."""
    H = np.zeros_like(M, dtype=np.float64)
    # axis of the [3,nz,ny,nx] array for x, y, z and the matching cell size
    for arr_axis, delta in ((3, d[0]), (2, d[1]), (1, d[2])):
        n = M.shape[arr_axis]
        if n < 2:
            continue
        lo = [slice(None)] * 4
        hi = [slice(None)] * 4
        lo[arr_axis] = slice(0, n - 1)
        hi[arr_axis] = slice(1, n)
        lo, hi = tuple(lo), tuple(hi)
        c = 2.0 * A / (MU0 * Ms * Ms) / (delta * delta)
        diff = M[hi] - M[lo]  # M(r+e) - M(r) on the lower cell of each bond
        if mask is not None:
            diff = diff * (mask[hi[1:]] * mask[lo[1:]])  # no bond to an empty cell
        H[lo] += c * diff
        H[hi] -= c * diff
    return H


def anisotropy(M, Ku, Ms):
    """Uniaxial anisotropy along x: H = (2Ku/(mu0 Ms^2)) Mx x (Q4)."""
    H = np.zeros_like(M, dtype=np.float64)
    H[0] = (2.0 * Ku / (MU0 * Ms * Ms)) * M[0]
    return H


def zeeman(M, hext):
    H = np.zeros_like(M, dtype=np.float64)
    for a in range(3):
        H[a] = hext[a]
    return H


def heff(M, demag_op, A, Ms, Ku, d, hext, mask=None):
    """Eq. (2): H_eff = H_exch + H_anis + H_demag + H_extern (0 in empty cells, Q26)."""
    H = exchange(M, A, Ms, d, mask) + anisotropy(M, Ku, Ms) + demag_op(M) + zeeman(M, hext)
    return H if mask is None else H * mask


def schedule_amplitude(k, start, decay, stop):
    """SPEC FieldSchedule (paper §5 input "Hx Hy Hz startTime decayTime
    stopTime"): amplitude at timestep index k -- 0 before start, 1 in [start, decay),
    a linear ramp from 1 to 0 across [decay, stop), 0 at and after stop."""
    if not (0 <= start <= decay <= stop):
        raise ValueError("schedule needs 0 <= start <= decay <= stop")
    if k < start or k >= stop:
        return 0.0
    if k < decay:
        return 1.0
    return 1.0 - (k - decay) / (stop - decay)
