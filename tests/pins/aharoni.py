"""Demagnetising factor of a uniformly magnetised rectangular prism.

A. Aharoni, "Demagnetizing factors for rectangular ferromagnetic prisms",
J. Appl. Phys. 83, 3432 (1998), Eq. (1): prism of sides 2a x 2b x 2c
(a along x, b along y, c along z), D_z in SI (D_x + D_y + D_z = 1).
Evaluated in mpmath at 60 digits; an independent closed form used to pin the
oracle's Newell tensor (self-terms and the whole-prism mean field).
"""
import mpmath as mp


def aharoni_dz(a, b, c):
    with mp.workdps(60):
        a, b, c = mp.mpf(a), mp.mpf(b), mp.mpf(c)
        abc = mp.sqrt(a * a + b * b + c * c)
        ab = mp.sqrt(a * a + b * b)
        bc = mp.sqrt(b * b + c * c)
        ac = mp.sqrt(a * a + c * c)
        t = ((b * b - c * c) / (2 * b * c)) * mp.log((abc - a) / (abc + a))
        t += ((a * a - c * c) / (2 * a * c)) * mp.log((abc - b) / (abc + b))
        t += (b / (2 * c)) * mp.log((ab + a) / (ab - a))
        t += (a / (2 * c)) * mp.log((ab + b) / (ab - b))
        t += (c / (2 * a)) * mp.log((bc - b) / (bc + b))
        t += (c / (2 * b)) * mp.log((ac - a) / (ac + a))
        t += 2 * mp.atan((a * b) / (c * abc))
        t += (a ** 3 + b ** 3 - 2 * c ** 3) / (3 * a * b * c)
        t += ((a * a + b * b - 2 * c * c) / (3 * a * b * c)) * abc
        t += (c / (a * b)) * (ac + bc)
        t -= ((a * a + b * b) ** mp.mpf(1.5) + (b * b + c * c) ** mp.mpf(1.5)
              + (c * c + a * a) ** mp.mpf(1.5)) / (3 * a * b * c)
        return float(t / mp.pi)


def aharoni_factors(lx, ly, lz):
    """(D_x, D_y, D_z) of a prism with edge lengths lx, ly, lz."""
    a, b, c = lx / 2, ly / 2, lz / 2
    dz = aharoni_dz(a, b, c)
    dx = aharoni_dz(b, c, a)  # rotate so x plays the role of z
    dy = aharoni_dz(c, a, b)
    return dx, dy, dz
