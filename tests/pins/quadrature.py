"""Cell-averaged demag tensor by direct quadrature of the dipole kernel.

Definition (the physics the Newell formulas integrate in closed form):
    N_ab(R) = -(1/(4 pi V)) int_obs int_src (3 r_a r_b - delta_ab r^2)/r^5 dV dV',
r = x_obs - x_src, for two dx*dy*dz cells whose centres differ by R.  The
difference of two uniform variables on [0, d] has the triangle density
(d - |u|), so the 6-D integral is a 3-D one with that weight; each axis is
split at the kink u = 0 and integrated by Gauss-Legendre.  Valid for cells
that do not touch (some |R_a| >= 2 d_a), where the integrand is smooth.
Independent of the oracle: it pins f, g and the 27-point stencil.
"""
import numpy as np

_IDX = {"xx": (0, 0), "xy": (0, 1), "xz": (0, 2), "yy": (1, 1), "yz": (1, 2), "zz": (2, 2)}


def cell_tensor_quad(comp, R, d, n=24):
    a, b = _IDX[comp]
    xg, wg = np.polynomial.legendre.leggauss(n)
    axes = []
    for ax in range(3):
        da = d[ax]
        # halves [-d,0] and [0,d]; weight (d - |u|)
        u = np.concatenate([(xg - 1.0) * da / 2.0, (xg + 1.0) * da / 2.0])
        w = np.concatenate([wg, wg]) * da / 2.0 * (da - np.abs(u))
        axes.append((R[ax] + u, w))
    X, Y, Z = np.meshgrid(axes[0][0], axes[1][0], axes[2][0], indexing="ij")
    W = axes[0][1][:, None, None] * axes[1][1][None, :, None] * axes[2][1][None, None, :]
    r = (X, Y, Z)
    r2 = X * X + Y * Y + Z * Z
    K = 3.0 * r[a] * r[b] - (r2 if a == b else 0.0)
    K = K / (r2 * r2 * np.sqrt(r2))
    V = d[0] * d[1] * d[2]
    return -float((W * K).sum()) / (4.0 * np.pi * V)
