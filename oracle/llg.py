"""Eq. (3) and the renormalised explicit Euler step, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. (3):  dM/dt = -gamma/(1+alpha^2) (M x mu0 H)
                          - alpha gamma/((1+alpha^2) Ms) M x (M x mu0 H).
Reading Q1: the argument ``gamma0`` is gamma*mu0 in m/(A s) (muMAG SP4 value
2.211e5), so H stays in A/m and no mu0 appears.  Reading Q2: the equation is
used as written (no small-alpha expansion).

"The time integration of the LLG equation is implemented with Euler method"
(P:L55): M* = M + dt dM/dt(M, H_eff(M)), with H_eff evaluated once at the
pre-step M (reading Q17), then M <- Ms M*/|M*| (reading Q16).
A non-finite result aborts with the step index and cell.
With a geometry mask (reading Q26) only magnetic cells are stepped and
renormalised; empty cells keep M = 0, and <m> averages over magnetic cells.
"""
import numpy as np

from .fields import heff as _heff
from .fields import schedule_amplitude


class NonFinite(RuntimeError):
    def __init__(self, step, cell):
        super().__init__(f"non-finite magnetisation at step {step}, cell {cell}")
        self.step = step
        self.cell = cell


def llg_rhs(M, H, alpha, gamma0, Ms):
    """Eq. (3) per cell; M, H: [3, ...]."""
    MxH = np.cross(M, H, axis=0)
    MxMxH = np.cross(M, MxH, axis=0)
    a = gamma0 / (1.0 + alpha * alpha)
    return -a * MxH - (alpha * a / Ms) * MxMxH


def renormalize(M, Ms, mask=None):
    """Scale every cell to |M| = Ms; empty cells (mask 0) stay 0 (Q26)."""
    n = np.sqrt(M[0] * M[0] + M[1] * M[1] + M[2] * M[2])
    if mask is None:
        return Ms * M / n
    return np.where(mask > 0, Ms * M / np.where(mask > 0, n, 1.0), 0.0)


class Sim:
    """State + parameters of one fp64 run (the oracle twin of a grace context)."""

    def __init__(self, M, demag_op, Ms, A, Ku, alpha, gamma0, d, hext=(0.0, 0.0, 0.0), schedule=None, mask=None):
        # geometry mask [nz,ny,nx] of 0/1 (Q26): M = 0 in empty cells
        self.mask = None if mask is None else (np.asarray(mask) != 0).astype(np.float64)
        self.M = np.array(M, dtype=np.float64)
        if self.mask is not None:
            self.M = self.M * self.mask
        self.demag = demag_op
        self.Ms, self.A, self.Ku = Ms, A, Ku
        self.alpha, self.gamma0 = alpha, gamma0
        self.d = tuple(d)
        self.hext = tuple(hext)
        # optional SPEC FieldSchedule: (H0, start, decay, stop); the
        # applied field at step k is hext + amplitude(k) H0
        self.schedule = schedule
        self.step_count = 0

    def field(self, k=None):
        k = self.step_count if k is None else k
        if self.schedule is None:
            return self.hext
        H0, start, decay, stop = self.schedule
        a = schedule_amplitude(k, start, decay, stop)
        return tuple(self.hext[q] + a * H0[q] for q in range(3))

    def heff(self, M=None):
        M = self.M if M is None else M
        return _heff(M, self.demag, self.A, self.Ms, self.Ku, self.d, self.field(), self.mask)

    def euler_step(self, dt):
        H = self.heff()
        Mstar = self.M + dt * llg_rhs(self.M, H, self.alpha, self.gamma0, self.Ms)
        Mn = renormalize(Mstar, self.Ms, self.mask)
        bad = ~np.isfinite(Mn).all(axis=0)
        if bad.any():
            raise NonFinite(self.step_count, int(np.flatnonzero(bad.ravel())[0]))
        self.M = Mn
        self.step_count += 1

    def heun_step(self, dt):
        """Heun (explicit trapezoid, RK2) with the same renormalisation -- SURVEY
        §8(f) #4(iv), beyond the paper's Euler (SPEC lists higher-order integrators
        as future work):
            f0 = rhs(M, H(M, t_k));  M* = renorm(M + dt f0)
            f1 = rhs(M*, H(M*, t_{k+1}));  M' = renorm(M + dt (f0 + f1) / 2)."""
        f0 = llg_rhs(self.M, self.heff(), self.alpha, self.gamma0, self.Ms)
        Mstar = renormalize(self.M + dt * f0, self.Ms, self.mask)
        k = self.step_count
        self.step_count = k + 1  # the corrector's field is the next timestep's
        H1 = self.heff(Mstar)
        self.step_count = k
        f1 = llg_rhs(Mstar, H1, self.alpha, self.gamma0, self.Ms)
        Mn = renormalize(self.M + (0.5 * dt) * (f0 + f1), self.Ms, self.mask)
        bad = ~np.isfinite(Mn).all(axis=0)
        if bad.any():
            raise NonFinite(self.step_count, int(np.flatnonzero(bad.ravel())[0]))
        self.M = Mn
        self.step_count += 1

    def adaptive_run(self, t_span, dt0, tol, safety=0.9, fac_min=0.2, fac_max=5.0, max_attempts=10**7):
        """Adaptive time steps ("adaptive time steps" -- the paper's stated
        future work) by the embedded Euler / Heun pair.

        One attempt from M_k with step dt (H_eff as in euler_step / heun_step):
            f0 = rhs(M_k, H(M_k));       M_E = renorm(M_k + dt f0)   (Euler, order 1)
            f1 = rhs(M_E, H(M_E));       M_H = renorm(M_k + dt (f0 + f1)/2)   (Heun, order 2)
            err = max over cells |M_H - M_E| / Ms   (estimate of the Euler step's local error, O(dt^2))
        err <= tol: accept (M <- M_H, t <- t + dt), else reject (M kept).  Either
        way the next dt = dt * min(fac_max, max(fac_min, safety * sqrt(tol / err)))
        (fac_max when err = 0), and the step that would pass t_span is shortened to
        end on it.  A constant applied field only (a step-indexed schedule has no
        meaning here).  Returns (log of (t, dt, err, accepted) per attempt, next dt)."""
        if self.schedule is not None:
            raise ValueError("adaptive steps take a constant applied field")
        t, dt, log = 0.0, float(dt0), []
        for _ in range(max_attempts):
            if t >= t_span:
                break
            last = t + dt >= t_span
            h = t_span - t if last else dt
            f0 = llg_rhs(self.M, self.heff(), self.alpha, self.gamma0, self.Ms)
            ME = renormalize(self.M + h * f0, self.Ms, self.mask)
            f1 = llg_rhs(ME, self.heff(ME), self.alpha, self.gamma0, self.Ms)
            MH = renormalize(self.M + (0.5 * h) * (f0 + f1), self.Ms, self.mask)
            d = MH - ME
            err = float(np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]).max()) / self.Ms
            if not np.isfinite(err) or not np.isfinite(MH).all():
                raise NonFinite(self.step_count, int(np.flatnonzero((~np.isfinite(MH).all(axis=0)).ravel())[0]))
            ok = err <= tol
            log.append((t, h, err, ok))
            fac = fac_max if err == 0.0 else min(fac_max, max(fac_min, safety * np.sqrt(tol / err)))
            if ok:
                self.M = MH
                self.step_count += 1
                t = t_span if last else t + h
            dt = h * fac
        return log, dt

    def run(self, n, dt, method="euler"):
        step = self.heun_step if method == "heun" else self.euler_step
        for _ in range(n):
            step(dt)

    def mavg(self):
        """<M>/Ms, summed in fixed (C) order, over the magnetic cells (Q26)."""
        ncell = self.M[0].size if self.mask is None else self.mask.sum()
        return np.array([self.M[a].sum() for a in range(3)]) / (ncell * self.Ms)
