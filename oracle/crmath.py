"""Correctly rounded fp64 log and atan (reading Q8 in DESIGN.md).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The demag-tensor setup must be bit-exact between this oracle and the GPU
(BASELINE.json north_star: "the demag-tensor setup is bit-exact between CPU and
GPU in fp64").  IEEE +,-,*,/,sqrt are correctly rounded on both sides; log and
atan are not, so both sides use the correctly rounded value: here, a 160-bit
mpmath evaluation rounded once to the nearest double.  (``float(mpf)`` rounds
toward zero in mpmath 1.3, so the explicit round-to-nearest conversion is
required.)
"""
import mpmath
from mpmath.libmp import to_float

_PREC = 160


def crlog(x: float) -> float:
    """log(x) rounded to the nearest double; x > 0 is a double."""
    with mpmath.workprec(_PREC):
        return to_float(mpmath.log(mpmath.mpf(x))._mpf_, rnd="n")


def cratan(x: float) -> float:
    """atan(x) rounded to the nearest double; x is a double."""
    with mpmath.workprec(_PREC):
        return to_float(mpmath.atan(mpmath.mpf(x))._mpf_, rnd="n")
