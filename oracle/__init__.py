"""fp64 CPU oracle for the Grace (arXiv 1411.2565) LLG hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1411_2565_b200``) never imports it, and it
never imports the product: the two share no code, tables or constants.

It is a plain, slow, obviously-correct transcription of what the paper
computes, in the paper's order and notation, each function citing the passage
it follows ("P:Lnn" = line of PAPER.md, "S:Lnn" = line of SPEC.md, "Qnn" = a
reading recorded in DESIGN.md §3 where the paper is silent or garbled):

* ``tensor``  -- cell-averaged Newell demag tensor, real-space octant (P:L45,
  P:L55 defer the formula to refs [3],[11]; reading Q5/Q6/Q7/Q8).
* ``demag``   -- H_demag as the O(N^2) direct sum ("direct calculation for
  N sources at N observers") and as the zero-padded FFT convolution (P:L55
  "discrete convolution theorem and FFT ... zero-padding method").
* ``fields``  -- six-neighbour exchange, uniaxial-x anisotropy,
  Zeeman, and H_eff = sum of the four (Eq. (2)).
* ``llg``     -- Eq. (3) and the renormalised explicit Euler step.
* ``energy``  -- Eq. (1) energy, used to pin the fields by finite
  differences.
* ``sp4``     -- muMAG standard problem #4 harness.

Pins (what fixes each function independently of itself) live in
``tests/test_oracle_*.py``; the one function without an independent pin is
listed as "parity unpinned" in DESIGN.md §4: the SP4 <m>(t) curves beyond
physics-sanity checks, because the paper's Figs. 2-5 carry no numbers.
"""

PI = 3.141592653589793  # the double nearest pi
MU0 = 4.0 * PI * 1e-7  # mu0 = 4*pi*1e-7 (reading Q21)

from . import crmath, tensor, demag, fields, llg, energy, sp4  # noqa: E402,F401
