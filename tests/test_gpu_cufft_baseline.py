"""The cuFFT comparison pipeline (baseline_cufft/, not part of libgrace) computes the
same method: its H_demag against the fp64 oracle (rel-L2 <= 1e-5, the north_star
bar) and its Euler steps against libgrace's (fp32 rounding of the same
arithmetic), so the bench_cufft.py timing compares like with like."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from bench_cufft import cufft_run  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, Workload, random_m  # noqa: E402


@pytest.mark.parametrize("n,d", [((40, 24, 6), (2e-9, 2e-9, 3e-9)), ((100, 25, 1), (5e-9, 5e-9, 3e-9))])
def test_cufft_baseline_demag_and_steps(n, d):
    w = Workload("t", n, d, 8e5, 1.3e-11, 1e4, 0.3, 2e-14, (1e3, -2e3, 5e2))
    M = random_m(n, w.Ms, seed=3).astype(np.float32)
    _, _, hd = cufft_run(w, M, 0, 0, want_m=False, want_hd=True)
    ho = DemagFFT(tensor_octant(*n, *d))(M.astype(np.float64))
    assert np.linalg.norm(hd - ho) / np.linalg.norm(ho) <= 1e-5
    _, mc, _ = cufft_run(w, M, 5, 0)
    g = pb.Grace(n, d, w.Ms, w.A, w.Ku, w.alpha, GAMMA0)
    g.set_m(M.astype(np.float64))
    g.set_hext(w.hext)
    g.step(5, w.dt)
    mg = g.get_m()
    g.close()
    assert np.abs(mg - mc).max() <= 1e-4 * w.Ms
