"""Distributed z-slab path on one GPU: P virtual ranks vs the single-GPU path.

grace_create_virtual runs the partitioned algorithm (K1 per slab, all-to-all to
kx blocks, K2..K4 per block, all-to-all back, halo planes, K5 per slab) with
device copies standing in for NCCL, so every index, pack and halo rule of the
distributed step is exercised here.  The per-pencil arithmetic
is the same, so H_eff and M(t) must agree with the single path to fp32
round-off (observed: bitwise), and with the oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1411_2565_b200 as pb  # noqa: E402
from paper_1411_2565_b200.dist import partition  # noqa: E402
from oracle.demag import DemagFFT  # noqa: E402
from oracle.fields import heff as oracle_heff  # noqa: E402
from oracle.tensor import tensor_octant  # noqa: E402
from workloads import GAMMA0, random_m  # noqa: E402

CASES = [
    ((16, 12, 8), (1e-9, 1e-9, 1e-9), (2, 4, 8)),
    ((100, 20, 4), (5e-9, 5e-9, 3e-9), (2, 4)),
    ((7, 5, 6), (1e-9, 2e-9, 1e-9), (2, 3, 6)),
    ((2, 3, 4), (1e-9, 1e-9, 1e-9), (4,)),       # Kx = 3 < 4 ranks: an empty kx block
    ((64, 48, 16), (2e-9, 2e-9, 2e-9), (2, 8)),
    ((6, 2048, 4), (1e-9, 1e-9, 1e-9), (2,)),    # Py = 4096: staged K2 on the distributed layout
]


@pytest.mark.parametrize("n,d,Ps", CASES)
def test_virtual_ranks_match_single_and_oracle(n, d, Ps):
    Ms, A, Ku, alpha = 8e5, 1.3e-11, 2e4, 0.3
    hext = (1e4, -2e3, 5e3)
    M = random_m(n, Ms, seed=31)
    ref = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0)
    ref.set_m(M)
    ref.set_hext(hext)
    H1 = ref.heff()
    Ho = oracle_heff(M, DemagFFT(tensor_octant(*n, *d)), A, Ms, Ku, d, hext)
    assert np.linalg.norm(H1 - Ho) <= 1e-5 * np.linalg.norm(Ho)
    ref.step(7, 1e-14)
    M1 = ref.get_m()
    m1 = ref.mavg()
    for P in Ps:
        g = pb.Grace(n, d, Ms, A, Ku, alpha, GAMMA0, virtual_ranks=P)
        part = pb.grace_partition(g.h)
        want = partition(n[0], n[2], 0, P)
        assert (part["P"], part["nz_local"], part["kx_block"], part["kx_columns"]) == \
            (P, want.nz_local, want.kx_block, want.kx_columns)
        g.set_m(M)
        g.set_hext(hext)
        H = g.heff()
        assert np.abs(H - H1).max() <= 1e-6 * np.abs(H1).max(), P
        g.step(7, 1e-14)
        Mp = g.get_m()
        assert np.abs(Mp - M1).max() <= 1e-6 * Ms, P
        np.testing.assert_allclose(g.mavg(), m1, rtol=0, atol=1e-9)
        g.close()
    ref.close()


def test_virtual_ranks_bitwise_on_slab_like_grid():
    n, d = (128, 64, 16), (1e-9, 1e-9, 1e-9)
    M = random_m(n, 1e6, seed=3)
    out = []
    for P in (None, 4):
        g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
        g.set_m(M)
        g.step(5, 1e-15)
        out.append(g.get_m())
        g.close()
    assert np.array_equal(out[0], out[1])


def test_virtual_errors():
    with pytest.raises(pb.GraceError) as e:
        pb.Grace((8, 8, 6), (1e-9,) * 3, 8e5, 1e-11, 0, 0.5, GAMMA0, virtual_ranks=4)
    assert e.value.code == pb.GRACE_EINVAL
    g = pb.Grace((8, 4, 4), (1e-9,) * 3, 8e5, 1e-11, 0, 0.5, GAMMA0, virtual_ranks=2)
    M = random_m((8, 4, 4), 8e5, seed=1)
    M[:, 3, 1, 2] = 0.0  # cell ((3*4)+1)*8+2 = 106, in rank 1's slab
    with pytest.raises(pb.GraceError) as e:
        g.set_m(M)
    assert e.value.code == pb.GRACE_EZEROCELL and "cell 106" in str(e.value)
    g.close()


def test_virtual_ranks_heun_matches_single():
    """Heun on the partitioned path: the predictor's halos are re-exchanged for M*."""
    n, d, Ms = (16, 12, 8), (1e-9, 1e-9, 1e-9), 8e5
    M = random_m(n, Ms, seed=47)
    out = []
    for kw in ({}, {"virtual_ranks": 4}):
        g = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, **kw)
        g.set_integrator("heun")
        g.set_m(M)
        g.set_hext((1e4, 0, -5e3))
        g.step(12, 2e-14)
        out.append(g.get_m())
        g.close()
    assert np.abs(out[0] - out[1]).max() <= 1e-6 * Ms


def test_nccl_path_one_rank_matches_single(monkeypatch):
    """The real NCCL path (dlopen'd libnccl, unique id, communicator, grouped send/recv
    for both transposes, ncclAllReduce for <M> and the diagnostics, destination-
    blocked layouts) on a one-rank communicator (GRACE_FORCE_NCCL): same results
    as the single-GPU context.  Multi-rank NCCL runs need more GPUs than this
    machine gives; the P > 1 index logic is covered by the virtual ranks above."""
    monkeypatch.setenv("GRACE_FORCE_NCCL", "1")
    n, d, Ms = (48, 20, 6), (2e-9, 2e-9, 3e-9), 8e5
    M = random_m(n, Ms, seed=53)
    h = pb.grace_create_dist(*n, *d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, 0, 1, pb.grace_nccl_unique_id())
    assert pb.grace_partition(h)["P"] == 1 and pb.grace_partition(h)["kx_block"] > 0  # distributed layouts, P = 1
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    for hh in (h, ref.h):
        pb.grace_set_m(hh, M.ravel().copy())
        pb.grace_set_hext(hh, 1e4, -3e3, 2e3)
    out = []
    for hh in (h, ref.h):
        H = np.empty(3 * M[0].size)
        pb.grace_heff(hh, H)
        pb.grace_step(hh, 7, 2e-14)
        Mo = np.empty(3 * M[0].size)
        pb.grace_get_m(hh, Mo)
        out.append((H, Mo, pb.grace_mavg(hh), pb.grace_energy(hh)))
    (Ha, Ma, ma, ea), (Hb, Mb, mb, eb) = out
    assert np.abs(Ha - Hb).max() <= 1e-6 * np.abs(Hb).max()
    assert np.abs(Ma - Mb).max() <= 1e-6 * Ms
    np.testing.assert_allclose(ma, mb, rtol=0, atol=1e-9)
    np.testing.assert_allclose(ea, eb, rtol=1e-9, atol=0)
    pb.grace_destroy(h)
    ref.close()


def test_nccl_path_one_rank_masked_matches_single(monkeypatch):
    """Geometry mask (reading Q26) on the NCCL path: the magnetic-cell count is
    all-reduced over the communicator for <m>; one rank = the single context."""
    from workloads import ellipse_mask

    monkeypatch.setenv("GRACE_FORCE_NCCL", "1")
    n, d, Ms = (48, 20, 6), (2e-9, 2e-9, 3e-9), 8e5
    M = random_m(n, Ms, seed=54)
    mask = ellipse_mask(n)
    h = pb.grace_create_dist(*n, *d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, 0, 1, pb.grace_nccl_unique_id())
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    out = []
    for hh in (h, ref.h):
        pb.grace_set_geometry(hh, mask.ctypes.data)
        pb.grace_set_m(hh, M.ravel().copy())
        pb.grace_step(hh, 5, 2e-14)
        Mo = np.empty(3 * M[0].size)
        pb.grace_get_m(hh, Mo)
        out.append((Mo, pb.grace_mavg(hh), pb.grace_energy(hh)))
    (Ma, ma, ea), (Mb, mb, eb) = out
    assert np.abs(Ma - Mb).max() <= 1e-6 * Ms
    assert np.all(Ma.reshape(3, -1)[:, mask.ravel() == 0] == 0.0)
    np.testing.assert_allclose(ma, mb, rtol=0, atol=1e-9)
    np.testing.assert_allclose(ea, eb, rtol=1e-9, atol=0)
    pb.grace_destroy(h)
    ref.close()


@pytest.mark.parametrize("n,P", [((128, 64, 16), 4), ((64, 48, 16), 2)])
def test_pipelined_graph_step_bitwise_equals_unpipelined_eager(n, P, monkeypatch):
    """Per-component pipelined transposes (comm stream, events) captured into CUDA
    graphs = the unpipelined eager distributed step = the single-GPU step, bitwise."""
    d = (1e-9, 1e-9, 1e-9)
    M = random_m(n, 1e6, seed=61)
    out = []
    for env in ({}, {"GRACE_NO_PIPE": "1"}, {"GRACE_DIST_EAGER": "1"}, {"GRACE_NO_PIPE": "1", "GRACE_DIST_EAGER": "1"}):
        for k in ("GRACE_NO_PIPE", "GRACE_DIST_EAGER"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
        part = pb.grace_partition(g.h)
        assert part["pipelined"] == (0 if "GRACE_NO_PIPE" in env else 1)
        assert part["graphs"] == (0 if "GRACE_DIST_EAGER" in env else 1)
        g.set_m(M)
        g.set_hext((1e4, 0, 0))
        g.step(19, 1e-15)  # one 16-step chunk + 3 single steps
        H = g.heff()
        out.append((g.get_m(), H))
        g.close()
    ref = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
    ref.set_m(M)
    ref.set_hext((1e4, 0, 0))
    ref.step(19, 1e-15)
    out.append((ref.get_m(), ref.heff()))
    ref.close()
    diffs = [(float(np.abs(out[0][0] - Mo).max()), float(np.abs(out[0][1] - Ho).max())) for Mo, Ho in out[1:]]
    assert all(dm == 0.0 and dh == 0.0 for dm, dh in diffs), diffs


def test_nccl_one_rank_graphs_pipeline_and_agreed_nonfinite(monkeypatch):
    """NCCL path on a one-rank communicator: the pipelined step is graph-captured
    (NCCL calls inside the graph), the halo has its own split communicator, and a
    non-finite step reports the same (step, global cell) as the single context."""
    monkeypatch.setenv("GRACE_FORCE_NCCL", "1")
    n, d, Ms = (64, 20, 8), (2e-9, 2e-9, 3e-9), 8e5
    M = random_m(n, Ms, seed=57)
    h = pb.grace_create_dist(*n, *d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, 0, 1, pb.grace_nccl_unique_id())
    part = pb.grace_partition(h)
    assert part["pipelined"] == 1 and part["graphs"] == 1
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    res = []
    for hh in (h, ref.h):
        pb.grace_set_m(hh, M.ravel().copy())
        pb.grace_step(hh, 20, 2e-14)
        Mo = np.empty(3 * M[0].size)
        pb.grace_get_m(hh, Mo)
        pb.grace_set_hext(hh, 3e38, 3e38, 3e38)
        with pytest.raises(pb.GraceError) as e:
            pb.grace_step(hh, 2, 1e-13)
        assert e.value.code == pb.GRACE_ENONFINITE
        res.append((Mo, pb.grace_last_nonfinite(hh)))
    assert np.array_equal(res[0][0], res[1][0])
    assert res[0][1] == res[1][1]
    pb.grace_destroy(h)
    ref.close()


@pytest.mark.parametrize("n,P", [((128, 64, 16), 4), ((100, 20, 4), 2)])
def test_fused_p2p_transposes_bitwise(n, P, monkeypatch):
    """GRACE_P2P: K1 / K4 store their destination blocks straight into the other
    ranks' receive buffers (no separate all-to-all): bitwise the pipelined NCCL-style
    exchange path and the single-GPU step."""
    d = (1e-9, 1e-9, 1e-9)
    M = random_m(n, 1e6, seed=62)
    out = []
    for p2p in (True, False):
        if p2p:
            monkeypatch.setenv("GRACE_P2P", "1")
        else:
            monkeypatch.delenv("GRACE_P2P", raising=False)
        g = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0, virtual_ranks=P)
        part = pb.grace_partition(g.h)
        assert part["p2p"] == (1 if p2p else 0)
        assert part["pipelined"] == (0 if p2p else 1)
        g.set_m(M)
        g.step(19, 1e-15)
        out.append((g.get_m(), g.heff()))
        g.close()
    monkeypatch.delenv("GRACE_P2P", raising=False)
    ref = pb.Grace(n, d, 1e6, 1e-11, 6.2832e4, 0.5, GAMMA0)
    ref.set_m(M)
    ref.step(19, 1e-15)
    out.append((ref.get_m(), ref.heff()))
    ref.close()
    for Mo, Ho in out[1:]:
        assert np.array_equal(out[0][0], Mo)
        assert np.array_equal(out[0][1], Ho)


def test_fused_p2p_nccl_one_rank(monkeypatch):
    """The fused transposes on the NCCL path (one rank: its own buffers as the peer
    table; the barrier all-reduce captured into the step graphs)."""
    monkeypatch.setenv("GRACE_FORCE_NCCL", "1")
    monkeypatch.setenv("GRACE_P2P", "1")
    n, d, Ms = (64, 20, 8), (2e-9, 2e-9, 3e-9), 8e5
    M = random_m(n, Ms, seed=58)
    h = pb.grace_create_dist(*n, *d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0, 0, 1, pb.grace_nccl_unique_id())
    assert pb.grace_partition(h)["p2p"] == 1
    monkeypatch.delenv("GRACE_P2P")
    ref = pb.Grace(n, d, Ms, 1.3e-11, 2e4, 0.3, GAMMA0)
    res = []
    for hh in (h, ref.h):
        pb.grace_set_m(hh, M.ravel().copy())
        pb.grace_step(hh, 20, 2e-14)
        Mo = np.empty(3 * M[0].size)
        pb.grace_get_m(hh, Mo)
        res.append(Mo)
    assert np.array_equal(res[0], res[1])
    pb.grace_destroy(h)
    ref.close()
