"""Host logic of the distributed z-slab path on CPU: world_size 2 over gloo.

Covers what runs on the host in a torchrun launch: rank/world
from the environment, broadcast of the 128-byte NCCL unique id, and the slab /
kx-block partition (every z plane and every kx column owned exactly once).
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1411_2565_b200.dist import partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1411_2565_b200 import dist as gd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = gd.env_ranks()
    payload = bytes(range(128)) if rank == 0 else bytes(128)
    got = gd.broadcast_bytes(payload, 0)
    slabs = {}
    for grid in [(1024, 32), (100, 4), (2, 8), (7, 6)]:
        s = gd.partition(grid[0], grid[1], rank, world)
        out = [None] * world
        dist.all_gather_object(out, s)
        slabs[grid] = out
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, (r, w, lr), got, slabs))


@pytest.mark.timeout(120)
def test_gloo_world2_broadcast_and_partition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    for rank, (r, w, lr), got, slabs in res:
        assert (r, w, lr) == (rank, world, rank)
        assert got == bytes(range(128))
        for (nx, nz), ss in slabs.items():
            z = sorted(p for s in ss for p in range(s.z_offset, s.z_offset + s.nz_local))
            assert z == list(range(nz))
            kx = sorted(c for s in ss for c in range(s.rank * s.kx_block, s.rank * s.kx_block + s.kx_columns))
            assert kx == list(range(partition(nx, nz, 0, 1).kx_columns))


def test_partition_edge_cases():
    with pytest.raises(ValueError):
        partition(16, 6, 0, 4)
    s = [partition(2, 4, r, 4) for r in range(4)]  # Kx = 3 < 4 ranks: one rank owns no kx column
    assert [x.kx_columns for x in s] == [2, 1, 0, 0]  # kx block rounded up to even
    assert partition(1024, 32, 7, 8) == type(s[0])(7, 8, 4, 28, 130, 115)


# ---------------------------------------------------------------- per-component transposes

def _xrow_global(c, z, y, k):
    """A synthetic x-row spectrum value, distinct per (component, z, y, kx)."""
    return complex(1000 * c + 10 * z + y, k + 0.5)


def _worker_transpose(rank, world, port, grid, q):
    """C1 and C2 of the pipelined step on CPU over gloo: per magnetisation component,
    sub-block `comp` of destination block `peer` ([P][3][nzl][ny][Kb]) goes to rank
    `peer`, received into block `rank` of its buffer -- the offsets grace_api.cu's
    alltoall(comp) uses (peer * block + comp * sub)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1411_2565_b200 import dist as gd

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz = grid
    s = gd.partition(nx, nz, rank, world)
    lay = gd.xrow_layout(nx, ny, nz, world)
    kb, nzl, blk, sub = lay["kb"], lay["nz_local"], lay["block"], lay["sub"]
    kx_all = gd.partition(nx, nz, 0, 1).kx_columns
    # K1's output on this rank: destination-blocked x rows of its z slab
    send = np.zeros(world * blk, dtype=np.complex64)
    for dst in range(world):
        for c in range(3):
            for zl in range(nzl):
                for y in range(ny):
                    for j in range(kb):
                        k = dst * kb + j
                        if k < kx_all:
                            send[dst * blk + ((c * nzl + zl) * ny + y) * kb + j] = \
                                _xrow_global(c, s.z_offset + zl, y, k)
    recv = np.zeros_like(send)
    for comp in range(3):  # C1(comp)
        reqs = []
        for peer in range(world):
            off = peer * blk + comp * sub
            if peer == rank:
                recv[off:off + sub] = send[off:off + sub]
                continue
            st = torch.from_numpy(send[off:off + sub].view(np.float32).copy())
            rt = torch.zeros(2 * sub, dtype=torch.float32)
            reqs.append((dist.isend(st, peer), None, None))
            reqs.append((dist.irecv(rt, peer), rt, off))
        for r, rt, off in reqs:
            r.wait()
            if rt is not None:
                recv[off:off + sub] = rt.numpy().view(np.complex64)
    # this rank now holds kx block `rank` for every z: block src = the source slab
    ok1 = True
    for src in range(world):
        for c in range(3):
            for zl in range(nzl):
                for y in range(ny):
                    for j in range(s.kx_columns):
                        want = _xrow_global(c, src * nzl + zl, y, rank * kb + j)
                        ok1 &= recv[src * blk + ((c * nzl + zl) * ny + y) * kb + j] == want
    # C2: the same per-component exchange back restores every rank's own slab
    back = np.zeros_like(send)
    for comp in range(3):
        reqs = []
        for peer in range(world):
            off = peer * blk + comp * sub
            if peer == rank:
                back[off:off + sub] = recv[off:off + sub]
                continue
            st = torch.from_numpy(recv[off:off + sub].view(np.float32).copy())
            rt = torch.zeros(2 * sub, dtype=torch.float32)
            reqs.append((dist.isend(st, peer), None, None))
            reqs.append((dist.irecv(rt, peer), rt, off))
        for r, rt, off in reqs:
            r.wait()
            if rt is not None:
                back[off:off + sub] = rt.numpy().view(np.complex64)
    ok2 = bool(np.array_equal(back, send))
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, bool(ok1), ok2))


@pytest.mark.timeout(120)
@pytest.mark.parametrize("grid", [(16, 6, 4), (10, 3, 8)])
def test_gloo_world2_per_component_transposes(grid):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_transpose, args=(r, world, port, grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    for rank, ok1, ok2 in res:
        assert ok1 and ok2, (rank, ok1, ok2)


def test_comm_schedule_and_overlap_model():
    from paper_1411_2565_b200.dist import comm_schedule, step_time_model, xrow_layout

    sched = comm_schedule(1024, 1024, 32, 8)
    assert [n for n, _, _ in sched] == ["C3 halo", "C1[0]", "C1[1]", "C1[2]", "C2[0]", "C2[1]", "C2[2]"]
    lay = xrow_layout(1024, 1024, 32, 8)
    assert lay["kb"] == 130 and lay["nz_local"] == 4 and lay["block"] == 3 * lay["sub"]
    # C1 of one component: 7 sub-blocks of 4 x 1024 x 130 complex64
    assert sched[1][2] == 7 * 8 * 4 * 1024 * 130
    assert comm_schedule(1024, 1024, 32, 8, pipelined=False)[1] == ("C1", "comm", 3 * sched[1][2])
    assert comm_schedule(64, 64, 8, 1) == []
    # the r02 slab split (ms): pipelining hides part of each transpose; never slower
    kern = {"K1": 0.28, "K2": 0.62, "K3": 1.00, "K4": 0.60, "K5": 0.27, "K6": 0.24}
    N = 1024 * 1024 * 32
    one, _ = step_time_model(kern, N, 1)
    assert abs(one - sum(kern.values())) < 1e-12
    for P in (2, 4, 8):
        t0, e0 = step_time_model(kern, N, P, pipelined=False)
        t1, e1 = step_time_model(kern, N, P)
        assert t1 <= t0 and e1 < e0
        assert t1 >= sum(kern.values()) / P
