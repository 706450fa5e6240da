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
