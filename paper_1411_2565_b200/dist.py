"""Host-side plumbing of the distributed z-slab path.

One process per GPU, launched by torchrun.  torch.distributed is used only for
the plumbing: reading RANK/WORLD_SIZE/LOCAL_RANK, broadcasting libgrace's NCCL
unique id from rank 0, barriers and max-over-ranks timing.  The exchanges of
the step itself (all-to-all transposes as grouped ncclSend/ncclRecv, halo
send/recv on a split communicator) run inside libgrace.

``partition`` restates the slab / kx-block arithmetic of libgrace's
``rank_geom`` (grace_api.cu) so the launcher can hand every rank its slab of a
global array; ``grace_partition`` reports the library's own values and the
tests check the two agree.
"""
import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    nz_local: int
    z_offset: int
    kx_block: int
    kx_columns: int


def padded(n):
    """Padded FFT length: smallest power of two >= 2n - 1, 1 for a singleton axis."""
    if n == 1:
        return 1
    p = 1
    while p < 2 * n - 1:
        p <<= 1
    return p


def partition(nx, nz, rank, nranks):
    """Slab of `rank`: z planes [z_offset, z_offset + nz_local) and kx columns
    [rank*kx_block, rank*kx_block + kx_columns) of the Kx = Px/2 + 1 spectrum."""
    if nranks < 1 or nz % nranks:
        raise ValueError(f"nz = {nz} must be a multiple of the rank count {nranks}")
    px = padded(nx)
    kx = 1 if px == 1 else px // 2 + 1
    if nranks == 1:
        return Slab(rank, 1, nz, 0, 0, kx)
    kb = (kx + nranks - 1) // nranks
    kb += kb & 1  # even, so TMA row strides are 16-byte multiples
    cols = max(0, min(kx, (rank + 1) * kb) - rank * kb)
    nzl = nz // nranks
    return Slab(rank, nranks, nzl, rank * nzl, kb, cols)


def xrow_layout(nx, ny, nz, nranks):
    """Sizes of the destination-blocked x-row layout [P][3][nz/P][ny][Kb] complex that
    K1 writes and the C1 transpose sends (grace_api.cu alltoall): elements per
    block (one destination rank) and per component sub-block."""
    s = partition(nx, nz, 0, nranks)
    kb = s.kx_block if nranks > 1 else s.kx_columns
    sub = s.nz_local * ny * kb
    return {"kb": kb, "nz_local": s.nz_local, "block": 3 * sub, "sub": sub}


def comm_schedule(nx, ny, nz, nranks, pipelined=True):
    """The exchanges of one distributed step in issue order, as libgrace enqueues
    them: (name, stream, bytes sent by one rank).  C3 = the two
    one-plane halos of M (own communicator and stream), C1 = z slabs -> kx blocks
    after K1, C2 = back after K4; pipelined: per magnetisation component."""
    if nranks == 1:
        return []
    lay = xrow_layout(nx, ny, nz, nranks)
    plane = 3 * ny * nx * 4
    out = [("C3 halo", "halo", 2 * plane)]
    per = 8 * lay["sub"] * (nranks - 1)  # one component's sub-block to every other rank
    comps = range(3) if pipelined else [None]
    for name in ("C1", "C2"):
        for q in comps:
            out.append((name if q is None else f"{name}[{q}]", "comm", per * (1 if q is not None else 3)))
    return out


def step_time_model(kernel_ms, cells, nranks, link_GBps=700.0, pipelined=True):
    """Per-step time of the z-slab partition of a grid of `cells` from a
    single-GPU kernel split (kernel_ms: K1..K6 in ms, e.g. the bench line's
    `kernels`) and an all-to-all bandwidth per GPU.  Compute scales as 1/P; one
    transpose sends 24 (P-1)/P^2 bytes per cell from each rank.
    A two-stream event simulation in the order libgrace enqueues the step:
    without pipelining both transposes sit on the critical path; with it C1(q)
    overlaps K1(q+1) and K2(q-1), and C2(q) overlaps K4(q+1) and K5(q-1).  The
    halo exchange (own stream and communicator) is taken as hidden.
    Returns (ms per step, ms of exposed communication)."""
    P = nranks
    k = {n: kernel_ms[n] / P for n in ("K1", "K2", "K3", "K4", "K5", "K6")}
    busy = sum(k.values())
    if P == 1:
        return busy, 0.0
    tr = 24.0 * cells * (P - 1) / (P * P) / (link_GBps * 1e6)  # ms per transpose
    if not pipelined:
        return busy + 2 * tr, 2 * tr
    comp = comm = 0.0  # the step stream's and the communication stream's clocks
    landed = [0.0] * 3
    for q in range(3):  # K1(q) -> C1(q)
        comp += k["K1"] / 3
        comm = max(comm, comp) + tr / 3
        landed[q] = comm
    for q in range(3):  # K2(q) waits for C1(q)
        comp = max(comp, landed[q]) + k["K2"] / 3
    comp += k["K3"]
    for q in range(3):  # K4(q) -> C2(q)
        comp += k["K4"] / 3
        comm = max(comm, comp) + tr / 3
        landed[q] = comm
    for q in range(3):  # K5(q) waits for C2(q)
        comp = max(comp, landed[q]) + k["K5"] / 3
    comp += k["K6"]
    return comp, comp - busy


def env_ranks():
    """(rank, world_size, local_rank) from the torchrun environment (1 process if absent)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def broadcast_bytes(payload, src=0, device=None):
    """Broadcast a bytes object (e.g. the 128-byte NCCL unique id) from `src` over the
    default torch.distributed process group (gloo: CPU tensors; nccl: `device`)."""
    import torch
    import torch.distributed as dist

    n = 128
    t = torch.zeros(n, dtype=torch.uint8, device=device)
    if dist.get_rank() == src:
        b = bytes(payload)
        if len(b) != n:
            raise ValueError("payload must be 128 bytes")
        t.copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().numpy().tobytes())


def create_context(w, rank, nranks, device_index):
    """libgrace context for this rank of the z-slab partition of workload `w`."""
    import torch.distributed as dist

    import paper_1411_2565_b200 as pb

    nid = pb.grace_nccl_unique_id() if rank == 0 else bytes(128)
    if nranks > 1:
        import torch

        nid = broadcast_bytes(nid, 0, device=torch.device("cuda", device_index)
                              if dist.get_backend() == "nccl" else None)
    force = bool(os.environ.get("GRACE_FORCE_NCCL"))  # one-rank NCCL path (plumbing tests)
    return pb.Grace(w.n, w.d, w.Ms, w.A, w.Ku, w.alpha, w.gamma0,
                    dist=(rank, nranks, nid) if (nranks > 1 or force) else None)
