"""Host-side plumbing of the distributed z-slab path.

One process per GPU, launched by torchrun.  torch.distributed is used only for
the plumbing: reading RANK/WORLD_SIZE/LOCAL_RANK, broadcasting libgrace's NCCL
unique id from rank 0, barriers and max-over-ranks timing.  The exchanges of
the step itself (ncclAlltoAll transposes, halo send/recv) run inside libgrace.

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
