"""Multi-GPU plumbing for the hot path: whole clusters per GPU.

torch.distributed (NCCL on the GPU box, gloo in the CPU tests) carries exactly the two exchanges
the path needs: the all-gather of subgraph embeddings before clustering and the combination of
per-query outputs. Cluster ownership is the library's LPT rule (sgc_lpt_assign), identical on
every rank because the labels are bit-identical.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def shard_range(m: int, world: int, rank: int):
    """Contiguous query shard of rank `rank` (encode is data-parallel over queries)."""
    return (rank * m) // world, ((rank + 1) * m) // world


def gather_rows(local, m: int, world: int, dist, device=None):
    """All-gather row shards of a [m_r x d] tensor into [m x d] in rank order (padded collective)."""
    import torch

    counts = [shard_range(m, world, r)[1] - shard_range(m, world, r)[0] for r in range(world)]
    mx = max(counts)
    d = local.shape[1]
    buf = torch.zeros(mx, d, dtype=local.dtype, device=device or local.device)
    buf[: local.shape[0]] = local
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def combine_first_tokens(first, dist):
    """Every query is served by exactly one rank; unserved entries are -1 -> element-wise MAX."""
    import torch

    t = first if isinstance(first, torch.Tensor) else torch.as_tensor(np.asarray(first, np.int64))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy().astype(np.int32)


class GlooTransport:
    """Host transport for the library's multi-rank path (sgc_comm_init_host) over a
    torch.distributed process group on CPU (gloo): the CPU tests and ranks sharing one GPU."""

    def __init__(self, dist, group=None):
        self.dist, self.group = dist, group

    def allgather(self, send: bytes, nbytes: int) -> bytes:
        import torch

        t = torch.frombuffer(bytearray(send), dtype=torch.uint8) if nbytes else torch.zeros(0, dtype=torch.uint8)
        parts = [torch.zeros(nbytes, dtype=torch.uint8) for _ in range(self.dist.get_world_size(self.group))]
        self.dist.all_gather(parts, t, group=self.group)
        return b"".join(p.numpy().tobytes() for p in parts)

    def exchange(self, sends, recvs):
        import torch

        reqs, outs = [], []
        for data, peer in sends:
            reqs.append(self.dist.isend(torch.frombuffer(bytearray(data), dtype=torch.uint8), peer, group=self.group))
        for nbytes, peer in recvs:
            buf = torch.zeros(nbytes, dtype=torch.uint8)
            outs.append(buf)
            reqs.append(self.dist.irecv(buf, peer, group=self.group))
        for r in reqs:
            r.wait()
        return [b.numpy().tobytes() for b in outs]


def init_library_comm(ctx, dist, backend: str):
    """Join the library context to the process group: NCCL (rank 0's unique id broadcast over
    the group) or the gloo host transport."""
    import torch

    world, rank = dist.get_world_size(), dist.get_rank()
    if backend == "nccl":
        from . import host

        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(host.comm_unique_id()), dtype=torch.uint8)
        obj = [uid.numpy().tobytes()]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_comm_nccl(obj[0], world, rank)
    else:
        ctx.init_comm_host(GlooTransport(dist), world, rank)


def lpt_assign(costs, world: int) -> np.ndarray:
    from . import _lib

    L = _lib.load()
    c = np.ascontiguousarray(costs, np.float64)
    out = np.zeros(len(c), np.uint32)
    _lib.check(L.sgc_lpt_assign(c.ctypes.data_as(C.POINTER(C.c_double)), len(c), world,
                                out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out
