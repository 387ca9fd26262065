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


def lpt_assign(costs, world: int) -> np.ndarray:
    from . import _lib

    L = _lib.load()
    c = np.ascontiguousarray(costs, np.float64)
    out = np.zeros(len(c), np.uint32)
    _lib.check(L.sgc_lpt_assign(c.ctypes.data_as(C.POINTER(C.c_double)), len(c), world,
                                out.ctypes.data_as(C.POINTER(C.c_uint32))))
    return out
