"""world_size-2 gloo run of the multi-GPU host logic on CPU: sharded encode -> all-gather ->
redundant clustering -> LPT ownership -> per-rank serving -> combined first tokens. The GPU
kernels are replaced by the CPU oracle here; the plumbing is the one bench.py uses."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2505_10951_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _embeddings(m, d=16, seed=0):
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(4, d))
    return (centers[np.arange(m) % 4] + 0.05 * rng.normal(size=(m, d))).astype(np.float32)


def _serve(labels, owner, rank):
    # stand-in for sgc_run_subgcache's per-rank output: queries of owned clusters only
    return np.array([(7 * q + 3) % 260 if owner[labels[q]] == rank else -1 for q in range(len(labels))],
                    np.int32)


def _worker(rank, world, port, m, out):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    emb = _embeddings(m)
    lo, hi = D.shard_range(m, world, rank)
    local = torch.from_numpy(emb[lo:hi])  # "encoded" shard
    full = D.gather_rows(local, m, world, dist).numpy()
    labels, *_ = oracle.agglomerate(full, "ward", 4)
    costs = np.bincount(labels, minlength=4).astype(np.float64) * 1000.0 + np.arange(4)
    owner = D.lpt_assign(costs, world)
    first = D.combine_first_tokens(_serve(labels, owner, rank), dist)
    out[rank] = (full.tobytes(), labels.tolist(), owner.tolist(), first.tolist())
    dist.destroy_process_group()


def test_shard_ranges_cover_every_query():
    for m in (1, 7, 64, 1024):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_lpt_is_balanced_and_deterministic():
    rng = np.random.default_rng(3)
    costs = rng.uniform(1, 100, 37)
    own = D.lpt_assign(costs, 8)
    assert own.max() < 8 and np.array_equal(own, D.lpt_assign(costs, 8))
    loads = np.bincount(own, weights=costs, minlength=8)
    assert loads.max() <= costs.sum() / 8 + costs.max()  # LPT bound
    assert np.array_equal(D.lpt_assign(costs, 1), np.zeros(37, np.uint32))


def test_two_rank_gloo_matches_single_process():
    m = 50
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    emb = _embeddings(m)
    labels, *_ = oracle.agglomerate(emb, "ward", 4)
    r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] == emb.tobytes()          # all-gather reassembles rank order exactly
    assert r0[1] == r1[1] == labels.tolist()        # redundant clustering agrees bit-exactly
    assert r0[2] == r1[2]                           # same ownership on every rank
    expected = [(7 * q + 3) % 260 for q in range(m)]
    assert r0[3] == r1[3] == expected               # every query served exactly once


def _balance(prefill, labels, mcost, world):
    import ctypes as C

    from paper_2505_10951_b200 import _lib

    L = _lib.load()
    pc = np.ascontiguousarray(prefill, np.float64)
    lb = np.ascontiguousarray(labels, np.uint32)
    mc = np.ascontiguousarray(mcost, np.float64)
    qo = np.zeros(len(lb), np.uint32)
    co = np.zeros(len(pc), np.uint32)
    _lib.check(L.sgc_balance_members(pc.ctypes.data_as(C.POINTER(C.c_double)), len(pc),
                                     lb.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     mc.ctypes.data_as(C.POINTER(C.c_double)), len(lb), world,
                                     qo.ctypes.data_as(C.POINTER(C.c_uint32)),
                                     co.ctypes.data_as(C.POINTER(C.c_uint32))))
    return qo, co


def _loads(prefill, labels, mcost, qo, world):
    load = np.zeros(world)
    for q, r in enumerate(qo):
        load[r] += mcost[q]
    for c in range(len(prefill)):
        for r in set(int(qo[q]) for q in range(len(labels)) if labels[q] == c):
            load[r] += prefill[c]  # every rank serving part of a cluster prefills it
    return load


def test_member_balance_splits_skewed_clusters_only():
    """a dominant cluster is split across ranks (each receiving rank pays
    a prefix replica); balanced inputs keep whole clusters (the plan degenerates to cluster LPT)."""
    # skewed: one cluster with 600 members, seven with 20
    labels = np.array([0] * 600 + [c for c in range(1, 8) for _ in range(20)])
    prefill = np.full(8, 30.0)
    mcost = np.ones(len(labels))
    for world in (2, 4, 8):
        qo, co = _balance(prefill, labels, mcost, world)
        assert qo.max() < world
        lpt = np.zeros(world)
        cost = prefill + np.bincount(labels, weights=mcost)
        for c in np.argsort(-cost, kind="stable"):
            lpt[np.argmin(lpt)] += cost[c]
        bal = _loads(prefill, labels, mcost, qo, world)
        assert bal.max() < 0.85 * lpt.max()                  # the 600-member cluster got split
        assert bal.max() - bal.min() <= prefill.max() + mcost.max()  # ~even after replicas
        assert len(set(qo[labels == 0].tolist())) >= 2
        assert np.array_equal(qo, _balance(prefill, labels, mcost, world)[0])  # deterministic
    # balanced: 16 equal clusters over 8 ranks -> no member moves, two whole clusters per rank
    labels = np.repeat(np.arange(16), 64)
    qo, co = _balance(np.full(16, 30.0), labels, np.ones(len(labels)), 8)
    for c in range(16):
        assert len(set(qo[labels == c].tolist())) == 1 and qo[labels == c][0] == co[c]
