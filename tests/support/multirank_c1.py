"""torchrun worker for tests/test_gpu_multirank.py: the C1 batch served by WORLD_SIZE ranks that
share the visible GPU(s).

Default: the library does the exchanges itself through its host transport over gloo
(sgc_comm_init_host): sharded GNN encode -> all-gather -> redundant clustering -> LPT cluster
ownership (+ member-level splits, optionally with the sealed prefix sent point to point) ->
per-rank serving -> outputs gathered to rank 0. Mode "py": the caller-driven path (embeddings
all-gathered in Python, first tokens combined with an all-reduce)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2505_10951_b200 import dist as D, host, workload as W  # noqa: E402


def main(out_path, modes):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    split = "split" in modes or "transfer" in modes
    w = W.c1_workload(64, 4)
    m = len(w.queries)
    ctx = host.Context(dev)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    dg = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w)
    gen = 32 if "gen" in modes else 0
    if "py" in modes:
        lo, hi = D.shard_range(m, world, rank)
        shard = host.encode_subgraphs(ctx, dg, w.retrieved[lo:hi], pb.gnn)
        emb = D.gather_rows(torch.from_numpy(shard), m, world, dist).numpy()
        res = host.run_subgcache(ctx, lm, dg, pb, embeddings=emb, rank=rank, world_size=world, waves=2,
                                 split_clusters=split)
        first = D.combine_first_tokens(torch.from_numpy(res.first_token.astype(np.int64)), dist).tolist()
    else:
        D.init_library_comm(ctx, dist, "gloo")
        res = host.run_subgcache(ctx, lm, dg, pb, waves=2, split_clusters=split,
                                 transfer_prefix=2 if "transfer" in modes else 1, max_new=gen)
        first = res.first_token.tolist()
    sent = torch.tensor([res.prefix_bytes_sent, res.prefix_bytes_received], dtype=torch.int64)
    moved = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(moved, sent)
    pref = torch.from_numpy(res.prefilled.astype(np.int64))
    pref_all = [torch.zeros_like(pref) for _ in range(world)]
    dist.all_gather(pref_all, pref)
    if rank == 0:
        qr = res.query_rank.tolist()
        with open(out_path, "w") as f:
            json.dump({"first": first, "labels": res.labels.tolist(), "owner": res.owner.tolist(),
                       "served": [qr.count(r) for r in range(world)], "server": qr,
                       "ttft": res.ttft_ms.tolist(), "prefix_len": res.prefix_len.tolist(),
                       "logits": res.logits.tolist() if res.logits is not None else None,
                       "tokens": [t.tolist() for t in res.tokens] if res.tokens is not None else None,
                       "moved": [x.tolist() for x in moved],
                       "prefilled": [p.tolist() for p in pref_all]}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], set(sys.argv[2:]))
