"""torchrun worker for tests/test_gpu_multirank.py: the C1 batch served by WORLD_SIZE ranks that
share the visible GPU(s) (gloo collectives): sharded GNN encode -> all-gather -> redundant
clustering -> LPT cluster ownership -> per-rank serving -> combined first tokens."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2505_10951_b200 import dist as D, host, workload as W  # noqa: E402


def main(out_path, split=False):
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    w = W.c1_workload(64, 4)
    m = len(w.queries)
    ctx = host.Context(dev)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    dg = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w)
    lo, hi = D.shard_range(m, world, rank)
    shard = host.encode_subgraphs(ctx, dg, w.retrieved[lo:hi], pb.gnn)
    emb = D.gather_rows(torch.from_numpy(shard), m, world, dist).numpy()
    res = host.run_subgcache(ctx, lm, dg, pb, embeddings=emb, rank=rank, world_size=world, waves=2,
                             split_clusters=split)
    first = D.combine_first_tokens(torch.from_numpy(res.first_token.astype(np.int64)), dist)
    served = int((res.first_token >= 0).sum())
    mine = torch.from_numpy((res.first_token >= 0).astype(np.int64))
    per_rank = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(per_rank, mine)
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([served], dtype=torch.int64))
    if rank == 0:
        with open(out_path, "w") as f:
            json.dump({"first": first.tolist(), "labels": res.labels.tolist(), "owner": res.owner.tolist(),
                       "served": [int(c.item()) for c in counts],
                       "server": [int(torch.stack(per_rank)[:, q].argmax()) for q in range(m)]}, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], split=len(sys.argv) > 2 and sys.argv[2] == "split")
