"""One C3 encode + clustering + representative build (for ncu captures of the GNN, clustering
and union / prompt kernels): python scripts/prof_embed.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host, workload as W  # noqa: E402

w = W.c3_workload()
ctx = host.Context(0)
ctx.set_option("gnn_tile", int(os.environ.get("GNN_TILE", "1")))
g = host.DeviceGraph(ctx, w.graph)
pb = host.PreparedBatch(w, with_own_prefix=False)
emb = host.encode_subgraphs(ctx, g, w.retrieved, pb.gnn)
a = host.agglomerate(ctx, emb, w.linkage, w.clusters)
reps = host.build_representatives(ctx, g, w.retrieved, a.labels, w.clusters, pb.budget)
print("ok", len(reps.prefix_tokens))
