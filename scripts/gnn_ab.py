"""A/B of the GNN layer-map GEMM tile (sgc_set_option gnn_tile) on C3's subgraphs: encode time."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host, workload as W  # noqa: E402

w = W.c3_workload()
ctx = host.Context(0)
g = host.DeviceGraph(ctx, w.graph)
pb = host.PreparedBatch(w, with_own_prefix=False)
ref = None
for tile in (0, 1, 2, 0, 1, 2):
    ctx.set_option("gnn_tile", tile)
    host.encode_subgraphs(ctx, g, w.retrieved, pb.gnn)
    ctx.set_timing(True)
    t0 = time.time()
    for _ in range(5):
        e = host.encode_subgraphs(ctx, g, w.retrieved, pb.gnn)
    wall = (time.time() - t0) / 5 * 1e3
    ms, n = ctx.kernel_time("gnn_encode")
    ctx.set_timing(False)
    rows, inst = ctx.gnn_stats()
    ref = e if ref is None else ref
    print(f"tile {tile}: gnn kernels {ms / 5:.2f} ms, wall {wall:.2f} ms, rows {rows}, "
          f"{rows * 2 * 4096**2 / (ms / 5 * 1e-3) / 1e12:.1f} TF/s, max|d| vs first {np.abs(e - ref).max():.2e}")
print("fp64 peak", ctx.fp64_tflops())
