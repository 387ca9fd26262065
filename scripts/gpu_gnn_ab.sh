#!/bin/bash
# GNN layer-map GEMM A/B at C3 (gnn_tile 1 = DFMA 64x128 register tiles, 3 = DMMA m16n8k4), with
# the dedup on (the bench default) and off; embeddings compared bit-for-bit across the two
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullwidth.py -q -x -k "gnn or labels or pipeline" --timeout 200 2>&1 | tail -2
python - <<'P'
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2505_10951_b200 import host, workload as W
w = W.c3_workload(); ctx = host.Context(0)
dg = host.DeviceGraph(ctx, w.graph); pb = host.PreparedBatch(w, with_own_prefix=False)
print("fp64 peak (max DFMA, DMMA):", round(ctx.fp64_tflops(), 2))
res = {}
for tile in (1, 3):
    ctx.set_option("gnn_tile", tile)
    for dd in (1, 0):
        ctx.set_option("gnn_dedup", dd)
        host.encode_subgraphs(ctx, dg, w.retrieved, pb.gnn)
        ctx.set_timing(True)
        for _ in range(3): e = host.encode_subgraphs(ctx, dg, w.retrieved, pb.gnn)
        ms, n = ctx.kernel_time("gnn_encode"); rows, inst = ctx.gnn_stats(); ctx.set_timing(False)
        fl = rows * 2.0 * 4096 * 4096
        res[(tile, dd)] = e
        print(f"tile {tile} dedup {dd}: {ms/3:.2f} ms/encode, {fl/(ms/3/1e3)/1e12:.2f} TFLOP/s")
    ctx.set_option("gnn_dedup", 1)
print("max |emb dfma - emb dmma|:", float(np.abs(res[(1,1)] - res[(3,1)]).max()), "dedup exact:", bool(np.array_equal(res[(3,1)], res[(3,0)])))
P
