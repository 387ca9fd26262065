import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2505_10951_b200 import host, workload as W
w = W.c3_workload(); ctx = host.Context(0)
lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed)); dg = host.DeviceGraph(ctx, w.graph)
pb = host.PreparedBatch(w, with_own_prefix=True)
for i in range(25):
    torch.cuda.synchronize(); t0 = time.time()
    res = host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2)
    torch.cuda.synchronize(); t1 = time.time()
    st = res.stage_ms
    print(f"step {i:2d} wall {1e3*(t1-t0):7.1f} ms  stages sum {sum(st[:5]):7.1f} total {st[5]:7.1f}", flush=True)
