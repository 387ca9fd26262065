"""Host-side stall probe: C3 steps as bench.py times them (device inputs, no embeddings out),
with nvidia-smi polling in the background like the bench's clock sampler, and SGC_TRACE_HOST
marks from inside sgc_run_subgcache."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_10951_b200 import host, workload as W
w = W.c3_workload(); ctx = host.Context(0)
lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed)); dg = host.DeviceGraph(ctx, w.graph)
pb = host.PreparedBatch(w, with_own_prefix=True)
smi = None
if os.environ.get("WITH_SMI"):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "200"],
                           stdout=subprocess.DEVNULL)
for i in range(12):
    torch.cuda.synchronize(); t0 = time.time()
    res = host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2, want_embeddings=False)
    torch.cuda.synchronize()
    st = res.stage_ms
    print(f"step {i:2d} wall {1e3 * (time.time() - t0):7.1f} ms  stages {sum(st[:5]):7.1f}  total {st[5]:7.1f}", file=sys.stderr, flush=True)
if smi:
    smi.terminate()
