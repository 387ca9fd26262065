"""Generation (C3, to EOS / max_new) vs the straggler-deferral threshold (sgc_set_option
"decode_defer_pct"): batch time and RT p50."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host, workload as W  # noqa: E402


def main():
    w = W.c3_workload()
    ctx = host.Context(0)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    dg = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w, with_own_prefix=True)
    mx = int(w.lm.get("max_new_tokens", 32))
    waves_list = [int(x) for x in os.environ.get("WAVES", "4").split(",")]
    pcts = [int(x) for x in os.environ.get("PCTS", "25,10,40").split(",")]
    for wv, pct in [(a, b) for a in waves_list for b in pcts] * 2:
        ctx.set_option("decode_defer_pct", pct)
        host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=wv, max_new=mx)
        torch.cuda.synchronize()
        t0 = time.time()
        r = host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=wv, max_new=mx)
        torch.cuda.synchronize()
        ms = (time.time() - t0) * 1e3
        rt = r.rt_ms[r.rt_ms >= 0]
        print(f"waves {wv}  defer {pct:3d}%  batch {ms:8.1f} ms  RT p50 {np.percentile(rt, 50):7.1f}  RT mean {rt.mean():7.1f}")


if __name__ == "__main__":
    main()
