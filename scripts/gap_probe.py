"""Host-gap probe: one C3 step under torch.profiler (CUPTI kernel timestamps), then the largest
idle gaps between consecutive kernels with the kernels around them."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host, workload as W  # noqa: E402


def main():
    w = W.c3_workload()
    ctx = host.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=w.seed))
    dg = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w, with_own_prefix=True)
    for _ in range(3):
        host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2,
                           verify_prefix=os.environ.get("GAP_NOVERIFY") is None)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2,
                           verify_prefix=os.environ.get("GAP_NOVERIFY") is None)
        torch.cuda.synchronize()
    api = sorted(((e.time_range.end - e.time_range.start, e.name) for e in prof.events()
                  if e.device_type.name == "CPU" and e.name.startswith("cuda")), reverse=True)
    print("longest CUDA runtime calls (host):")
    for dur, nm in api[:12]:
        print(f"  {dur / 1e3:8.3f} ms  {nm}")
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[0])
    print("events", len(ks))
    gaps = []
    for a, b in zip(ks, ks[1:]):
        g = b[0] - a[1]
        if g > 0:
            gaps.append((g, a[2][:60], b[2][:60]))
    tot = sum(g for g, _, _ in gaps)
    span = ks[-1][1] - ks[0][0]
    print(f"span {span / 1e3:.1f} ms, summed gaps {tot / 1e3:.2f} ms over {len(gaps)} gaps")
    for g, a, b in sorted(gaps, reverse=True)[:25]:
        print(f"{g / 1e3:8.3f} ms  after {a}  before {b}")
    # context of the largest gaps: the kernels / copies before and after
    idx = sorted(range(len(ks) - 1), key=lambda i: -(ks[i + 1][0] - ks[i][1]))[:3]
    for i in idx:
        print(f"--- gap {(ks[i + 1][0] - ks[i][1]) / 1e3:.3f} ms at event {i}:")
        for j in range(max(0, i - 6), min(len(ks), i + 6)):
            print(f"   {j:5d} {(ks[j][1] - ks[j][0]) / 1e3:8.3f} ms  {ks[j][2][:90]}")
    small = [g for g, _, _ in gaps if g < 50]
    print(f"gaps < 50 us: {len(small)}, total {sum(small) / 1e3:.2f} ms")


if __name__ == "__main__":
    main()
