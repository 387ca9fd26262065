"""Decode-phase probe: one C3 generation batch (max_new 32, 2 waves) under torch.profiler (CUPTI
kernel timestamps). Kernels shorter than 0.3 ms are the decode regime; prints their per-name
time, launch count, and the idle time between consecutive decode kernels (host-bound launches
show up here, not in the CUDA-event kernel timers)."""
import collections
import os
import sys

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
    mx = int(w.lm.get("max_new_tokens", 32))
    for _ in range(2):
        host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2, max_new=mx)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        host.run_subgcache(ctx, lm, dg, pb, want_logits=False, device_inputs=True, waves=2, max_new=mx)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[0])
    short = 300.0  # us
    per = collections.defaultdict(lambda: [0.0, 0])
    gap_dec, n_dec, busy_dec = 0.0, 0, 0.0
    for i, (a, b, nm) in enumerate(ks):
        if b - a < short and "Memcpy" not in nm and "Memset" not in nm:
            key = nm.replace("void ", "").replace("sgc::(anonymous namespace)::", "")[:60]
            per[key][0] += b - a
            per[key][1] += 1
            busy_dec += b - a
            n_dec += 1
            if i + 1 < len(ks) and ks[i + 1][1] - ks[i + 1][0] < short:
                g = ks[i + 1][0] - b
                if 0 < g < 5000:
                    gap_dec += g
    print(f"decode-regime kernels: {n_dec}, busy {busy_dec / 1e3:.1f} ms, gaps between them {gap_dec / 1e3:.1f} ms")
    for k, (t, n) in sorted(per.items(), key=lambda x: -x[1][0])[:16]:
        print(f"  {t / 1e3:8.2f} ms  {n:6d}  {t / max(n, 1):7.1f} us  {k}")
    span = ks[-1][1] - ks[0][0]
    print(f"span {span / 1e3:.1f} ms")


if __name__ == "__main__":
    main()
