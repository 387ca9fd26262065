"""C4 cluster-count sweep quality: first-token agreement of the cached path at
c clusters with the no-cache baseline (c = m: every query prefills its own representative, which
acceptance.cpp:108-124 shows is byte-identical to baseline mode), plus the reuse ratio.

    python scripts/c4_quality.py [m] [c ...]
"""
import dataclasses
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_10951_b200 import host, workload as W  # noqa: E402


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    cs = [int(x) for x in sys.argv[2:]] or [8, 16, 64, 256]
    w0 = W.c4_workload(m=m, clusters=cs[0])
    ctx = host.Context(0)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w0.lm, seed=w0.seed))
    dg = host.DeviceGraph(ctx, w0.graph)
    out = {}
    for c in cs + [m]:
        w = dataclasses.replace(w0, clusters=c)
        pb = host.PreparedBatch(w, with_own_prefix=True)
        t0 = time.time()
        res = host.run_subgcache(ctx, lm, dg, pb, want_logits=False, waves=2)
        dt = time.time() - t0
        plen = [int(x) for x in res.prefix_len]
        cached = sum(plen) + sum(len(q) for q in pb.q)
        base = sum(len(o) + len(q) for o, q in zip(pb.own, pb.q))
        out[c] = {"first": np.asarray(res.first_token).copy(), "reuse": base / cached, "s": dt,
                  "fallbacks": int(np.sum(res.fallback)) if res.fallback is not None else 0}
        print(f"c={c:5d} done in {dt:.1f} s, reuse {base / cached:.2f}x", flush=True)
    ref = out[m]["first"]
    rows = []
    for c in cs:
        agree = float(np.mean(out[c]["first"] == ref))
        rows.append({"clusters": c, "reuse_ratio": round(out[c]["reuse"], 3),
                     "first_token_agreement_vs_c_eq_m": round(agree, 4), "fallbacks": out[c]["fallbacks"]})
        print(json.dumps(rows[-1]))


if __name__ == "__main__":
    main()
