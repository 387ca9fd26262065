"""C3's clustering result and representative prompt lengths, for the CPU reference arm of bench.py
(`--impl reference` cannot embed 1024 subgraphs at d 4096 on the CPU within its time budget).

Runs on a GPU box (the library's encode + agglomerate + build_prompt); the labels are checked
bit-exact against the C restatement of the reference's agglomerate on the same embeddings here
and in tests/test_gpu_fullwidth.py::test_c3_labels_fixture.

    python tests/golden/make_c3_labels.py   (GPU)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2505_10951_b200 import host, workload as W  # noqa: E402

if __name__ == "__main__":
    w = W.c3_workload()
    ctx = host.Context(0)
    g = host.DeviceGraph(ctx, w.graph)
    pb = host.PreparedBatch(w, with_own_prefix=False)
    emb = host.encode_subgraphs(ctx, g, w.retrieved, pb.gnn)
    a = host.agglomerate(ctx, emb, w.linkage, w.clusters)
    ref, *_ = oracle.agglomerate(emb, w.linkage, w.clusters)
    assert np.array_equal(a.labels, ref)
    reps = host.build_representatives(ctx, g, w.retrieved, a.labels, w.clusters, pb.budget)
    out = {"workload": w.name, "clusters": w.clusters, "labels": a.labels.tolist(),
           "prefix_len": [len(t) for t in reps.prefix_tokens]}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3_labels.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("c3 labels", np.bincount(a.labels).tolist(), out["prefix_len"])
