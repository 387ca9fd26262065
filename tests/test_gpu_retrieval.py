"""GPU retrieval (retrieve(), retrieval.cpp:96-239) vs the reference (golden
tests/golden/retrieval.json produced by oracle/_ref): retrieved node/edge sets must be
BIT-EXACT for both strategies, the default and a non-default RetrievalConfig, on the C1
two-star dataset, a seeded community graph and the bundled scene graph."""
import json
import os

import pytest

from paper_2505_10951_b200 import host, workload as W

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _graph(gj):
    return W.TextualGraph({int(n): a.encode("latin1") for n, a in gj["nodes"]},
                          [(int(s), a.encode("latin1"), int(d)) for s, a, d in gj["edges"]])


def test_retrieval_bit_exact_vs_reference(ctx):
    G = gold("retrieval.json")
    scene = gold("scene_graph.json")
    graphs = {name: (_graph(v["graph"]) if "graph" in v else _graph(scene["graph"]), v["questions"], v["dim"])
              for name, v in G["graphs"].items()}
    dgs = {name: host.DeviceGraph(ctx, g) for name, (g, _, _) in graphs.items()}
    checked = 0
    for key, case in G.items():
        if key == "graphs":
            continue
        name = key.split("|")[0]
        _, qs, dim = graphs[name]
        cfg = dict(case["cfg"])
        strategy = cfg.pop("strategy")
        got = host.retrieve(ctx, dgs[name], qs, strategy=strategy, dim=dim, **cfg)
        assert [s.to_json() for s in got] == case["out"], key
        checked += len(got)
    assert checked > 400


def test_c1_retrieval_is_the_injected_input(ctx):
    """The hot path's injected retrieval (workload.c1_workload) equals the GPU retrieval with the
    reference's C1 settings (ego-topk, model_dim 64), which equals the reference's retrieve()."""
    w = W.c1_workload(64, 4)
    dg = host.DeviceGraph(ctx, w.graph)
    got = host.retrieve(ctx, dg, [q.question for q in w.queries], strategy="ego-topk", dim=64)
    assert [s.to_json() for s in got] == [s.to_json() for s in w.retrieved]
    assert [s.to_json() for s in got] == gold("c1_pipeline.json")["retrieved"]


def test_retrieval_config_errors(ctx):
    w = W.c1_workload(4, 2)
    dg = host.DeviceGraph(ctx, w.graph)
    for bad in ({"k": 0}, {"ego_hops": 0}, {"edge_cost": -1.0}):
        with pytest.raises(host.DomainError):
            host.retrieve(ctx, dg, ["engine part 1?"], **bad)
    with pytest.raises(host.DomainError):
        host.retrieve(ctx, dg, ["x"], strategy="bm25")
