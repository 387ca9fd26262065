"""Pin the CPU restatement (oracle/sgc_oracle.c) to the reference's own outputs.

The golden fixtures were produced by the unmodified reference (tests/golden/make_golden.py);
when oracle/_ref is built here, a few checks also run the reference live."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2505_10951_b200 import workload as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_lm_restatement_vs_reference():
    G = gold("lm_tiny.json")
    lm = oracle.ToyLm(max_seq_len=1024)
    for case, out in zip(G["cases"], G["out"]):
        if out["status"] == 2:
            with pytest.raises(OverflowError):
                lm.prefill(case["prefix"], case.get("soft"))
            continue
        kv = lm.prefill(case["prefix"], case.get("soft"))
        # scalar vs AVX2 reduction order only (test_lm_core.cpp:241-262 allows 2e-4)
        assert np.abs(kv.last_logits - np.array(out["prefix_logits"])).max() <= 2e-4
        if case.get("collect"):  # prefill_collect_logits never takes a soft prefix
            allg = lm.prefill(case["prefix"], collect=True).all_logits
            assert np.abs(allg - np.array(out["all_logits"])).max() <= 2e-4
        if case.get("suffix"):
            lg = lm.extend(kv.fork(), case["suffix"])
            assert np.abs(lg - np.array(out["ext_logits"])).max() <= 2e-4


@pytest.mark.parametrize("name", ["lm_hd64.json", "lm_hd128.json"])
def test_lm_restatement_vs_reference_wide(name):
    G = gold(name)
    c = G["cfg"]
    lm = oracle.ToyLm(c["layers"], c["heads"], c["model_dim"], c["ffn_hidden"], c["max_seq_len"], c["seed"])
    for case, out in zip(G["cases"], G["out"]):
        kv = lm.prefill(case["prefix"])
        assert np.abs(kv.last_logits - np.array(out["prefix_logits"])).max() <= 2e-4
        lg = lm.extend(kv.fork(), case["suffix"])
        assert np.abs(lg - np.array(out["ext_logits"])).max() <= 2e-4


def test_clustering_restatement_bit_exact():
    G = gold("cluster.json")
    for case, out in zip(G["cases"], G["out"]):
        emb = np.array(case["embeddings"], np.float32)
        if out["status"]:
            with pytest.raises(ValueError):
                oracle.agglomerate(emb, case["linkage"], case["c"])
            continue
        labels, left, right, dist, ops = oracle.agglomerate(emb, case["linkage"], case["c"])
        assert labels.tolist() == out["labels"]
        m = np.array(out["merges"]).reshape(-1, 3)
        assert left.tolist() == m[:, 0].astype(int).tolist()
        assert np.array_equal(dist, m[:, 2])
        assert ops == out["op_count"]
        if "pairwise" in out:
            assert np.array_equal(oracle.pairwise(emb).reshape(-1), np.array(out["pairwise"]))
        if "naive_labels" in out:
            nl, nd = oracle.naive_agglomerate(emb, case["linkage"], case["c"])
            assert nl.tolist() == out["naive_labels"]
            assert np.allclose(nd, out["naive_dist"], rtol=1e-12, atol=0)


def test_text_and_gnn_restatement_vs_reference():
    G = gold("scene_graph.json")
    g = G["graph"]
    nodes = {n: a for n, a in g["nodes"]}
    ids = sorted(nodes)
    for dim in (64, 128):
        ref = G[f"gnn_{dim}"]
        proj = oracle.text_projection(dim)
        for t, exp in zip(ref["texts"], ref["out"]["texts"]):
            got = oracle.text_embed(proj, dim, t.encode())
            assert np.array_equal(got, np.array(exp, np.float32))
        w = oracle.gnn_weights(4, 4, dim, ref["seed"])
        feat = {t: oracle.text_embed(proj, dim, t.encode()) for t in ref["texts"]}
        for s, exp in zip(G["subgraphs"][:20], ref["out"]["embeddings"]):
            loc = {n: i for i, n in enumerate(s["nodes"])}
            nf = np.array([feat[nodes[n]] for n in s["nodes"]])
            src = [loc[g["edges"][e][0]] for e in s["edges"]]
            dst = [loc[g["edges"][e][2]] for e in s["edges"]]
            gate = np.array([feat[g["edges"][e][1]] for e in s["edges"]]).reshape(len(s["edges"]), dim)
            got = oracle.gnn_encode(w, 4, 4, dim, nf, src, dst, gate)
            assert np.array_equal(got, np.array(exp, np.float32))


def test_prompt_restatement_vs_reference():
    G = gold("scene_graph.json")
    g = G["graph"]
    nodes = {n: a.encode() for n, a in g["nodes"]}
    nrow = {n: W.render_node_row(n, a) for n, a in nodes.items()}
    erow = [W.render_edge_row(s, a.encode(), d) for s, a, d in g["edges"]]
    for b in G["budgets"]:
        bud = b["budget"]
        res = bud["max_seq_len"] - bud["question_budget"] - bud["max_new_tokens"]
        for cl, out in zip(G["clusters"], b["out"]["clusters"]):
            ns = sorted(set().union(*[G["subgraphs"][i]["nodes"] for i in cl]))
            es = sorted(set().union(*[G["subgraphs"][i]["edges"] for i in cl]))
            assert {"nodes": ns, "edges": es} == out.get("rep", {"nodes": ns, "edges": es})
            if out["status"] == 2:
                with pytest.raises(OverflowError):
                    oracle.build_prefix([nrow[n] for n in ns], [erow[e] for e in es], res)
                continue
            toks, dn, de = oracle.build_prefix([nrow[n] for n in ns], [erow[e] for e in es], res)
            assert toks.tolist() == out["prefix_tokens"]
            assert (dn, de) == (out["dropped_nodes"], out["dropped_edges"])
        for q, exp in zip(["What is the color of the cords?", "x" * 500, ""], b["out"]["questions"]):
            assert oracle.question_tokens(q.encode(), bud["question_budget"]).tolist() == exp


def test_c1_workload_matches_reference_pipeline_inputs():
    G = gold("c1_pipeline.json")
    w = W.c1_workload(64, 4)
    assert [s.to_json() for s in w.retrieved] == G["retrieved"]
    assert [[q.id, q.question.decode(), q.answer.decode()] for q in w.queries] == G["queries"]
    # measured C1 behaviour: clusters 32/30/1/1, prefixes 526/540/540/540
    sizes = np.bincount(G["labels"])
    assert sorted(sizes.tolist(), reverse=True) == [32, 30, 1, 1]
    assert sorted(len(t) for t in G["prefix_tokens"]) == [526, 540, 540, 540]


def test_c1_restatement_end_to_end():
    """The restated pipeline pieces reproduce the reference's C1 labels and logits."""
    G = gold("c1_pipeline.json")
    emb = np.array(G["embeddings"], np.float32)
    labels, *_ = oracle.agglomerate(emb, "ward", 4)
    assert labels.tolist() == G["labels"]
    lm = oracle.ToyLm(seed=7)
    for ci, pt in enumerate(G["prefix_tokens"]):
        kv = lm.prefill(pt)
        q = [i for i, l in enumerate(G["labels"]) if l == ci][0]
        lg = lm.extend(kv.fork(), G["question_tokens"][q])
        assert np.abs(lg - np.array(G["logits"][q])).max() <= 2e-4


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_live_reference_agrees_with_restatement_on_fresh_inputs():
    rng = np.random.default_rng(99)
    emb = rng.uniform(-1, 1, (40, 8)).astype(np.float32)
    out = oracle.run_ref({"cmd": "cluster", "cases": [{"embeddings": emb.tolist(), "linkage": "ward", "c": 3}]})[0]
    assert oracle.agglomerate(emb, "ward", 3)[0].tolist() == out["labels"]
