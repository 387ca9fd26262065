"""subgcache-report-v1 from a GPU run vs the reference's own run() report (golden
tests/golden/c1_report.json, produced by oracle/_ref running pipeline.cpp:114-320 on the C1
dataset). CPU part: the report arithmetic (dataset digest, integer proxies, answer scoring)
against the golden; GPU part: the whole report of a generation run."""
import json
import os

import pytest

from paper_2505_10951_b200 import report as R, workload as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _c1_files(tmp_path):
    w = W.c1_workload(64, 4)
    w.write_dataset(str(tmp_path))
    return w, {"nodes": str(tmp_path / "nodes.csv"), "edges": str(tmp_path / "edges.csv"),
               "queries": str(tmp_path / "queries.jsonl")}


def test_dataset_digest_and_proxies_match_reference(tmp_path):
    G = gold("c1_report.json")
    w, paths = _c1_files(tmp_path)
    assert R.dataset_digest(paths["nodes"], paths["edges"], paths["queries"], 64) == G["dataset_digest"]
    lm = w.lm
    shape = (lm["layers"], lm["heads"], lm["model_dim"] // lm["heads"], lm["ffn_hidden"])
    for e in G["ledger"]:
        assert R.flop_proxy(0, e["prefix_tokens"], *shape) == e["prefix_flop_proxy"]
    for q, row in zip(w.queries, G["queries"]):
        assert R.score_answer(row["generated"].encode(), q.answer) == row["correct"]
        assert row["pftt_proxy"] == R.flop_proxy(row["context_tokens"] - row["prefill_tokens"],
                                                 row["prefill_tokens"], *shape)
    assert R.agglomerate_op_count(64, lm["model_dim"], 4) == G["cluster_processing"]["cluster_ops"]


def test_compare_rejects_foreign_reports():
    G = gold("c1_report.json")
    other = dict(G, dataset_digest=G["dataset_digest"] ^ 1)
    with pytest.raises(ValueError):
        R.compare(G, other)
    s = R.compare(G, G)
    assert s["proxy"]["rt"] == 1.0 and s["acc_delta_pp"] == 0.0


@pytest.mark.gpu
def test_c1_report_matches_reference_run(ctx, tmp_path):
    from paper_2505_10951_b200 import host

    G = gold("c1_report.json")
    w, paths = _c1_files(tmp_path)
    pb = host.PreparedBatch(w)
    lm = host.ToyLm(ctx, host.ToyLmConfig(**w.lm, seed=7))
    dg = host.DeviceGraph(ctx, w.graph)
    res = host.run_subgcache(ctx, lm, dg, pb, waves=2, max_new=w.lm["max_new_tokens"])
    rep = R.build_report(w, pb, res, paths)
    json.dumps(rep)  # serializable
    assert rep["schema"] == G["schema"] and rep["dataset_digest"] == G["dataset_digest"]
    assert rep["lm_seed"] == G["lm_seed"]
    exact = ("id", "cluster", "fallback", "correct", "generated", "n_generated", "rt_proxy", "ttft_proxy",
             "pftt_proxy", "prefill_tokens", "context_tokens")
    for a, b in zip(rep["queries"], G["queries"]):
        assert {k: a[k] for k in exact} == {k: b[k] for k in exact}
        assert 0 < a["pftt_ms"] <= a["ttft_ms"] <= a["rt_ms"]
    for k in ("m", "n_clusters", "n_fallbacks", "total_prefill_tokens", "total_llm_flop_proxy"):
        assert rep["aggregate"][k] == G["aggregate"][k], k
    for k in ("acc_percent", "mean_rt_proxy", "mean_ttft_proxy", "mean_pftt_proxy"):
        assert rep["aggregate"][k] == pytest.approx(G["aggregate"][k], rel=1e-12), k
    for a, b in zip(rep["ledger"], G["ledger"]):
        for k in ("cluster_id", "prefix_tokens", "prefix_flop_proxy", "hits", "fallbacks"):
            assert a[k] == b[k], k
        assert 0 <= a["seal_ms"] <= a["release_ms"]
        # the sealed prefix's digest (this library's bf16 pages, re-verified after serving)
        if a["hits"] > 0:
            assert a["prefix_digest"] != 0
    for k in ("encode_ops", "cluster_ops", "merge_ops"):
        assert rep["cluster_processing"][k] == G["cluster_processing"][k], k
    s = R.compare(G, rep)  # the reference's compare semantics: CPU report vs GPU report
    assert s["acc_delta_pp"] == 0.0 and s["proxy"]["rt"] == pytest.approx(1.0)
    assert s["wall"]["ttft"] > 0
