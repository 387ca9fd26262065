"""subgcache-report-v1 / cache ledger emitted by a GPU run.

The reference's `run()` writes a JSON report (`BatchReport::to_json`, pipeline.cpp:388-452) and a
ledger (`CacheLedger::to_json`, cache_engine.cpp:235-251); `compare --base a.json --treat b.json`
(`compare_reports`, pipeline.cpp:538-556) turns two reports of the same dataset and LM seed into
a speed-up table. This module builds the same document from a `SubgCacheResult` produced with
generation on (`run_subgcache(..., max_new=ToyLmConfig::max_new_tokens)`) so a CPU report of the
reference and a GPU report of this library compare unchanged:

* integer proxies (`flop_proxy`, cost_model.hpp:24-29) are exact -- same token counts, same
  formula; PFTT/TTFT/RT proxies follow `finish_outcome` / `process_cluster`
  (cache_engine.cpp:76-108, :140-215): the representative's prefill proxy is charged to the
  cluster's first member, the decode proxy is one `flop_proxy(context, 1)` per extended token;
* wall times are the GPU run's (submission -> first / last token per query, device events);
* `correct` is `score_answer` (pipeline.cpp:60-79) on the detokenized generation;
* `dataset_digest` is `file_digest` over the dataset files (pipeline.cpp:27-35, :125-128);
* `prefix_digest` / `resident_kv_bytes` describe this library's bf16 KV (the reference hashes its
  fp32 KV, so digests are comparable only run-to-run, not across implementations).
"""
from __future__ import annotations

import json

import numpy as np

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
MASK = (1 << 64) - 1
EOS = 257


def fnv1a64(data: bytes, h: int = FNV_OFFSET) -> int:
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & MASK
    return h


def file_digest(path: str, h: int) -> int:
    """pipeline.cpp:27-35."""
    with open(path, "rb") as f:
        return fnv1a64(f.read(), h)


def dataset_digest(nodes_csv: str, edges_csv: str, queries_jsonl: str, m: int) -> int:
    """pipeline.cpp:125-128 (queries truncated to the batch size before the count is hashed)."""
    h = file_digest(nodes_csv, FNV_OFFSET)
    h = file_digest(edges_csv, h)
    h = file_digest(queries_jsonl, h)
    return fnv1a64(str(m).encode(), h)


def flop_proxy(prefix_cached: int, new_tokens: int, layers: int, heads: int, head_dim: int,
               ffn_hidden: int) -> int:
    """cost_model.hpp:24-29 (pure integers)."""
    attention = new_tokens * (prefix_cached + new_tokens) * heads * head_dim * layers
    ffn = new_tokens * (2 * heads * head_dim * ffn_hidden) * layers
    return attention + ffn


def normalize_answer(text: bytes) -> bytes:
    """pipeline.cpp:60-73."""
    out = bytearray()
    pending = False
    for c in text:
        if (48 <= c <= 57) or (65 <= c <= 90) or (97 <= c <= 122) or c >= 0x80:
            if pending and out:
                out += b" "
            pending = False
            out.append(c + 32 if 65 <= c <= 90 else c)
        else:
            pending = True
    return bytes(out)


def score_answer(generated: bytes, gold: bytes) -> bool:
    """pipeline.cpp:75-79."""
    return normalize_answer(gold) in normalize_answer(generated)


def detokenize(tokens) -> bytes:
    """tokenizer.cpp:20-27: byte tokens only."""
    return bytes(int(t) for t in tokens if 0 <= int(t) < 256)


def encode_ops_of(n_nodes: int, n_edges: int, layers: int, heads: int, dim: int) -> int:
    """pipeline.cpp:37-42."""
    return layers * (n_nodes * heads * dim * dim + 2 * n_edges * dim)


def agglomerate_op_count(m: int, dim: int, c: int) -> int:
    """clustering.cpp:71,99,130 op proxy (distance evals + scanned pairs + recurrence updates)."""
    ops = m * (m - 1) // 2 * dim
    for a in range(m, c, -1):
        ops += a * (a - 1) // 2 + (a - 2)
    return ops


def _json_text(b: bytes) -> str:
    # nlohmann dump(..., error_handler_t::replace): invalid UTF-8 -> U+FFFD
    return b.decode("utf-8", errors="replace")


def build_report(w, pb, res, paths: dict, cfg_extra: dict | None = None) -> dict:
    """subgcache-report-v1 for a SubgCache run of workload `w` (host.PreparedBatch `pb`, result
    `res` from run_subgcache with max_new > 1). `paths` = {"nodes", "edges", "queries"} of the
    dataset files the reference run reads (digest)."""
    if res.tokens is None:
        raise ValueError("build_report needs a run with generation (max_new > 1)")
    lm = w.lm
    L, H, d, ffn = lm["layers"], lm["heads"], lm["model_dim"], lm["ffn_hidden"]
    hd = d // H
    mx_seq, mx_new = lm["max_seq_len"], lm["max_new_tokens"]
    m, k = len(w.queries), w.clusters
    soft = 1 if w.soft_prefix else 0

    def proxy(prefix, new):
        return flop_proxy(prefix, new, L, H, hd, ffn)

    labels = [int(x) for x in res.labels]
    plen = [int(x) for x in res.prefix_len]  # incl. the soft slot
    members = [[] for _ in range(k)]
    for q in range(m):
        members[labels[q]].append(q)
    rows, total_prefill, total_proxy = [], 0, 0
    hits, fbs = [0] * k, [0] * k
    for q in range(m):
        c = labels[q]
        toks = [int(t) for t in res.tokens[q]]
        S = len(pb.q[q])
        fb = bool(res.fallback[q])
        if fb:
            allowed = mx_seq - min(mx_seq, mx_new + soft)
            total = min(len(pb.own[q]) + S, allowed) + soft
            context, own_tokens = total, total
            pftt_p = proxy(0, total)
            ttft_p = pftt_p
            fbs[c] += 1
        else:
            context, own_tokens = plen[c] + S, S
            pftt_p = proxy(plen[c], S)
            ttft_p = pftt_p + (proxy(0, plen[c]) if members[c][0] == q else 0)
            hits[c] += 1
        decode_p = sum(proxy(context + t, 1) for t in range(len(toks) - 1))
        gen = detokenize(toks)
        rows.append({"id": w.queries[q].id, "cluster": c, "fallback": fb,
                     "correct": bool(score_answer(gen, w.queries[q].answer)),
                     "generated": _json_text(gen), "n_generated": len(toks),
                     "rt_ms": float(res.rt_ms[q]), "ttft_ms": float(res.ttft_ms[q]),
                     "pftt_ms": float(res.pftt_ms[q]) if res.pftt_ms is not None else 0.0,
                     "rt_proxy": ttft_p + decode_p, "ttft_proxy": ttft_p, "pftt_proxy": pftt_p,
                     "prefill_tokens": own_tokens, "context_tokens": context})
        total_prefill += own_tokens
        total_proxy += pftt_p + decode_p
    ledger = []
    for c in range(k):
        release = max((res.rt_ms[q] for q in members[c]), default=-1.0)
        ledger.append({"cluster_id": c, "seal_ms": float(res.seal_ms[c]) if res.seal_ms is not None else 0.0,
                       "release_ms": float(release),
                       "resident_kv_bytes": plen[c] * L * 2 * d * 2,  # bf16 K/V of the sealed prefix
                       "prefix_tokens": plen[c], "prefix_flop_proxy": proxy(0, plen[c]),
                       "prefix_digest": int(res.prefix_digest[c]) if res.prefix_digest is not None else 0,
                       "hits": hits[c], "fallbacks": fbs[c]})
        total_prefill += plen[c]
        total_proxy += proxy(0, plen[c])
    n = float(m)
    agg = {"m": m, "n_clusters": k, "n_fallbacks": int(sum(fbs)),
           "acc_percent": 100.0 * sum(r["correct"] for r in rows) / n,
           "mean_rt_ms": sum(r["rt_ms"] for r in rows) / n,
           "mean_ttft_ms": sum(r["ttft_ms"] for r in rows) / n,
           "mean_pftt_ms": sum(r["pftt_ms"] for r in rows) / n,
           "mean_rt_proxy": sum(r["rt_proxy"] for r in rows) / n,
           "mean_ttft_proxy": sum(r["ttft_proxy"] for r in rows) / n,
           "mean_pftt_proxy": sum(r["pftt_proxy"] for r in rows) / n,
           "total_prefill_tokens": total_prefill, "total_llm_flop_proxy": total_proxy}
    gnn_layers, gnn_heads = pb.gnn.layers, pb.gnn.heads
    enc_ops = sum(encode_ops_of(len(s.node_ids), len(s.edge_indices), gnn_layers, gnn_heads, d)
                  for s in w.retrieved)
    merge_ops = sum(len(s.node_ids) + len(s.edge_indices) for s in w.retrieved)
    cp = {"retrieval_ms": 0.0, "encode_ms": float(res.stage_ms[0]), "cluster_ms": float(res.stage_ms[1]),
          "merge_ms": float(res.stage_ms[2]), "encode_ops": enc_ops,
          "cluster_ops": agglomerate_op_count(m, d, k), "merge_ops": merge_ops}
    from . import workload as W

    config = {"graph_nodes": paths["nodes"], "graph_edges": paths["edges"], "queries": paths["queries"],
              "undirected": bool(w.undirected), "mode": "subgcache", "batch_size": m,
              "retrieval": dict(w.retrieval),
              "cluster": {"linkage": w.linkage, "count": k},
              "lm": {"layers": L, "heads": H, "model_dim": d, "ffn_hidden": ffn, "max_seq": mx_seq,
                     "max_new": mx_new},
              "effective_seeds": {"lm": w.seed, "gnn": W.splitmix64_once(w.seed ^ 0x62),
                                  "text_encoder": w.text_encoder_seed, "hash_salt": w.hash_salt},
              "question_budget": w.question_budget, "seed": w.seed,
              "soft_prefix": "on" if w.soft_prefix else "off", "answer_lookup": bool(w.answer_lookup),
              "parallel_queries": False, "kernel_backend": "b200-sm100a"}  # one batched GPU pass
    if cfg_extra:
        config.update(cfg_extra)
    return {"schema": "subgcache-report-v1", "mode": "subgcache",
            "dataset_digest": dataset_digest(paths["nodes"], paths["edges"], paths["queries"], m),
            "lm_seed": w.seed, "config": config, "aggregate": agg, "cluster_processing": cp,
            "queries": rows, "ledger": ledger}


def ledger_json(report: dict) -> str:
    """CacheLedger::to_json (cache_engine.cpp:235-251)."""
    return json.dumps(report["ledger"], indent=2)


def compare(base: dict, treat: dict) -> dict:
    """compare_reports + SpeedupTable::to_json (pipeline.cpp:538-566)."""
    if base["dataset_digest"] != treat["dataset_digest"]:
        raise ValueError("compare: reports were produced from different datasets")
    if base["lm_seed"] != treat["lm_seed"]:
        raise ValueError("compare: reports use different LM seeds")
    a, b = base["aggregate"], treat["aggregate"]

    def ratio(x, y):
        return x / y if y > 0 else 0.0

    return {"acc_delta_pp": b["acc_percent"] - a["acc_percent"],
            "wall": {"rt": ratio(a["mean_rt_ms"], b["mean_rt_ms"]),
                     "ttft": ratio(a["mean_ttft_ms"], b["mean_ttft_ms"]),
                     "pftt": ratio(a["mean_pftt_ms"], b["mean_pftt_ms"])},
            "proxy": {"rt": ratio(a["mean_rt_proxy"], b["mean_rt_proxy"]),
                      "ttft": ratio(a["mean_ttft_proxy"], b["mean_ttft_proxy"]),
                      "pftt": ratio(a["mean_pftt_proxy"], b["mean_pftt_proxy"])}}
