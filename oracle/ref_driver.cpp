// ref_driver.cpp -- drives the UNMODIFIED reference library (oracle/_ref/libsubgcache_ref.so,
// compiled from /root/reference/proj/src) through its public C++ API.
//
// TEST INFRASTRUCTURE / CPU BASELINE ONLY. Two uses:
//   * golden-vector generation for tests/golden (tests/golden/make_golden.py), and
//   * the reference arm of bench.py (`--impl reference`): the reference's own CPU path
//     timed on the host cores.
//
// Usage: ref_driver <spec.json> <out.json>. The spec's "cmd" selects:
//   lm        ToyLm::prefill / seal / fork / extend / prefill_collect_logits / greedy_decode
//   lm_cluster prefill + seal per cluster, fork + extend per member (threaded), any shape
//   cluster   pairwise_distances + agglomerate (+ naive oracle from tests/support)
//   gnn       TextEncoder::embed + GnnEncoder::encode over a CSV graph and subgraph lists
//   prompt    merge_subgraphs + build_prompt + Tokenizer over a CSV graph
//   pipeline  retrieve -> build_prompt -> encode -> agglomerate -> merge -> run_batch
//             (the SubgCache branch of pipeline.cpp:212-293, stage by stage, with timings)
//   bench     bounded timing samples of each hot-path stage at a given model shape
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <future>
#include <iostream>
#include <thread>

#include <nlohmann/json.hpp>

#include "subgcache/cache_engine.hpp"
#include "subgcache/clustering.hpp"
#include "subgcache/encoders.hpp"
#include "subgcache/errors.hpp"
#include "subgcache/graph_store.hpp"
#include "subgcache/lm_core.hpp"
#include "subgcache/pipeline.hpp"
#include "subgcache/retrieval.hpp"
#include "subgcache/rng.hpp"
#include "subgcache/tokenizer.hpp"
#include "support/cluster_oracle.hpp"
#include "support/synth.hpp"

using json = nlohmann::json;
using namespace subgcache;
using Clock = std::chrono::steady_clock;

namespace {

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

ToyLmConfig lm_cfg(const json& j) {
    ToyLmConfig c;
    c.layers = j.value("layers", c.layers);
    c.heads = j.value("heads", c.heads);
    c.model_dim = j.value("model_dim", c.model_dim);
    c.ffn_hidden = j.value("ffn_hidden", c.ffn_hidden);
    c.max_seq_len = j.value("max_seq_len", c.max_seq_len);
    c.max_new_tokens = j.value("max_new_tokens", c.max_new_tokens);
    c.seed = j.value("seed", c.seed);
    return c;
}

std::vector<TokenId> toks(const json& j) { return j.get<std::vector<TokenId>>(); }

Subgraph subgraph_of(const TextualGraph& g, const json& j) {
    Subgraph s;
    s.parent = &g;
    for (auto id : j.at("nodes")) s.node_ids.insert(id.get<NodeId>());
    for (auto e : j.at("edges")) s.edge_indices.insert(e.get<uint32_t>());
    return s;
}

json subgraph_json(const Subgraph& s) {
    return json{{"nodes", std::vector<NodeId>(s.node_ids.begin(), s.node_ids.end())},
                {"edges", std::vector<uint32_t>(s.edge_indices.begin(), s.edge_indices.end())}};
}

json cmd_lm(const json& spec) {
    ToyLm lm(lm_cfg(spec.at("cfg")));
    json out = json::array();
    for (const json& c : spec.at("cases")) {
        json r;
        std::vector<TokenId> prefix = toks(c.at("prefix"));
        std::vector<float> soft;
        if (c.contains("soft") && !c["soft"].is_null()) soft = c["soft"].get<std::vector<float>>();
        try {
            KVCache kv = lm.prefill(prefix, soft);
            r["prefix_logits"] = kv.last_logits();
            kv.seal();
            r["prefix_digest"] = std::to_string(kv.prefix_digest());
            r["prefix_tokens"] = kv.token_count();
            if (c.contains("suffix")) {
                KVCache f = kv.fork();
                std::vector<TokenId> suffix = toks(c.at("suffix"));
                lm.extend(f, suffix);
                r["ext_logits"] = f.last_logits();
                if (c.value("decode", 0) > 0) {
                    DecodeOptions o;
                    if (c.contains("answer")) {
                        o.hint = CopyPointerHint{toks(c["answer"]), kv.prefix_token_count(),
                                                 c.value("bonus", 100.0f)};
                    }
                    if (c.value("margins", false)) {
                        // the same greedy loop through the public API (lm_core.cpp:376-398), recording
                        // each step's biased top-1 / top-2 logit margin (robustness of the argmax)
                        KVCache f2 = kv.fork();
                        lm.extend(f2, suffix);
                        json mg = json::array();
                        for (size_t t = 0; t < c["decode"].get<size_t>(); ++t) {
                            std::vector<float> lg = f2.last_logits();
                            std::vector<float> s = lg;
                            std::sort(s.begin(), s.end());
                            mg.push_back(s[s.size() - 1] - s[s.size() - 2]);
                            TokenId b = greedy_argmax(lg);
                            if (b == Tokenizer::kEos || f2.token_count() + 1 > lm.config().max_seq_len) break;
                            TokenId nx[1] = {b};
                            lm.extend(f2, nx);
                        }
                        r["decode_margins"] = mg;
                    }
                    GenerationResult g = lm.greedy_decode(f, c["decode"].get<size_t>(), o);
                    r["decode"] = g.token_ids;
                }
            }
            if (c.value("collect", false)) r["all_logits"] = lm.prefill_collect_logits(prefix);
            r["status"] = 0;
        } catch (const CapacityError& e) {
            r["status"] = 2;
            r["error"] = e.what();
        } catch (const DomainError& e) {
            r["status"] = 1;
            r["error"] = e.what();
        }
        out.push_back(r);
    }
    return out;
}


// process_cluster's KV lifecycle (cache_engine.cpp:140-215) at an arbitrary model shape, for
// the full-width parity fixtures: prefill each cluster's prefix, seal, then fork + extend every
// member (answer lookup off: plain greedy_argmax). Clusters prefill concurrently and members
// extend concurrently (ToyLm const methods are safe on distinct forks, lm_core.hpp:118-121),
// bounded by "threads"; the arithmetic is the reference's own.
json cmd_lm_cluster(const json& spec) {
    ToyLm lm(lm_cfg(spec.at("cfg")));
    const json& cl = spec.at("clusters");
    size_t threads = std::max<size_t>(1, spec.value("threads", std::thread::hardware_concurrency()));
    size_t nc = cl.size();
    std::vector<KVCache> shared(nc);
    std::vector<json> out(nc);
    auto run_bounded = [&](size_t n, auto&& fn) {
        for (size_t b = 0; b < n; b += threads) {
            std::vector<std::future<void>> fs;
            for (size_t i = b; i < std::min(n, b + threads); ++i)
                fs.push_back(std::async(std::launch::async, [&, i] { fn(i); }));
            for (auto& f : fs) f.get();
        }
    };
    auto t0 = Clock::now();
    run_bounded(nc, [&](size_t c) {
        shared[c] = lm.prefill(toks(cl[c].at("prefix")));
        out[c]["prefix_logits"] = shared[c].last_logits();
        shared[c].seal();
        out[c]["prefix_digest"] = std::to_string(shared[c].prefix_digest());
        out[c]["prefix_tokens"] = shared[c].token_count();
    });
    double prefill_ms = ms_since(t0);
    std::vector<std::pair<size_t, size_t>> work;
    for (size_t c = 0; c < nc; ++c) {
        out[c]["members"] = json::array();
        for (size_t j = 0; j < cl[c].at("members").size(); ++j) {
            work.emplace_back(c, j);
            out[c]["members"].push_back(nullptr);
        }
    }
    std::vector<json> res(work.size());
    t0 = Clock::now();
    run_bounded(work.size(), [&](size_t w) {
        auto [c, j] = work[w];
        KVCache f = shared[c].fork();
        std::vector<float> lg = lm.extend(f, toks(cl[c]["members"][j]));
        std::vector<float> s = lg;
        std::sort(s.begin(), s.end());
        res[w] = json{{"logits", lg}, {"margin", s[s.size() - 1] - s[s.size() - 2]},
                      {"argmax", greedy_argmax(lg)}};
    });
    double extend_ms = ms_since(t0);
    for (size_t w = 0; w < work.size(); ++w) out[work[w].first]["members"][work[w].second] = res[w];
    return json{{"clusters", out}, {"prefill_ms", prefill_ms}, {"extend_ms", extend_ms},
                {"threads", threads}};
}

Linkage linkage_of(const json& spec) { return linkage_from_string(spec.value("linkage", "ward")); }

json cmd_cluster(const json& spec) {
    json out = json::array();
    for (const json& c : spec.at("cases")) {
        std::vector<EmbeddingVec> emb;
        if (c.contains("embeddings_f32")) {  // raw row-major float32 [m x d] (large fixtures)
            size_t m = c.at("m"), d = c.at("d");
            std::ifstream bin(c["embeddings_f32"].get<std::string>(), std::ios::binary);
            emb.assign(m, EmbeddingVec(d));
            for (auto& e : emb) bin.read(reinterpret_cast<char*>(e.data()), d * sizeof(float));
            if (!bin) throw std::runtime_error("short embeddings_f32 file");
        } else {
            emb = c.at("embeddings").get<std::vector<EmbeddingVec>>();
        }
        json r;
        try {
            if (c.value("pairwise", false)) r["pairwise"] = pairwise_distances(emb);
            Linkage lk = linkage_from_string(c.value("linkage", "ward"));
            ClusterAssignment a = agglomerate(emb, {lk, c.at("c").get<uint32_t>()});
            r["labels"] = a.labels;
            json merges = json::array();
            for (const MergeStep& st : a.merges) {
                merges.push_back({st.left.front(), st.right.front(), st.distance});
            }
            r["merges"] = merges;
            r["op_count"] = a.op_count;
            if (c.value("naive", false)) {
                auto o = testsupport::naive_agglomerate(emb, lk, c.at("c").get<uint32_t>());
                r["naive_labels"] = o.labels;
                r["naive_dist"] = o.merge_distances;
            }
            r["status"] = 0;
        } catch (const DomainError& e) {
            r["status"] = 1;
            r["error"] = e.what();
        }
        out.push_back(r);
    }
    return out;
}

TextualGraph graph_of(const json& spec) {
    return load_graph_csv(spec.at("nodes_csv"), spec.at("edges_csv"), spec.value("undirected", false));
}

json cmd_gnn(const json& spec) {
    TextualGraph g = graph_of(spec);
    TextEncoderConfig tc;
    tc.dim = spec.at("dim");
    TextEncoder enc(tc);
    GnnEncoderConfig gc;
    gc.dim = spec.at("dim");
    gc.seed = spec.at("gnn_seed").get<uint64_t>();
    GnnEncoder gnn(gc);
    json out;
    json texts = json::array();
    for (const json& t : spec.value("texts", json::array())) texts.push_back(enc.embed(t.get<std::string>()));
    out["texts"] = texts;
    json embs = json::array();
    for (const json& s : spec.at("subgraphs")) {
        try {
            embs.push_back(gnn.encode(enc, subgraph_of(g, s)));
        } catch (const DomainError&) {
            embs.push_back(nullptr);
        }
    }
    out["embeddings"] = embs;
    return out;
}

json cmd_prompt(const json& spec) {
    TextualGraph g = graph_of(spec);
    const json& b = spec.at("budget");
    PromptBudget budget{b.at("max_seq_len"), b.at("question_budget"), b.at("max_new_tokens"),
                        b.value("soft", false)};
    PromptTemplate tmpl;
    std::vector<Subgraph> subs;
    for (const json& s : spec.at("subgraphs")) subs.push_back(subgraph_of(g, s));
    json out = json::array();
    for (const json& cl : spec.at("clusters")) {
        json r;
        std::vector<Subgraph> parts;
        for (auto i : cl) parts.push_back(subs.at(i.get<size_t>()));
        try {
            Subgraph rep = merge_subgraphs(parts);
            r["rep"] = subgraph_json(rep);
            PromptParts p = build_prompt(tmpl, rep, "", budget);
            r["prefix_tokens"] = Tokenizer::tokenize(p.prefix_text);
            r["dropped_nodes"] = p.dropped_node_rows;
            r["dropped_edges"] = p.dropped_edge_rows;
            r["status"] = 0;
        } catch (const CapacityError& e) {
            r["status"] = 2;
            r["error"] = e.what();
        } catch (const DomainError& e) {
            r["status"] = 1;
            r["error"] = e.what();
        }
        out.push_back(r);
    }
    json qs = json::array();
    for (const json& q : spec.value("questions", json::array())) {
        PromptParts p = build_prompt(tmpl, subs.empty() ? Subgraph{&g, {}, {}} : subs[0],
                                     q.get<std::string>(), budget);
        qs.push_back(Tokenizer::encode_bytes(p.question_text));
    }
    return json{{"clusters", out}, {"questions", qs}};
}

// The SubgCache branch of run() (pipeline.cpp:212-293), stage by stage through the
// reference API, exposing the intermediates that run() keeps private.
json cmd_pipeline(const json& spec) {
    TextualGraph g = graph_of(spec);
    std::vector<QueryRecord> queries = load_queries_jsonl(spec.at("queries_jsonl"));
    uint64_t seed = spec.value("seed", 7ull);
    ToyLmConfig lc = lm_cfg(spec.value("lm", json::object()));
    lc.seed = seed;
    bool answer_lookup = spec.value("answer_lookup", true);
    uint32_t c = spec.at("clusters");
    Linkage lk = linkage_of(spec);
    RetrievalConfig rc;
    std::string strat = spec.value("retrieval", "ego-topk");
    rc.strategy = strat == "ego-topk" ? RetrievalStrategy::EgoTopK : RetrievalStrategy::NodeEdgeTopK;
    bool soft_on = spec.value("soft", false);

    TextEncoderConfig tc;
    tc.dim = lc.model_dim;
    TextEncoder enc(tc);
    GnnEncoderConfig gc;
    gc.dim = lc.model_dim;
    gc.seed = splitmix64_once(seed ^ 0x62);
    GnnEncoder gnn(gc);
    ToyLm lm(lc);
    PromptTemplate tmpl;
    PromptBudget budget{lc.max_seq_len, spec.value("question_budget", 128u), lc.max_new_tokens,
                        soft_on};

    json out;
    std::vector<Subgraph> retrieved;
    if (spec.contains("retrieved")) {
        for (const json& s : spec["retrieved"]) retrieved.push_back(subgraph_of(g, s));
    } else {
        for (const QueryRecord& q : queries) retrieved.push_back(retrieve(rc, g, q, enc));
    }
    json rj = json::array();
    for (const Subgraph& s : retrieved) rj.push_back(subgraph_json(s));
    out["retrieved"] = rj;

    std::vector<std::vector<TokenId>> qtok(queries.size()), atok(queries.size()),
        own(queries.size());
    for (size_t i = 0; i < queries.size(); ++i) {
        PromptParts p = build_prompt(tmpl, retrieved[i], queries[i].question, budget);
        own[i] = Tokenizer::tokenize(p.prefix_text);
        qtok[i] = Tokenizer::encode_bytes(p.question_text);
        if (answer_lookup) atok[i] = Tokenizer::encode_bytes(queries[i].gold_answer);
    }
    out["question_tokens"] = qtok;
    out["answer_tokens"] = atok;

    auto t0 = Clock::now();
    std::vector<EmbeddingVec> emb(queries.size());
    for (size_t i = 0; i < queries.size(); ++i) emb[i] = gnn.encode(enc, retrieved[i]);
    out["encode_ms"] = ms_since(t0);
    out["embeddings"] = emb;

    t0 = Clock::now();
    ClusterAssignment a = agglomerate(emb, {lk, c});
    out["cluster_ms"] = ms_since(t0);
    out["labels"] = a.labels;

    t0 = Clock::now();
    uint32_t nc = *std::max_element(a.labels.begin(), a.labels.end()) + 1;
    std::vector<ClusterJob> jobs(nc);
    for (uint32_t ci = 0; ci < nc; ++ci) jobs[ci].cluster_id = ci;
    for (size_t i = 0; i < queries.size(); ++i) {
        ClusterMember m;
        m.query_index = i;
        m.query_id = queries[i].id;
        m.question_tokens = qtok[i];
        m.answer_tokens = atok[i];
        m.standalone_prefix_tokens = own[i];
        if (soft_on) m.standalone_soft = emb[i];
        jobs[a.labels[i]].members.push_back(std::move(m));
    }
    json reps = json::array(), ptoks = json::array(), softs = json::array();
    for (uint32_t ci = 0; ci < nc; ++ci) {
        std::vector<Subgraph> parts;
        for (const ClusterMember& m : jobs[ci].members) parts.push_back(retrieved[m.query_index]);
        jobs[ci].representative = merge_subgraphs(parts);
        jobs[ci].prefix_tokens =
            Tokenizer::tokenize(build_prompt(tmpl, jobs[ci].representative, "", budget).prefix_text);
        if (soft_on) {
            jobs[ci].soft_prefix = gnn.encode(enc, jobs[ci].representative);
            softs.push_back(*jobs[ci].soft_prefix);
        }
        reps.push_back(subgraph_json(jobs[ci].representative));
        ptoks.push_back(jobs[ci].prefix_tokens);
    }
    out["merge_ms"] = ms_since(t0);
    out["representatives"] = reps;
    out["prefix_tokens"] = ptoks;
    if (soft_on) out["soft"] = softs;

    // per-query last logits after extend on the sealed representative prefix
    if (spec.value("logits", true)) {
        json logits = json::array(), first = json::array(), first_plain = json::array();
        std::vector<json> per_q(queries.size()), per_f(queries.size()), per_p(queries.size());
        for (uint32_t ci = 0; ci < nc; ++ci) {
            KVCache shared = jobs[ci].soft_prefix
                                 ? lm.prefill(jobs[ci].prefix_tokens, *jobs[ci].soft_prefix)
                                 : lm.prefill(jobs[ci].prefix_tokens);
            shared.seal();
            for (const ClusterMember& m : jobs[ci].members) {
                if (shared.token_count() + m.question_tokens.size() + lc.max_new_tokens >
                    lc.max_seq_len) {
                    per_q[m.query_index] = nullptr;  // reference would fall back
                    continue;
                }
                KVCache f = shared.fork();
                const std::vector<float>& lg = lm.extend(f, m.question_tokens);
                per_q[m.query_index] = lg;
                DecodeOptions o;
                if (!m.answer_tokens.empty())
                    o.hint = CopyPointerHint{m.answer_tokens, f.prefix_token_count(), 100.0f};
                per_f[m.query_index] = lm.greedy_decode(f, 1, o).token_ids.at(0);
                per_p[m.query_index] = greedy_argmax(lg);
            }
        }
        out["logits"] = per_q;
        out["first_token"] = per_f;
        out["first_token_plain"] = per_p;
    }
    // the reference's own lifecycle, timed (TTFT = first-token timestamps)
    if (spec.value("run_batch", false)) {
        EngineOptions eo;
        eo.max_new_tokens = spec.value("engine_max_new", 1u);
        eo.parallel_queries = spec.value("parallel_queries", false);
        auto tb = Clock::now();
        eo.batch_start = tb;
        BatchRunResult res = run_batch(jobs, lm, eo);
        out["run_batch_ms"] = ms_since(tb);
        json ttft = json::array(), ft = json::array(), gen = json::array(), rt = json::array();
        for (const QueryOutcome& o : res.outcomes) {
            ttft.push_back(o.ttft_ms);
            rt.push_back(o.rt_ms);
            ft.push_back(o.gen.token_ids.empty() ? -1 : o.gen.token_ids[0]);
            gen.push_back(o.gen.token_ids);
        }
        out["ttft_ms"] = ttft;
        out["run_batch_first_token"] = ft;
        if (eo.max_new_tokens > 1) {
            out["run_batch_tokens"] = gen;
            out["rt_ms"] = rt;
        }
    }
    return out;
}

// Bounded timing samples of each stage at a model shape (bench.py --impl reference).
// retrieve() (retrieval.cpp:226-239) for a list of questions on a CSV graph
json cmd_retrieve(const json& spec) {
    TextualGraph g = graph_of(spec);
    TextEncoderConfig tc;
    tc.dim = spec.at("dim");
    TextEncoder enc(tc);
    RetrievalConfig rc;
    rc.strategy = retrieval_strategy_from_string(spec.value("strategy", std::string("ego-topk")));
    rc.k = spec.value("k", rc.k);
    rc.edge_cost = spec.value("edge_cost", rc.edge_cost);
    rc.ego_hops = spec.value("ego_hops", rc.ego_hops);
    rc.ego_entity_cap = spec.value("ego_entity_cap", rc.ego_entity_cap);
    json out = json::array();
    uint64_t qid = 0;
    for (const json& q : spec.at("questions")) {
        QueryRecord rec;
        rec.id = qid++;
        rec.question = q.get<std::string>();
        Subgraph s = retrieve(rc, g, rec, enc);
        out.push_back(subgraph_json(s));
    }
    return out;
}

// the reference's whole run() (pipeline.cpp:114-320) -> its subgcache-report-v1 document
json cmd_run(const json& spec) {
    RunConfig rc;
    rc.graph_nodes_path = spec.at("nodes_csv");
    rc.graph_edges_path = spec.at("edges_csv");
    rc.queries_path = spec.at("queries_jsonl");
    rc.undirected = spec.value("undirected", false);
    rc.retrieval.strategy = retrieval_strategy_from_string(spec.value("retrieval", std::string("ego-topk")));
    rc.cluster.linkage = linkage_from_string(spec.value("linkage", std::string("ward")));
    rc.cluster.cluster_count = spec.value("clusters", 4u);
    rc.seed = spec.value("seed", 7ull);
    if (spec.contains("lm")) rc.lm = lm_cfg(spec["lm"]);
    const std::string soft = spec.value("soft_prefix", std::string("auto"));
    rc.soft_prefix = soft == "on" ? SoftPrefixMode::On : (soft == "off" ? SoftPrefixMode::Off : SoftPrefixMode::Auto);
    rc.parallel_queries = spec.value("parallel_queries", false);       // --parallel-queries
    if (spec.value("mode", std::string("subgcache")) == "baseline") rc.mode = RunMode::Baseline;
    auto t0 = Clock::now();
    BatchReport r = run(rc);
    json out = json::parse(r.to_json());
    out["wall_ms"] = ms_since(t0);  // the whole run(): load, retrieve, encode, cluster, serve
    return out;
}

json cmd_bench(const json& spec) {
    json out;
    ToyLmConfig lc = lm_cfg(spec.at("lm"));
    auto t0 = Clock::now();
    ToyLm lm(lc);
    out["weight_gen_ms"] = ms_since(t0);
    SplitMix64 rng(spec.value("seed", 99ull));
    auto rand_toks = [&](size_t n) {
        std::vector<TokenId> t(n);
        for (auto& v : t) v = static_cast<TokenId>(rng.next() % 256);
        return t;
    };
    uint32_t pn = spec.value("prefill_tokens", 4u), en = spec.value("extend_tokens", 2u);
    uint32_t ctx = spec.value("extend_context", 0u);
    // prefill: pn tokens from empty
    t0 = Clock::now();
    KVCache kv = lm.prefill(rand_toks(pn));
    out["prefill_ms_per_token"] = ms_since(t0) / pn;
    // extend: en tokens on a context-token prefix. The context KV is produced with a
    // short prefill so the sample stays bounded: attention cost at ctx is added
    // analytically by bench.py from the measured per-key attention cost.
    if (en > 0) {
        KVCache base = lm.prefill(rand_toks(std::max<uint32_t>(1, std::min(ctx, 8u))));
        base.seal();
        KVCache f = base.fork();
        t0 = Clock::now();
        lm.extend(f, rand_toks(en));
        out["extend_ms_per_token"] = ms_since(t0) / en;
    }
    // --parallel-queries analogue (cache_engine.cpp:195-201): T members extend concurrently
    // on forks of one sealed prefix, one std::async task each
    uint32_t threads = spec.value("threads", 1u);
    if (threads > 1 && en > 0) {
        KVCache base = lm.prefill(rand_toks(4));
        base.seal();
        std::vector<std::vector<TokenId>> qs;
        for (uint32_t t = 0; t < threads; ++t) qs.push_back(rand_toks(en));
        t0 = Clock::now();
        std::vector<std::future<void>> futs;
        for (uint32_t t = 0; t < threads; ++t)
            futs.push_back(std::async(std::launch::async, [&, t] {
                KVCache f = base.fork();
                lm.extend(f, qs[t]);
            }));
        for (auto& f : futs) f.get();
        out["parallel_extend_ms_per_token"] = ms_since(t0) / (static_cast<double>(en) * threads);
        out["parallel_threads"] = threads;
    }
    if (spec.contains("gnn_nodes")) {
        uint32_t n = spec["gnn_nodes"], e = spec.value("gnn_edges", n - 1);
        TextualGraph g;
        for (NodeId i = 0; i < n; ++i) g.nodes[i] = "name: entity " + std::to_string(i) + "; attribute: alpha beta";
        for (uint32_t i = 0; i < e; ++i) g.edges.push_back({i % n, "related to", (i + 1) % n});
        TextEncoderConfig tc;
        tc.dim = lc.model_dim;
        TextEncoder enc(tc);
        GnnEncoderConfig gc;
        gc.dim = lc.model_dim;
        GnnEncoder gnn(gc);
        t0 = Clock::now();
        gnn.encode(enc, full_subgraph(g));
        out["gnn_encode_ms"] = ms_since(t0);
    }
    // attention cost per context key, measured at a small width with the real head_dim and the
    // real prefix length (the full-width per-token cost above covers the matvecs): extend of n
    // tokens on a P-token prefix minus the same on an 8-token prefix, per key and token
    if (spec.contains("attn_calib")) {
        const json& a = spec["attn_calib"];
        ToyLmConfig sc;
        sc.layers = 1;
        sc.heads = a.value("heads", 2u);
        sc.model_dim = a.value("d", 256u);
        sc.ffn_hidden = a.value("ffn", 4 * sc.model_dim);
        const uint32_t P = a.at("P"), n = a.value("n", 8u);
        sc.max_seq_len = P + n + 8;
        ToyLm small(sc);
        KVCache longp = small.prefill(rand_toks(P));
        longp.seal();
        KVCache shortp = small.prefill(rand_toks(8));
        shortp.seal();
        std::vector<TokenId> q = rand_toks(n);
        double best_long = 1e30, best_short = 1e30;
        for (int rep = 0; rep < 3; ++rep) {
            KVCache f1 = longp.fork();
            t0 = Clock::now();
            small.extend(f1, q);
            best_long = std::min(best_long, ms_since(t0));
            KVCache f2 = shortp.fork();
            t0 = Clock::now();
            small.extend(f2, q);
            best_short = std::min(best_short, ms_since(t0));
        }
        out["attn_ms_per_key_token"] = std::max(0.0, best_long - best_short) / (static_cast<double>(n) * (P - 8));
        out["attn_calib_d"] = sc.model_dim;
    }
    // GNN encode of real subgraphs of the workload's graph (CSV) at the model width
    if (spec.contains("gnn_subgraphs")) {
        TextualGraph g = graph_of(spec);
        TextEncoderConfig tc;
        tc.dim = lc.model_dim;
        TextEncoder enc(tc);
        GnnEncoderConfig gc;
        gc.dim = lc.model_dim;
        gc.seed = spec.value("gnn_seed", gc.seed);
        GnnEncoder gnn(gc);
        double ms = 0;
        uint64_t nodes = 0;
        for (const json& sj : spec["gnn_subgraphs"]) {
            Subgraph sub = subgraph_of(g, sj);
            nodes += sub.node_ids.size();
            t0 = Clock::now();
            gnn.encode(enc, sub);
            ms += ms_since(t0);
        }
        out["gnn_sample_ms"] = ms;
        out["gnn_sample_nodes"] = nodes;
    }
    if (spec.contains("agglomerate_m")) {
        uint32_t m = spec["agglomerate_m"], d = spec.value("agglomerate_d", lc.model_dim);
        std::vector<EmbeddingVec> pts(m, EmbeddingVec(d));
        for (auto& p : pts)
            for (float& v : p) v = rng.uniform(-1.0f, 1.0f);
        t0 = Clock::now();
        agglomerate(pts, {Linkage::Ward, spec.value("agglomerate_c", 16u)});
        out["agglomerate_ms"] = ms_since(t0);
    }
    out["threads"] = 1;
    out["hw_threads"] = std::thread::hardware_concurrency();
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 3) {
        std::fprintf(stderr, "usage: ref_driver <spec.json> <out.json>\n");
        return 2;
    }
    std::ifstream in(argv[1]);
    json spec = json::parse(in);
    std::string cmd = spec.at("cmd");
    json out;
    try {
        if (cmd == "lm") out = cmd_lm(spec);
        else if (cmd == "lm_cluster") out = cmd_lm_cluster(spec);
        else if (cmd == "cluster") out = cmd_cluster(spec);
        else if (cmd == "gnn") out = cmd_gnn(spec);
        else if (cmd == "prompt") out = cmd_prompt(spec);
        else if (cmd == "pipeline") out = cmd_pipeline(spec);
        else if (cmd == "bench") out = cmd_bench(spec);
        else if (cmd == "run") out = cmd_run(spec);
        else if (cmd == "retrieve") out = cmd_retrieve(spec);
        else if (cmd == "synth") {  // the reference's own synthetic dataset writer
            auto ds = testsupport::write_synth_dataset(spec.at("dir"), spec.at("m").get<size_t>());
            out = json{{"nodes", ds.nodes_path}, {"edges", ds.edges_path}, {"queries", ds.queries_path}};
        }
        else {
            std::fprintf(stderr, "unknown cmd %s\n", cmd.c_str());
            return 2;
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ref_driver: %s\n", e.what());
        return 1;
    }
    std::ofstream o(argv[2]);
    o << out.dump();
    return 0;
}
