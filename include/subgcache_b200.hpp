// subgcache_b200.hpp -- header-only C++ facade over the C ABI (sgc_b200.h) with the reference's
// hot-path API shapes and exception types (paths relative to /root/reference/proj):
//
//   subgcache::Error/DomainError/CapacityError/...   include/subgcache/errors.hpp:9-32
//   ToyLmConfig, ToyLm::prefill / extend              include/subgcache/lm_core.hpp:16-27,128-147
//   agglomerate -> ClusterAssignment/MergeStep        include/subgcache/clustering.hpp:21-44
//   pairwise_distances                                include/subgcache/clustering.hpp:35
//   GnnEncoder::encode (batched)                      include/subgcache/encoders.hpp:61
//   merge_subgraphs + build_prompt + tokenize         graph_store.hpp:77, cache_engine.hpp:45
//
// Value semantics and exceptions as in the reference; every call runs sm_100a kernels.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgc_b200.h"

namespace subgcache_b200 {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DomainError : Error {
    using Error::Error;
};
struct CapacityError : Error {
    using Error::Error;
};
struct IntegrityError : Error {
    using Error::Error;
};
struct ParseError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

inline void check(int st) {
    if (st == SGC_OK) return;
    std::string msg = sgc_last_error();
    switch (st) {
        case SGC_DOMAIN: throw DomainError(msg);
        case SGC_CAPACITY: throw CapacityError(msg);
        case SGC_INTEGRITY: throw IntegrityError(msg);
        case SGC_PARSE: throw ParseError(msg);
        case SGC_LOGIC: throw std::logic_error(msg);
        default: throw CudaError(msg);
    }
}

using TokenId = int32_t;
using EmbeddingVec = std::vector<float>;

class Context {
public:
    explicit Context(int device = 0) {
        sgc_ctx* c = nullptr;
        check(sgc_ctx_create(device, &c));
        h_.reset(c);
    }
    sgc_ctx* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(sgc_ctx* c) const { sgc_ctx_destroy(c); }
    };
    std::unique_ptr<sgc_ctx, Del> h_;
};

// lm_core.hpp:16-27
struct ToyLmConfig {
    uint32_t layers = 4, heads = 4, model_dim = 64, ffn_hidden = 256, max_seq_len = 1024,
             max_new_tokens = 32;
    uint64_t seed = 3;
};

// Sealed prefix segments (KVCache after seal(), lm_core.cpp:60-80) living in HBM.
class SealedPrefixes {
public:
    explicit SealedPrefixes(sgc_kv* kv) : h_(kv) {}
    uint32_t count() const { return sgc_kv_count(h_.get()); }
    size_t token_count(uint32_t i) const { return sgc_kv_tokens(h_.get(), i); }
    uint64_t prefix_digest(uint32_t i) const { return sgc_kv_digest(h_.get(), i); }
    size_t resident_kv_bytes() const { return sgc_kv_resident_bytes(h_.get()); }
    sgc_kv* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(sgc_kv* k) const { sgc_kv_release(k); }
    };
    std::unique_ptr<sgc_kv, Del> h_;
};

inline sgc_token_lists pack(const std::vector<std::vector<TokenId>>& lists, std::vector<uint64_t>& off,
                            std::vector<TokenId>& flat) {
    off.assign(1, 0);
    flat.clear();
    for (const auto& l : lists) {
        flat.insert(flat.end(), l.begin(), l.end());
        off.push_back(flat.size());
    }
    if (flat.empty()) flat.push_back(0);
    return sgc_token_lists{static_cast<uint32_t>(lists.size()), off.data(), flat.data()};
}

class ToyLm {
public:
    ToyLm(Context& ctx, const ToyLmConfig& cfg) : ctx_(ctx), cfg_(cfg) {
        sgc_lm_config c{cfg.layers, cfg.heads, cfg.model_dim, cfg.ffn_hidden, cfg.max_seq_len,
                        cfg.max_new_tokens, cfg.seed};
        sgc_model* m = nullptr;
        check(sgc_model_create(ctx.get(), &c, &m));
        h_.reset(m);
    }
    const ToyLmConfig& config() const { return cfg_; }

    // ToyLm::prefill + KVCache::seal for many prompts at once; last_logits [n][260]
    SealedPrefixes prefill(const std::vector<std::vector<TokenId>>& prompts,
                           std::vector<std::vector<float>>* last_logits = nullptr) const {
        std::vector<uint64_t> off;
        std::vector<TokenId> flat;
        sgc_token_lists tl = pack(prompts, off, flat);
        std::vector<float> lg(prompts.size() * SGC_VOCAB);
        sgc_kv* kv = nullptr;
        check(sgc_prefill(ctx_.get(), h_.get(), &tl, nullptr, nullptr, &kv, lg.data()));
        if (last_logits) {
            last_logits->assign(prompts.size(), std::vector<float>(SGC_VOCAB));
            for (size_t i = 0; i < prompts.size(); ++i)
                std::copy(lg.begin() + i * SGC_VOCAB, lg.begin() + (i + 1) * SGC_VOCAB, (*last_logits)[i].begin());
        }
        return SealedPrefixes(kv);
    }

    // KVCache::fork + ToyLm::extend (+ first greedy token with the copy pointer) per member
    std::vector<std::vector<float>> extend(const SealedPrefixes& kv, const std::vector<uint32_t>& segment,
                                           const std::vector<std::vector<TokenId>>& questions,
                                           std::vector<TokenId>* first_token = nullptr,
                                           const std::vector<std::vector<TokenId>>* answers = nullptr,
                                           float bonus = 100.0f) const {
        std::vector<uint64_t> qo, ao;
        std::vector<TokenId> qf, af;
        sgc_token_lists ql = pack(questions, qo, qf);
        sgc_token_lists al{};
        if (answers) al = pack(*answers, ao, af);
        std::vector<float> lg(questions.size() * SGC_VOCAB);
        std::vector<TokenId> ft(questions.size());
        check(sgc_extend(ctx_.get(), h_.get(), kv.get(), segment.data(), &ql, answers ? &al : nullptr, bonus,
                         lg.data(), ft.data()));
        if (first_token) *first_token = ft;
        std::vector<std::vector<float>> out(questions.size(), std::vector<float>(SGC_VOCAB));
        for (size_t i = 0; i < questions.size(); ++i)
            std::copy(lg.begin() + i * SGC_VOCAB, lg.begin() + (i + 1) * SGC_VOCAB, out[i].begin());
        return out;
    }
    // KVCache::fork + ToyLm::extend + ToyLm::greedy_decode (lm_core.cpp:352-404) per member,
    // all members batched; returns GenerationResult::token_ids per member
    std::vector<std::vector<TokenId>> generate(const SealedPrefixes& kv, const std::vector<uint32_t>& segment,
                                               const std::vector<std::vector<TokenId>>& questions,
                                               const std::vector<std::vector<TokenId>>* answers = nullptr,
                                               uint32_t max_new = 0, float bonus = 100.0f) const {
        const uint32_t mx = max_new ? max_new : cfg_.max_new_tokens;
        std::vector<uint64_t> qo, ao;
        std::vector<TokenId> qf, af;
        sgc_token_lists ql = pack(questions, qo, qf);
        sgc_token_lists al{};
        if (answers) al = pack(*answers, ao, af);
        std::vector<TokenId> toks(questions.size() * mx, -1);
        std::vector<uint32_t> cnt(questions.size());
        check(sgc_extend_generate(ctx_.get(), h_.get(), kv.get(), segment.data(), &ql, answers ? &al : nullptr,
                                  bonus, mx, nullptr, nullptr, toks.data(), cnt.data()));
        std::vector<std::vector<TokenId>> out(questions.size());
        for (size_t i = 0; i < questions.size(); ++i)
            out[i].assign(toks.begin() + i * mx, toks.begin() + i * mx + cnt[i]);
        return out;
    }
    sgc_model* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(sgc_model* m) const { sgc_model_destroy(m); }
    };
    Context& ctx_;
    ToyLmConfig cfg_;
    std::unique_ptr<sgc_model, Del> h_;
};

// clustering.hpp:11-32
enum class Linkage { Ward = SGC_WARD, Single = SGC_SINGLE, Average = SGC_AVERAGE, Complete = SGC_COMPLETE,
                     Centroid = SGC_CENTROID };
struct ClusterConfig {
    Linkage linkage = Linkage::Ward;
    uint32_t cluster_count = 1;
};
struct MergeStep {
    uint32_t left_min = 0, right_min = 0;  // min member of left / right (members are recoverable)
    double distance = 0.0;
};
struct ClusterAssignment {
    std::vector<uint32_t> labels;
    std::vector<MergeStep> merges;
    uint64_t op_count = 0;
};

inline std::vector<double> pairwise_distances(Context& ctx, const std::vector<EmbeddingVec>& embs) {
    if (embs.empty()) throw DomainError("pairwise_distances: need at least one embedding");
    const uint32_t m = static_cast<uint32_t>(embs.size()), d = static_cast<uint32_t>(embs[0].size());
    std::vector<float> flat;
    for (const auto& e : embs) {
        if (e.size() != d) throw DomainError("embedding dim mismatch");
        flat.insert(flat.end(), e.begin(), e.end());
    }
    std::vector<double> out(static_cast<size_t>(m) * m);
    check(sgc_pairwise_distances(ctx.get(), flat.data(), m, d, out.data()));
    return out;
}

inline ClusterAssignment agglomerate(Context& ctx, const std::vector<EmbeddingVec>& embs,
                                     const ClusterConfig& cfg) {
    const uint32_t m = static_cast<uint32_t>(embs.size());
    if (cfg.cluster_count < 1) throw DomainError("cluster count must be >= 1");
    if (cfg.cluster_count > m) throw DomainError("cluster count exceeds point count");
    const uint32_t d = static_cast<uint32_t>(embs[0].size());
    std::vector<float> flat;
    for (const auto& e : embs) {
        if (e.size() != d) throw DomainError("embedding dim mismatch");
        flat.insert(flat.end(), e.begin(), e.end());
    }
    ClusterAssignment a;
    a.labels.resize(m);
    const uint32_t k = m - cfg.cluster_count;
    std::vector<uint32_t> l(k + 1), r(k + 1);
    std::vector<double> dist(k + 1);
    check(sgc_agglomerate(ctx.get(), flat.data(), m, d, static_cast<int>(cfg.linkage), cfg.cluster_count,
                          a.labels.data(), l.data(), r.data(), dist.data(), &a.op_count));
    for (uint32_t i = 0; i < k; ++i) a.merges.push_back({l[i], r[i], dist[i]});
    return a;
}

}  // namespace subgcache_b200
