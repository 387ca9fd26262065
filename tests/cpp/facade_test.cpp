// Exercises the header-only C++ facade (include/subgcache_b200.hpp) on the GPU the way the
// reference's doctest suites exercise its API (test_lm_core.cpp, test_clustering.cpp).
#include <cmath>
#include <cstdio>

#include "subgcache_b200.hpp"

using namespace subgcache_b200;

#define CHECK(x)                                                         \
    do {                                                                 \
        if (!(x)) {                                                      \
            std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #x); \
            return 1;                                                    \
        }                                                                \
    } while (0)

int main() {
    Context ctx(0);
    ToyLmConfig cfg;
    cfg.max_seq_len = 128;
    ToyLm lm(ctx, cfg);
    // prefill(A ++ B) == prefill(A) + extend(B) (test_lm_core.cpp:58-75)
    std::vector<TokenId> a = {256, 1, 2, 3, 4, 5, 6, 7}, b = {8, 9, 10};
    std::vector<TokenId> ab = a;
    ab.insert(ab.end(), b.begin(), b.end());
    std::vector<std::vector<float>> full_lg;
    SealedPrefixes full = lm.prefill({ab}, &full_lg);
    SealedPrefixes pa = lm.prefill({a});
    auto ext = lm.extend(pa, {0}, {b});
    float gap = 0;
    for (int v = 0; v < SGC_VOCAB; ++v) gap = std::fmax(gap, std::fabs(ext[0][v] - full_lg[0][v]));
    CHECK(gap < 0.05f);
    CHECK(full.token_count(0) == ab.size());
    // capacity error (test_lm_core.cpp:86-95)
    bool threw = false;
    try {
        lm.prefill({std::vector<TokenId>(129, 1)});
    } catch (const CapacityError&) {
        threw = true;
    }
    CHECK(threw);
    // exact ties resolve by smallest member indices (test_clustering.cpp:106-118)
    std::vector<EmbeddingVec> pts(4, EmbeddingVec{1.0f, 2.0f});
    ClusterAssignment asg = agglomerate(ctx, pts, {Linkage::Ward, 2});
    CHECK(asg.merges.size() == 2);
    CHECK(asg.merges[0].left_min == 0 && asg.merges[0].right_min == 1);
    CHECK(asg.merges[1].left_min == 0 && asg.merges[1].right_min == 2);
    CHECK((asg.labels == std::vector<uint32_t>{0, 0, 0, 1}));
    threw = false;
    try {
        agglomerate(ctx, pts, {Linkage::Ward, 5});
    } catch (const DomainError&) {
        threw = true;
    }
    CHECK(threw);
    // greedy decode with the copy pointer: answer then EOS (lm_core.cpp:376-387)
    std::vector<TokenId> prompt = {256, 'c', 'o', 'l', 'o', 'r', ':', ' ', 'b', 'l', 'u', 'e', '.'};
    SealedPrefixes pp = lm.prefill({prompt});
    std::vector<std::vector<TokenId>> ans = {{'b', 'l', 'u', 'e'}};
    auto gen = lm.generate(pp, {0}, {{'?', ' '}}, &ans, 8);
    CHECK((gen[0] == std::vector<TokenId>{'b', 'l', 'u', 'e', SGC_EOS}));
    auto d = pairwise_distances(ctx, {{1.f, 0.f, 0.f}, {-1.f, 0.f, 0.f}});
    CHECK(d[1] == 2.0 && d[2] == 2.0 && d[0] == 0.0);
    std::printf("facade ok (logit gap %.4f)\n", gap);
    return 0;
}
