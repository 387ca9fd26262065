// graph_kernels.cuh -- host interface of graph_kernels.cu
#pragma once
#include <stdint.h>

namespace sgc {
struct Ctx;

void text_features(Ctx* c, float* out, const uint32_t* bucket, const int8_t* sign,
                   const uint64_t* tok_off, int n_elem, const float* proj_t, int dim);
void node_index(Ctx* c, int32_t* out, const uint32_t* ids, uint64_t n, const uint32_t* sorted_ids,
                int n_nodes);

// retrieval (retrieval.cpp): cosine_similarity's three sums (encoders.cpp:28-38) in the
// reference's order -- sequential over the feature index, products rounded before the add --
// so the scores and every top-k decision taken on them are bit-identical.
// dot[i * nb + j] = sum_k a_i[k] * b_j[k]; sq_a[i] = sum_k a_i[k]^2 (sq_b likewise)
void retrieval_dots(Ctx* c, double* dot, double* sq_a, double* sq_b, const float* A, int na, const float* B,
                    int nb, int d);
// ego nets: pooled[e] = float(mean over members (nodes then edges, given order) of feat rows);
// then pair_dot[e] = sum_k q[qi[e]][k] * pooled[e][k] and pair_sq[e] = sum_k pooled[e][k]^2
void ego_pool_dots(Ctx* c, float* pooled, double* pair_dot, double* pair_sq, const float* feat,
                   const uint32_t* mem_off, const uint32_t* mem_idx, const float* q, const int32_t* qi,
                   int n_ego, int d);

struct UnionArgs {
    int clusters;
    const int32_t* sub_nodes;  // dense node indices
    const uint64_t* sub_node_off;
    const uint32_t* sub_edges;
    const uint64_t* sub_edge_off;
    const uint32_t* members;
    const uint64_t* member_off;
    uint32_t* node_bm;
    uint32_t* edge_bm;
    int node_words, edge_words;
    const uint32_t* node_row_len;
    const uint32_t* edge_row_len;
    int n_nodes, n_edges;
    uint32_t budget_bytes, base_bytes;
    uint32_t* sel_nodes;
    uint32_t* sel_edges;
    uint32_t* node_pre;
    uint32_t* edge_pre;
    uint32_t* stats;
    int* status;
};
void union_prompt(Ctx* c, const UnionArgs& a);

struct GatherArgs {
    int clusters;
    uint64_t max_tokens;
    int32_t* tokens;
    const uint64_t* tok_off;
    const uint32_t* stats;
    const uint32_t* sel_nodes;
    const uint32_t* sel_edges;
    const uint32_t* node_pre;
    const uint32_t* edge_pre;
    const char* node_text;  // rendered node rows
    const uint64_t* node_text_off;
    const char* edge_text;  // rendered edge rows
    const uint64_t* edge_text_off;
    int n_nodes, n_edges;
    int head_len, ehead_len;
    const char* head;   // host bytes: header + node csv header + '\n' (build_prompt, cache_engine.cpp:29-71)
    const char* ehead;  // host bytes: edge csv header + '\n'
};
void prompt_gather(Ctx* c, const GatherArgs& a);
}  // namespace sgc
