/*
 * sgc_oracle.h -- CPU restatement of the SubGCache hot path (TEST INFRASTRUCTURE).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. It restates, in plain C, the
 * reference algorithm each function cites (paths relative to
 * /root/reference/proj). Parity of this restatement is pinned against the
 * compiled reference (oracle/_ref/ref_driver) by tests/test_oracle_pin.py and
 * the committed fixtures under tests/golden/.
 *
 * Floating point follows the reference exactly where the reference is exact
 * (fp64 encoders / clustering: every mul and add rounded separately, no FMA,
 * sequential reduction order) and the reference's *scalar* kernel backend for
 * the fp32 LM (kernels_scalar.cpp), which differs from the AVX2 backend only in
 * dot-product reduction order (<=2e-4 logits per test_lm_core.cpp:241-262).
 */
#ifndef SGC_ORACLE_H
#define SGC_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng (rng.hpp:12-57) ---- */
uint64_t sgo_splitmix64_once(uint64_t x);
uint64_t sgo_fnv1a64(const void* data, size_t n, uint64_t h);
/* rng.hpp:25-28 uniform(lo,hi) over a stream seeded with `state0` (already mixed) */
void sgo_fill_uniform_state(float* w, size_t n, uint64_t state0, float lo, float hi);
/* lm_core.cpp:19-23 fill_uniform(w, seed, fan_in) */
void sgo_fill_uniform(float* w, size_t n, uint64_t seed, size_t fan_in);

/* ---- text encoder (encoders.cpp:50-93) ---- */
#define SGO_BUCKETS 4096u
void sgo_text_projection(float* proj /*[dim*4096]*/, uint32_t dim, uint64_t seed);
/* Token hashing: writes up to cap (bucket, sign) pairs, returns token count. */
size_t sgo_text_hash(const char* text, size_t len, uint64_t salt, uint32_t* buckets,
                     int8_t* signs, size_t cap);
void sgo_text_embed(const float* proj, uint32_t dim, uint64_t salt, const char* text, size_t len,
                    float* out /*[dim]*/);

/* ---- GNN encoder (encoders.cpp:95-186) ---- */
void sgo_gnn_weights(float* w /*[L*H*d*d]*/, uint32_t layers, uint32_t heads, uint32_t dim,
                     uint64_t seed);
/* node_feat [n*d] float (text features, nodes ascending by id); msgs in
 * ascending edge-index order with local src/dst and gate [e*d] float. */
int sgo_gnn_encode(const float* w, uint32_t layers, uint32_t heads, uint32_t dim,
                   const float* node_feat, uint32_t n, const uint32_t* msg_src,
                   const uint32_t* msg_dst, const float* msg_gate, uint32_t e, float* out);

/* ---- clustering (clustering.cpp:33-174; tests/support/cluster_oracle.hpp) ---- */
enum { SGO_WARD = 0, SGO_SINGLE = 1, SGO_AVERAGE = 2, SGO_COMPLETE = 3, SGO_CENTROID = 4 };
void sgo_pairwise(const float* emb, uint32_t m, uint32_t d, double* out /*[m*m]*/);
/* merges: keep slot (== min member of left), kill slot (== min member of right), distance */
int sgo_agglomerate(const float* emb, uint32_t m, uint32_t d, int linkage, uint32_t c,
                    uint32_t* labels, uint32_t* merge_left_min, uint32_t* merge_right_min,
                    double* merge_dist, uint64_t* op_count);
int sgo_naive_agglomerate(const float* emb, uint32_t m, uint32_t d, int linkage, uint32_t c,
                          uint32_t* labels, double* merge_dist);

/* ---- representative construction (graph_store.cpp:223-262, cache_engine.cpp:29-71) ---- */
/* Union of member element lists (ids < universe) -> ascending unique list; returns count. */
uint32_t sgo_union(const uint32_t* const* lists, const uint32_t* lens, uint32_t n_lists,
                   uint32_t universe, uint32_t* out);
/* csv_quote(field) appended to dst; returns bytes written (dst may be NULL to size). */
size_t sgo_csv_quote(const char* field, size_t len, char* dst);
/* Build the prefix tokens (BOS + bytes) from pre-rendered rows of the selected
 * nodes/edges (already in ascending order).  Returns token count or -1 when the
 * headers alone exceed the budget (CapacityError).  budget_tokens = PromptBudget::prefix_budget(). */
long sgo_build_prefix(const char* const* node_rows, const uint32_t* node_len, uint32_t n_nodes,
                      const char* const* edge_rows, const uint32_t* edge_len, uint32_t n_edges,
                      uint32_t budget_tokens, int32_t* tokens, uint32_t* dropped_nodes,
                      uint32_t* dropped_edges);
/* question wrapper (cache_engine.cpp:34-41) -> byte tokens, returns count or -1 */
long sgo_question_tokens(const char* q, size_t len, uint32_t question_budget, int32_t* tokens);

/* ---- ToyLm (lm_core.cpp:122-406), scalar kernel order ---- */
typedef struct sgo_lm sgo_lm;
typedef struct sgo_kv sgo_kv;
sgo_lm* sgo_lm_create(uint32_t layers, uint32_t heads, uint32_t dim, uint32_t ffn,
                      uint32_t max_seq, uint64_t seed);
void sgo_lm_destroy(sgo_lm* lm);
/* raw weight access for the GPU parity tests (fp32, reference layout) */
const float* sgo_lm_weight(const sgo_lm* lm, int which, uint32_t layer, size_t* n);
sgo_kv* sgo_kv_create(const sgo_lm* lm);
sgo_kv* sgo_kv_fork(const sgo_kv* kv); /* deep copy (the oracle has no sharing) */
void sgo_kv_destroy(sgo_kv* kv);
uint32_t sgo_kv_tokens(const sgo_kv* kv);
/* K or V of layer l as [tokens*dim] float */
const float* sgo_kv_data(const sgo_kv* kv, int is_v, uint32_t layer);
/* prefill/extend: forward `n` tokens; soft (dim floats) replaces position 0's
 * embedding and token 259 is prepended (prefill only). logits: last position
 * [260]; all_logits (optional) [n*260]. Returns 0, or 2 on CapacityError,
 * 1 on DomainError. */
int sgo_lm_prefill(const sgo_lm* lm, sgo_kv* kv, const int32_t* tokens, uint32_t n,
                   const float* soft, float* logits, float* all_logits);
int sgo_lm_extend(const sgo_lm* lm, sgo_kv* kv, const int32_t* tokens, uint32_t n, float* logits,
                  float* all_logits);
/* lm_core.cpp:39-50 */
int32_t sgo_greedy_argmax(const float* logits, uint32_t n, int32_t bias_target, float bonus);
/* lm_core.cpp:360-374: does `answer` occur in ctx[0:limit)? */
int sgo_hint_found(const int32_t* ctx, uint32_t ctx_len, uint32_t limit, const int32_t* answer,
                   uint32_t ans_len);

#ifdef __cplusplus
}
#endif
#endif
