/*
 * sgc_b200.h -- C ABI of the B200-native SubGCache in-batch serving hot path.
 *
 * Drop-in boundary for the reference's hot-path C++ API (paths relative to
 * /root/reference/proj). Each entry point names the reference interface it
 * replaces; INTEGRATION.md shows the reference-side binding. All calls are
 * synchronous at return, stream-ordered on the context's stream, and report
 * errors through an int status plus a thread-local message (sgc_last_error),
 * mirroring the reference's exception taxonomy (include/subgcache/errors.hpp:9-32):
 *
 *   SGC_OK 0, SGC_DOMAIN 1 (DomainError), SGC_CAPACITY 2 (CapacityError),
 *   SGC_INTEGRITY 3 (IntegrityError), SGC_PARSE 4 (ParseError),
 *   SGC_LOGIC 5 (std::logic_error), SGC_CUDA 6 (device / runtime failure).
 *
 * Pointers to array data may be host or device memory (unified addressing); the
 * library copies as needed. No torch types cross this boundary.
 */
#ifndef SGC_B200_H
#define SGC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    SGC_OK = 0,
    SGC_DOMAIN = 1,
    SGC_CAPACITY = 2,
    SGC_INTEGRITY = 3,
    SGC_PARSE = 4,
    SGC_LOGIC = 5,
    SGC_CUDA = 6
};

/* clustering.hpp:11 enum class Linkage */
enum { SGC_WARD = 0, SGC_SINGLE = 1, SGC_AVERAGE = 2, SGC_COMPLETE = 3, SGC_CENTROID = 4 };

#define SGC_VOCAB 260 /* tokenizer.hpp:15-19: 256 bytes + BOS/EOS/PAD/GRAPH_SOFT_SLOT */
#define SGC_BOS 256   /* Tokenizer::kBos */
#define SGC_EOS 257   /* Tokenizer::kEos (greedy_decode stops on it, lm_core.cpp:387) */

typedef struct sgc_ctx sgc_ctx;     /* one CUDA device + stream + scratch arena */
typedef struct sgc_model sgc_model; /* ToyLm weights, bf16 in HBM (lm_core.hpp:114-171) */
typedef struct sgc_graph sgc_graph; /* TextualGraph pre-rendered rows + text features */
typedef struct sgc_kv sgc_kv;       /* sealed prefix segments (KVCache::seal, lm_core.cpp:60-80) */
typedef struct sgc_fork sgc_fork;   /* KVCache::fork of one sealed segment + private suffix */

/* lm_core.hpp:16-27 ToyLmConfig */
typedef struct {
    uint32_t layers, heads, model_dim, ffn_hidden, max_seq_len, max_new_tokens;
    uint64_t seed;
} sgc_lm_config;

/* encoders.hpp:17-21 TextEncoderConfig + :44-49 GnnEncoderConfig */
typedef struct {
    uint32_t layers, heads, dim;
    uint64_t seed;      /* GnnEncoderConfig::seed (pipeline.cpp:138: splitmix64_once(seed^0x62)) */
    uint64_t text_seed; /* TextEncoderConfig::seed, default 1 */
    uint64_t text_salt; /* TextEncoderConfig::hash_salt, default 55 */
} sgc_gnn_config;

/* A batch of subgraphs of one graph in CSR form: subgraph i owns node ids
 * nodes[node_off[i] .. node_off[i+1]) and edge indices edges[edge_off[i] .. edge_off[i+1]),
 * both ascending (std::set order, graph_store.hpp:39-49). */
typedef struct {
    uint32_t count;
    const uint64_t* node_off;
    const uint32_t* nodes;
    const uint64_t* edge_off;
    const uint32_t* edges;
} sgc_subgraphs;

/* Ragged int32 token lists: list i = tokens[off[i] .. off[i+1]). */
typedef struct {
    uint32_t count;
    const uint64_t* off;
    const int32_t* tokens;
} sgc_token_lists;

const char* sgc_last_error(void);
const char* sgc_version(void);

/* ---- context ------------------------------------------------------------------ */
int sgc_ctx_create(int device, sgc_ctx** out);
/* Release every handle created on the context (sgc_kv, then sgc_model / sgc_graph) first:
 * their destructors free device memory on the context's stream. */
int sgc_ctx_destroy(sgc_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the own stream. */
int sgc_ctx_set_stream(sgc_ctx* ctx, void* stream);
/* Number of kernel launches issued by this context since creation (bench evidence). */
uint64_t sgc_ctx_launch_count(const sgc_ctx* ctx);

/* ---- multi-GPU transport -----------------------------------------------
 * A context joins a group of `world` ranks (one process or thread per GPU); sgc_run_subgcache
 * then does the path's only exchanges itself: the all-gather of subgraph embeddings before
 * clustering, the point-to-point copy of a split cluster's sealed prefix K/V to the ranks serving
 * the rest of its members (instead of a replica prefill; the reference's fork shares the sealed
 * prefix by pointer, cache_engine.cpp:183), and the gather of per-query outputs to rank 0.
 * NCCL (NVLink / NVSwitch): rank 0 makes an id with sgc_comm_unique_id, every rank passes the same
 * 128 bytes to sgc_comm_init_nccl (libnccl.so.2 is resolved at run time). Host transport: C
 * callbacks over HOST buffers (e.g. torch.distributed gloo, or in-process ranks); both return
 * 0 on success. */
typedef struct {
    void* user;
    /* recv[world * bytes] <- every rank's send[bytes], in rank order */
    int (*allgather)(void* user, const void* send, void* recv, size_t bytes);
    /* post every send and receive of this rank together, return when all completed */
    int (*exchange)(void* user, int n_send, const void* const* send_buf, const size_t* send_bytes,
                    const int* send_peer, int n_recv, void* const* recv_buf, const size_t* recv_bytes,
                    const int* recv_peer);
} sgc_host_transport;
int sgc_comm_unique_id(uint8_t id[128]);
int sgc_comm_init_nccl(sgc_ctx* ctx, const uint8_t id[128], int world, int rank);
int sgc_comm_init_host(sgc_ctx* ctx, const sgc_host_transport* t, int world, int rank);
int sgc_comm_destroy(sgc_ctx* ctx);
/* 1 if the context has a transport with world > 1 (out: world, rank, kind 0 none / 1 nccl / 2 host) */
int sgc_comm_info(const sgc_ctx* ctx, int* world, int* rank, int* kind);

/* ---- model: ToyLm::ToyLm (lm_core.cpp:122-161) -------------------------------------
 * Weights are generated ON DEVICE from the seed, element-for-element identical to the
 * reference's fp32 SplitMix64 streams, then stored as bf16 (GEMM operands) and fp32
 * (token embedding, head). RoPE tables are computed on the host exactly as the reference. */
int sgc_model_create(sgc_ctx* ctx, const sgc_lm_config* cfg, sgc_model** out);
int sgc_model_destroy(sgc_model* model);
/* Copy one generated fp32 weight tensor to `out` (test hook): which = 0 tok_embedding,
 * 1 head, 2 wqkv, 3 wo, 4 w1, 5 w2 (fp32 values reconstructed from the bf16 copy for 2..5
 * when fp32 == 0, or the exact fp32 stream when fp32 == 1). */
int sgc_model_weight(sgc_model* model, int which, uint32_t layer, int fp32, float* out, size_t n);

/* ---- graph: TextualGraph (graph_store.hpp:28-35) -------------------------------------
 * Node ids ascending; node i's attribute text is node_text[node_off[i] .. node_off[i+1]).
 * Edge e = (edge_src[e], edge_text[..], edge_dst[e]). Rows are pre-rendered once
 * (serialize_subgraph_rows, graph_store.cpp:249-262) and the text encoder's token hashes
 * computed (encoders.cpp:62-80): host string work, done at ingest. */
int sgc_graph_upload(sgc_ctx* ctx, uint32_t n_nodes, const uint32_t* node_ids,
                     const char* node_text, const uint64_t* node_off, uint32_t n_edges,
                     const uint32_t* edge_src, const uint32_t* edge_dst, const char* edge_text,
                     const uint64_t* edge_off, sgc_graph** out);
int sgc_graph_destroy(sgc_graph* g);

/* ---- (0) retrieval: retrieve() (retrieval.hpp, retrieval.cpp:96-239) ------------------
 * The step before the hot path: each question is embedded with the
 * TextEncoder (dim, seed, salt), nodes (and for node-edge-topk edges) are scored by cosine
 * similarity on the GPU in the reference's exact fp64 order, and the selection -- top-k with
 * ties toward the smaller index, edge rule, BFS path connection (node-edge-topk) or ego nets
 * with pooled-feature re-ranking (ego-topk, pooling and scoring on the GPU) -- follows the
 * reference step for step, so retrieved node/edge sets are bit-identical.
 * Questions: text q_text[q_off[i] .. q_off[i+1]). Outputs (host or device) CSR:
 *   node_off [m+1], nodes (ascending ids), edge_off [m+1], edges (ascending indices); SGC_CAPACITY
 *   if a capacity is too small. DomainError for k < 1, ego_hops < 1, edge_cost < 0, empty graph. */
enum { SGC_RETRIEVE_NODE_EDGE_TOPK = 0, SGC_RETRIEVE_EGO_TOPK = 1 };
typedef struct {
    int strategy;             /* SGC_RETRIEVE_* (RetrievalConfig::strategy) */
    uint32_t k;               /* RetrievalConfig::k (3) */
    double edge_cost;         /* RetrievalConfig::edge_cost (0.5) */
    uint32_t ego_hops;        /* RetrievalConfig::ego_hops (2) */
    uint32_t ego_entity_cap;  /* RetrievalConfig::ego_entity_cap (10) */
    uint32_t dim;             /* TextEncoderConfig::dim */
    uint64_t text_seed;       /* TextEncoderConfig::seed (1) */
    uint64_t hash_salt;       /* TextEncoderConfig::hash_salt (55) */
} sgc_retrieval_config;
int sgc_retrieve(sgc_ctx* ctx, sgc_graph* g, const sgc_retrieval_config* cfg, uint32_t m,
                 const char* q_text, const uint64_t* q_off, uint64_t* node_off, uint32_t* nodes,
                 uint64_t node_cap, uint64_t* edge_off, uint32_t* edges, uint64_t edge_cap);

/* ---- (1) subgraph embedding: GnnEncoder::encode (encoders.hpp:61, encoders.cpp:122-186) --
 * Batched over subgraphs; out [count * dim] fp32. DomainError on an empty subgraph. */
int sgc_encode_subgraphs(sgc_ctx* ctx, sgc_graph* g, const sgc_gnn_config* cfg,
                         const sgc_subgraphs* subs, float* out);
/* TextEncoder::embed of every node then every edge text, out [(n_nodes+n_edges) * dim]. */
int sgc_text_features(sgc_ctx* ctx, sgc_graph* g, uint32_t dim, uint64_t seed, uint64_t salt,
                      float* out);

/* ---- (2) clustering (clustering.hpp:35,44; clustering.cpp:33-174) -------------------- */
int sgc_pairwise_distances(sgc_ctx* ctx, const float* emb, uint32_t m, uint32_t dim,
                           double* out /* [m*m] */);
/* labels [m]; merge_left/right [m-c] = min member of the kept / absorbed cluster
 * (MergeStep::left.front()/right.front()); merge_dist [m-c] = MergeStep::distance;
 * op_count = ClusterAssignment::op_count. Any of the outputs may be NULL. */
int sgc_agglomerate(sgc_ctx* ctx, const float* emb, uint32_t m, uint32_t dim, int linkage,
                    uint32_t c, uint32_t* labels, uint32_t* merge_left, uint32_t* merge_right,
                    double* merge_dist, uint64_t* op_count);

/* ---- (3) representative construction ------------------------------------------------
 * merge_subgraphs (graph_store.cpp:223-235) + build_prompt (cache_engine.cpp:29-71) +
 * Tokenizer::tokenize (tokenizer.cpp:5-11) for every cluster in one pass: members of
 * cluster k are the subgraphs i with labels[i] == k. Outputs (host or device):
 *   rep_nodes/rep_edges : CSR of the union (ascending) -- offsets [c+1]
 *   prefix              : BOS + prefix bytes per cluster -- offsets [c+1]
 *   dropped             : [2c] dropped node rows, dropped edge rows per cluster
 * Capacities are checked; SGC_CAPACITY if headers alone exceed the budget.
 * budget_tokens = PromptBudget::prefix_budget() (cache_engine.hpp:27-30). */
int sgc_build_representatives(sgc_ctx* ctx, sgc_graph* g, const sgc_subgraphs* subs,
                              const uint32_t* labels, uint32_t c, uint32_t budget_tokens,
                              uint64_t* rep_node_off, uint32_t* rep_nodes, uint64_t rep_node_cap,
                              uint64_t* rep_edge_off, uint32_t* rep_edges, uint64_t rep_edge_cap,
                              uint64_t* prefix_off, int32_t* prefix, uint64_t prefix_cap,
                              uint32_t* dropped);

/* ---- (4) KV precompute: ToyLm::prefill + KVCache::seal (lm_core.cpp:299-327, :60-80) --
 * Prefills `seqs.count` sequences in one batched pass (varlen causal attention) into the
 * model's paged bf16 KV pool (128-token pages, one block table per sequence) and seals them. soft (optional) [count * model_dim] with
 * soft_mask[i] != 0 selecting sequences that carry a GRAPH_SOFT_SLOT at position 0.
 * last_logits (optional) [count * 260]. CapacityError if a sequence exceeds max_seq_len. */
int sgc_prefill(sgc_ctx* ctx, sgc_model* model, const sgc_token_lists* seqs, const float* soft,
                const uint8_t* soft_mask, sgc_kv** out, float* last_logits);
int sgc_kv_release(sgc_kv* kv);
uint32_t sgc_kv_count(const sgc_kv* kv);
/* KVCache::token_count of sealed segment i */
uint64_t sgc_kv_tokens(const sgc_kv* kv, uint32_t i);
/* KVCache::prefix_digest analogue (lm_core.cpp:108-116) over the bf16 pages: FNV-1a over each
 * row's 64-bit words, those row digests folded per (layer, K|V) in row order, the folds folded in
 * layer order (K before V) -- computed on the device. The reference hashes fp32 bytes, so the
 * values are this library's own; equality before / after serving is what the path checks. */
uint64_t sgc_kv_digest(const sgc_kv* kv, uint32_t i);
/* KVCache::resident_kv_bytes analogue for the whole handle: its pages (K + V, all layers, bf16) */
uint64_t sgc_kv_resident_bytes(const sgc_kv* kv);
/* Paged KV cache: the block table of segment i (page ids of the model's pool; token t of the
 * segment is row t % 128 of page pages[t / 128]). Returns the page count; pages may be NULL. */
uint32_t sgc_kv_pages(const sgc_kv* kv, uint32_t i, int32_t* pages);
/* Copy segment i, layer l, K (is_v=0) or V as fp32 [tokens * model_dim] (test hook). */
int sgc_kv_read(const sgc_kv* kv, uint32_t i, uint32_t layer, int is_v, float* out);

/* ---- fork handles: the KVCache object model (lm_core.hpp:35-92, lm_core.cpp:82-99) --------
 * A fork shares sealed segment `seg` of `kv` (the segment stays alive while forks use it, like the
 * reference's shared_ptr prefix; sgc_kv_release only drops the handle's reference) and owns a
 * private suffix in pages of the same pool. sgc_fork_extend = ToyLm::extend (lm_core.cpp:329-339)
 * on n forks in one batched pass: fork j appends tokens[j]; logits [n * 260] (optional) are the
 * last-position logits (also kept per fork). CapacityError past max_seq_len. truncate: SGC_LOGIC
 * into the sealed prefix (std::logic_error in the reference), SGC_DOMAIN beyond the token count. */
int sgc_kv_fork(sgc_kv* kv, uint32_t seg, sgc_fork** out);
int sgc_fork_fork(const sgc_fork* f, sgc_fork** out); /* deep copy of the private suffix */
int sgc_fork_extend(sgc_ctx* ctx, sgc_model* model, sgc_fork* const* forks, uint32_t n,
                    const sgc_token_lists* tokens, float* logits);
uint64_t sgc_fork_tokens(const sgc_fork* f);        /* KVCache::token_count */
uint64_t sgc_fork_prefix_tokens(const sgc_fork* f); /* KVCache::prefix_token_count */
int sgc_fork_last_logits(const sgc_fork* f, float* out);
int sgc_fork_truncate(sgc_fork* f, uint64_t tokens);  /* KVCache::truncate_to */
int sgc_fork_release_suffix(sgc_fork* f);             /* KVCache::release_suffix */
int sgc_fork_destroy(sgc_fork* f);

/* ---- (5) per-query reuse: KVCache::fork + ToyLm::extend + first greedy token ----------
 * (lm_core.cpp:82-90, :329-339, :352-390; cache_engine.cpp:183-189)
 * Member j forks sealed segment member_seg[j] and extends it with its question tokens;
 * all members of all segments run in ONE batched pass (cascade attention: shared prefix
 * KV read once per query tile for every member of the segment). Private suffixes are
 * released at return (KVCache::release_suffix). Outputs (optional):
 *   logits      [count * 260]  last-position logits after the extend
 *   first_token [count]        greedy_argmax with the copy-pointer bias: answer j (may be
 *                              empty) searched in the segment's prefix tokens
 *                              (CopyPointerHint::search_limit = prefix length).
 * CapacityError if prefix + question exceeds max_seq_len. */
int sgc_extend(sgc_ctx* ctx, sgc_model* model, sgc_kv* kv, const uint32_t* member_seg,
               const sgc_token_lists* questions, const sgc_token_lists* answers,
               float pointer_bonus, float* logits, int32_t* first_token);

/* ---- (5') per-query reuse with generation: sgc_extend followed by ToyLm::greedy_decode on
 * every fork (lm_core.cpp:352-404), batched: one decode row per still-generating member per
 * step (cascade attention: the segment's prefix on the tensor cores, the member's own question
 * and generated keys per row, merged by log-sum-exp). tokens [count * max_new] (-1 padded),
 * n_tokens [count]; logits / first_token as sgc_extend. The copy pointer biases answer[t]
 * (then EOS) when the answer occurs in the segment's prefix. */
int sgc_extend_generate(sgc_ctx* ctx, sgc_model* model, sgc_kv* kv, const uint32_t* member_seg,
                        const sgc_token_lists* questions, const sgc_token_lists* answers,
                        float pointer_bonus, uint32_t max_new, float* logits, int32_t* first_token,
                        int32_t* tokens, uint32_t* n_tokens);

/* ---- the whole SubgCache branch: run() lines pipeline.cpp:212-293 + run_batch -------- */
typedef struct {
    sgc_subgraphs retrieved;   /* per query (retrieval is outside the hot path) */
    sgc_token_lists questions; /* per query: question wrapper bytes (Tokenizer::encode_bytes) */
    sgc_token_lists answers;   /* per query: copy-pointer target, count 0 = lookup off */
    sgc_token_lists own_prefix;/* per query: BOS + own prompt prefix (fallback path) */
    uint32_t clusters;         /* ClusterConfig::cluster_count */
    int linkage;               /* SGC_WARD .. */
    uint32_t question_budget;  /* RunConfig::question_budget (128) */
    int soft_prefix;           /* RunConfig::soft_prefix_enabled() */
    float pointer_bonus;       /* EngineOptions::pointer_bonus (100) */
    sgc_gnn_config gnn;
    /* multi-GPU (whole clusters per GPU): with world_size > 1 every rank
     * clusters the gathered embeddings redundantly (bit-identical labels), assigns clusters
     * to ranks by LPT on their cost (prefix + member rows, FLOP-weighted) and serves only its
     * own. cluster_owner (optional) forces the assignment. */
    const float* precomputed_embeddings; /* [m * dim] (all-gathered) or NULL to encode here */
    const uint32_t* cluster_owner;       /* [c] or NULL = LPT over world_size */
    int rank;                            /* ignored when the context has a transport (its rank) */
    int world_size;                      /* 0 or 1 = single GPU; with a transport: 0 or its world */
    /* clusters are served in `waves` groups of balanced cost (index order): members of an early
     * wave get their first token before later waves run (lower TTFT); 0/1 = one pass */
    uint32_t waves;
    /* greedy decode past the first token (ToyLm::greedy_decode, lm_core.cpp:352-404, batched over
     * every member of a wave): 0 or 1 = first token only; N > 1 = up to N tokens per query
     * (run() uses ToyLmConfig::max_new_tokens, pipeline.cpp:186) */
    uint32_t max_new_tokens;
    /* world_size > 1: rebalance skewed clusters at member level: after the
     * cluster LPT, members of the busiest rank's largest cluster move to the idlest rank while that
     * beats replicating the cluster's prefix there (the receiving rank prefills the identical
     * representative itself; sgc_balance_members is the plan) */
    int split_clusters;
    /* split clusters with a context transport: 1 = the rank that prefilled the representative
     * sends its sealed K/V to the other serving ranks (point to point) when the copy costs less
     * than a prefill (bytes over NVLink vs FLOPs on the tensor cores), else they prefill an
     * identical replica; 2 = always send; 0 = always replicate. Ignored without a transport. */
    int transfer_prefix;
    /* KVCache::prefix_digest at seal and again after the cluster's members are served
     * (cache_engine.cpp:189, :210): SGC_LOGIC if the sealed K/V changed. 0 = skip the check. */
    int verify_prefix;
} sgc_batch;

typedef struct {
    float* embeddings;      /* [m * dim] optional */
    uint32_t* labels;       /* [m] optional */
    uint32_t* merge_left;   /* [m - c] optional */
    uint32_t* merge_right;  /* [m - c] optional */
    double* merge_dist;     /* [m - c] optional */
    uint64_t* prefix_len;   /* [c] optional: representative prompt tokens (incl. soft slot) */
    float* logits;          /* [m * 260] optional, HOST memory (rows of unserved queries untouched) */
    int32_t* first_token;   /* [m] optional, HOST memory (untouched for queries not served here) */
    uint8_t* fallback;      /* [m] optional, HOST memory */
    uint32_t* owner;        /* [c] optional: rank serving each cluster */
    float* ttft_ms;         /* [m] optional: submission -> first token (-1 if not served here) */
    uint32_t waves;         /* waves actually run */
    double stage_ms[8];     /* encode, cluster, represent (host clock); prefill, extend (device events,
                             * summed over waves); total; decode (host clock); - */
    uint64_t prefill_rows, extend_rows; /* tokens pushed through prefill / extend */
    /* with batch.max_new_tokens > 1 (all optional, HOST memory): */
    int32_t* tokens;        /* [m * max_new_tokens] generated ids, -1 padded (GenerationResult::token_ids) */
    uint32_t* n_tokens;     /* [m] tokens generated (stops on EOS, max_new, full context) */
    float* rt_ms;           /* [m] submission -> last token (QueryOutcome::rt_ms semantics) */
    uint64_t decode_rows;   /* member-steps pushed through the decode forward */
    /* ledger / report timings (optional, HOST memory; ms since submission like ttft_ms):
     * seal_ms [c]  the cluster's prefix sealed (its wave's prefill done), -1 if not served here
     * pftt_ms [m]  QueryOutcome::pftt_ms: the query's own work start (its wave's extend, or its
     *              standalone prefill for a fallback) -> first token */
    float* seal_ms;
    float* pftt_ms;
    /* multi-GPU bookkeeping (optional, HOST memory): query_rank [m] = rank that served each query;
     * prefilled [c] = 1 if THIS rank ran the representative's prefill (0 for a received copy).
     * With a context transport, logits / first_token / fallback / ttft_ms / pftt_ms / tokens /
     * n_tokens / rt_ms of every query are gathered to rank 0 (other ranks hold their own). */
    uint32_t* query_rank;
    uint8_t* prefilled;
    uint64_t prefix_bytes_sent, prefix_bytes_received; /* sealed K/V moved point to point */
    /* paged KV cache: [c] digest of each sealed prefix this rank held (0 otherwise; see
     * sgc_kv_digest), peak pages in use during the batch, bytes per page (K + V, all layers) */
    uint64_t* prefix_digest;
    uint64_t kv_pages_peak, kv_page_bytes;
    /* [m] optional, HOST: the reference's TTFT semantics (QueryOutcome::ttft_ms, cache_engine.cpp:
     * 149, 169, 97-100): cluster dequeue -> first token. A cluster is dequeued when its wave starts
     * (its representative's prefill), so this excludes encode / cluster / represent and earlier
     * waves; -1 if not served here. ttft_ms above is the paper's submission -> first token. */
    float* ttft_dequeue_ms;
} sgc_batch_out;

int sgc_run_subgcache(sgc_ctx* ctx, sgc_model* model, sgc_graph* g, const sgc_batch* batch,
                      sgc_batch_out* out);

/* Cluster -> rank assignment used by sgc_run_subgcache when world_size > 1: longest
 * processing time first (descending cost, ties by cluster index) onto the least-loaded rank
 * (ties by rank). Host-only (no device needed). */
int sgc_lpt_assign(const double* cost, uint32_t clusters, int world_size, uint32_t* owner);
/* Member-level plan used with sgc_batch.split_clusters: cluster LPT on prefill + member cost, then
 * members of the busiest rank's largest cluster move to the idlest rank while max load drops even
 * after paying that rank a prefix replica (prefill_cost). query_owner [m], cluster_owner [c] (the
 * rank that prefills the cluster first; replicas are implied by query_owner). Host-only. */
int sgc_balance_members(const double* prefill_cost, uint32_t clusters, const uint32_t* labels,
                        const double* member_cost, uint32_t m, int world_size, uint32_t* query_owner,
                        uint32_t* cluster_owner);

/* ---- GEMM building block (exposed for parity tests and the roofline bench) -----------
 * D[M x N] = A[M x K] (bf16, row-major) * B[N x K]^T (bf16, row-major), fp32 accumulate in
 * TMEM via tcgen05.mma; epi 0 = store fp32 D, 1 = store bf16 D, 2 = D += into fp32 `d`,
 * 3 = bf16(tanh(D)); epi | 256 = a decode-step GEMM (few rows: the stream-K / split-K kernels
 * may run, fp32 summation order differs). All pointers device. K % 64 == 0, N % 64 == 0. */
int sgc_gemm_bf16(sgc_ctx* ctx, const void* a, const void* b, void* d, uint32_t M, uint32_t N,
                  uint32_t K, int epi);
/* ---- cascade attention building block (parity tests at full size; lm_core.cpp:246-274) ----
 * out[r, h*hd:(h+1)*hd] = softmax over { prefix keys pfx_kv0 .. pfx_kv0+pfx_len-1 of (k_pfx, v_pfx) }
 * U { own keys seg_lo[r] .. r of (k_loc, v_loc) } with scale 1/sqrt(hd), for every row r of every
 * work unit. `work` is a HOST array of n_work x {row0, nrows, pfx_kv0, pfx_len}; units hold
 * <= 256 rows (hd 64/128, tcgen05 kernel) or <= 64 rows (hd 16/32), rows of one unit share
 * one prefix. q/out/k_loc/v_loc are [rows x d] bf16, k_pfx/v_pfx [pfx_rows x d] bf16, seg_lo
 * [rows] int32; all device pointers. */
int sgc_attention_bf16(sgc_ctx* ctx, const void* q, const void* k_pfx, const void* v_pfx,
                       uint32_t pfx_rows, const void* k_loc, const void* v_loc, const int32_t* seg_lo,
                       const int32_t* work, uint32_t n_work, uint32_t rows, uint32_t d, uint32_t heads,
                       void* out);
/* Measured FP64 throughput of the context's device (TFLOP/s): the larger of the FMA pipe (DFMA
 * chains) and the FP64 tensor pipe (DMMA chains) -- the GNN layer map's roofline denominator
 * (bench.py). */
int sgc_probe_fp64_tflops(sgc_ctx* ctx, double* tflops);
/* Work of the context's last GNN encode: unique node states computed over all layers (identical
 * in-neighbourhood signatures are computed once) and the reference's node instances x layers. */
int sgc_gnn_stats(const sgc_ctx* ctx, uint64_t* state_rows, uint64_t* node_instances);
/* Enable/disable per-kernel CUDA-event timing; sgc_get_timing reads the accumulated totals. */
int sgc_set_timing(sgc_ctx* ctx, int enable);
/* Tuning knobs (A/B switches; the defaults are the measured best):
 * "gemm_pairs" (1 = CTA-pair tcgen05 GEMM for 256-wide tiles, default; 0 = 1-CTA);
 * "gemm_raster" (CTA-pair raster: 0 = M-groups, default; 1 = by estimated DRAM bytes; 2 = N-groups);
 * "gemm_streamk" (decode-step GEMMs on the stream-K CTA-pair kernel: 1 = where measured faster,
 * default; 2 = every decode shape; 0 = off);
 * "decode_defer_pct" (generation: a wave decodes on its own until fewer than this percentage of
 * its queries still generate, the stragglers of every wave then finish in one shared loop;
 * default 25, 0 = each wave to completion, >= 100 = all decoding after the last wave);
 * "attn_split" (1 = two softmax warpgroups per query tile; default 0);
 * "attn_kernel" / "attn_kernel_partial" (tcgen05 attention for prefill / extend and for the
 * decode prefix partials: 0 = two-tile kernel, 1 = one-tile S-triple-buffered kernel; defaults
 * 0 / 1);
 * "gnn_tile" (GNN layer-map FP64 GEMM: 0 = 64x64, 1 = 64x128, 2 = 128x128 DFMA tiles, 3 = DMMA
 * tensor pipe, default); "gnn_dedup" (1 = identical node states computed once, default);
 * "agglomerate_global" (1 = the merge loop keeps its per-row state in global memory at any m, as
 * it always does above ~8k points; default 0).
 * Unknown names return SGC_DOMAIN. */
int sgc_set_option(sgc_ctx* ctx, const char* name, int64_t value);
int sgc_get_timing(sgc_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* SGC_B200_H */
