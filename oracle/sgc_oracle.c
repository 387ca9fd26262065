/*
 * sgc_oracle.c -- CPU restatement of the SubGCache hot path.
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA path, never the thing
 * measured or shipped. Every function cites the reference lines it restates
 * (relative to /root/reference/proj). Compiled with -ffp-contract=off so each
 * float/double operation rounds exactly as written, like the reference's
 * Release objects (no vfmadd outside kernels_avx2.cpp).
 */
#include "sgc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */

/* rng.hpp:17-22 SplitMix64::next with counter state */
static inline uint64_t sm_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:36-39 */
uint64_t sgo_splitmix64_once(uint64_t x) {
    uint64_t s = x;
    return sm_next(&s);
}

/* rng.hpp:50-57 fnv1a64_bytes */
uint64_t sgo_fnv1a64(const void* data, size_t n, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* rng.hpp:25-28 uniform: lo + (hi-lo)*u, u = top 24 bits * 2^-24 (no FMA) */
void sgo_fill_uniform_state(float* w, size_t n, uint64_t state0, float lo, float hi) {
    uint64_t st = state0;
    for (size_t i = 0; i < n; ++i) {
        float u = (float)(sm_next(&st) >> 40) * 0x1.0p-24f;
        w[i] = lo + (hi - lo) * u;
    }
}

/* lm_core.cpp:19-23 */
void sgo_fill_uniform(float* w, size_t n, uint64_t seed, size_t fan_in) {
    float scale = sqrtf(3.0f / (float)fan_in);
    sgo_fill_uniform_state(w, n, sgo_splitmix64_once(seed), -scale, scale);
}

/* --------------------------------------------------------- text encoder */

/* encoders.cpp:50-55 */
void sgo_text_projection(float* proj, uint32_t dim, uint64_t seed) {
    sgo_fill_uniform_state(proj, (size_t)dim * SGO_BUCKETS,
                           sgo_splitmix64_once(seed ^ 0x7e87a11dULL), -1.0f, 1.0f);
}

/* encoders.cpp:20-24 is_token_char: isalnum (C locale) or byte >= 0x80 */
static int is_token_char(unsigned char c) {
    return (c >= '0' && c <= '9') || (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') ||
           c >= 0x80;
}

/* encoders.cpp:62-80: lowercased tokens -> (bucket, sign) */
size_t sgo_text_hash(const char* text, size_t len, uint64_t salt, uint32_t* buckets,
                     int8_t* signs, size_t cap) {
    size_t count = 0;
    uint64_t h = 0xcbf29ce484222325ULL;
    size_t tok_len = 0;
    for (size_t i = 0; i <= len; ++i) {
        if (i < len && is_token_char((unsigned char)text[i])) {
            unsigned char c = (unsigned char)text[i];
            if (c >= 'A' && c <= 'Z') c = (unsigned char)(c - 'A' + 'a');
            h ^= c;
            h *= 0x100000001b3ULL;
            ++tok_len;
            continue;
        }
        if (tok_len) {
            uint64_t hh = sgo_splitmix64_once(h ^ salt);
            if (count < cap) {
                buckets[count] = (uint32_t)(hh % SGO_BUCKETS);
                signs[count] = ((hh >> 32) & 1) ? 1 : -1;
            }
            ++count;
            h = 0xcbf29ce484222325ULL;
            tok_len = 0;
        }
    }
    return count;
}

/* encoders.cpp:57-93 */
void sgo_text_embed(const float* proj, uint32_t dim, uint64_t salt, const char* text, size_t len,
                    float* out) {
    size_t cap = len + 1;
    uint32_t* b = (uint32_t*)malloc(cap * sizeof(uint32_t));
    int8_t* s = (int8_t*)malloc(cap);
    size_t nt = sgo_text_hash(text, len, salt, b, s, cap);
    double* acc = (double*)calloc(dim, sizeof(double));
    for (size_t t = 0; t < nt; ++t) {
        double sign = s[t] > 0 ? 1.0 : -1.0;
        const float* col = proj + b[t];
        for (uint32_t d = 0; d < dim; ++d) acc[d] += sign * col[(size_t)d * SGO_BUCKETS];
    }
    for (uint32_t d = 0; d < dim; ++d) out[d] = 0.0f;
    if (nt) {
        double norm = 0;
        for (uint32_t d = 0; d < dim; ++d) norm += acc[d] * acc[d];
        norm = sqrt(norm);
        if (norm > 0)
            for (uint32_t d = 0; d < dim; ++d) out[d] = (float)(acc[d] / norm);
    }
    free(acc);
    free(b);
    free(s);
}

/* ---------------------------------------------------------- GNN encoder */

/* encoders.cpp:95-104 */
void sgo_gnn_weights(float* w, uint32_t layers, uint32_t heads, uint32_t dim, uint64_t seed) {
    float scale = sqrtf(3.0f / (float)dim);
    sgo_fill_uniform_state(w, (size_t)layers * heads * dim * dim,
                           sgo_splitmix64_once(seed ^ 0x6e6eULL), -scale, scale);
}

/* encoders.cpp:106-120 apply_layer */
static void apply_layer(const float* w, uint32_t layer, uint32_t heads, uint32_t d,
                        const double* x, double* z) {
    for (uint32_t r = 0; r < d; ++r) z[r] = 0.0;
    for (uint32_t h = 0; h < heads; ++h) {
        const float* wh = w + ((size_t)layer * heads + h) * d * d;
        for (uint32_t r = 0; r < d; ++r) {
            double acc = 0;
            const float* row = wh + (size_t)r * d;
            for (uint32_t c = 0; c < d; ++c) acc += (double)row[c] * x[c];
            z[r] += acc;
        }
    }
    double inv_heads = 1.0 / heads;
    for (uint32_t r = 0; r < d; ++r) z[r] = tanh(z[r] * inv_heads);
}

/* encoders.cpp:122-186 encode */
int sgo_gnn_encode(const float* w, uint32_t layers, uint32_t heads, uint32_t dim,
                   const float* node_feat, uint32_t n, const uint32_t* msg_src,
                   const uint32_t* msg_dst, const float* msg_gate, uint32_t e, float* out) {
    if (n == 0) return 1; /* DomainError: empty subgraph */
    size_t d = dim;
    double* state = (double*)malloc(n * d * sizeof(double));
    double* agg = (double*)malloc(n * d * sizeof(double));
    uint32_t* fanin = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (size_t i = 0; i < n * d; ++i) state[i] = node_feat[i];
    for (uint32_t layer = 0; layer < layers; ++layer) {
        memcpy(agg, state, n * d * sizeof(double));
        for (uint32_t v = 0; v < n; ++v) fanin[v] = 1;
        for (uint32_t m = 0; m < e; ++m) {
            double* a = agg + msg_dst[m] * d;
            const double* s = state + msg_src[m] * d;
            const float* g = msg_gate + m * d;
            for (size_t k = 0; k < d; ++k) a[k] += s[k] * (double)g[k];
            ++fanin[msg_dst[m]];
        }
        for (uint32_t v = 0; v < n; ++v) {
            double inv = 1.0 / fanin[v];
            for (size_t k = 0; k < d; ++k) agg[v * d + k] *= inv;
            apply_layer(w, layer, heads, dim, agg + v * d, state + v * d);
        }
    }
    double* pooled = (double*)calloc(d, sizeof(double));
    for (uint32_t v = 0; v < n; ++v)
        for (size_t k = 0; k < d; ++k) pooled[k] += state[v * d + k];
    double inv_n = 1.0 / (double)n;
    double norm = 0;
    for (size_t k = 0; k < d; ++k) {
        pooled[k] *= inv_n;
        norm += pooled[k] * pooled[k];
    }
    norm = sqrt(norm);
    for (size_t k = 0; k < d; ++k) out[k] = norm > 0 ? (float)(pooled[k] / norm) : 0.0f;
    free(pooled);
    free(state);
    free(agg);
    free(fanin);
    return 0;
}

/* ----------------------------------------------------------- clustering */

/* encoders.cpp:40-48 euclidean_distance */
static double euclid(const float* a, const float* b, uint32_t d) {
    double acc = 0;
    for (uint32_t i = 0; i < d; ++i) {
        double v = (double)a[i] - b[i];
        acc += v * v;
    }
    return sqrt(acc);
}

/* clustering.cpp:33-45 */
void sgo_pairwise(const float* emb, uint32_t m, uint32_t d, double* out) {
    for (uint32_t i = 0; i < m; ++i) {
        out[(size_t)i * m + i] = 0.0;
        for (uint32_t j = i + 1; j < m; ++j) {
            double v = euclid(emb + (size_t)i * d, emb + (size_t)j * d, d);
            out[(size_t)i * m + j] = v;
            out[(size_t)j * m + i] = v;
        }
    }
}

/* clustering.cpp:60-174 agglomerate (Lance-Williams) */
int sgo_agglomerate(const float* emb, uint32_t m, uint32_t d, int linkage, uint32_t c,
                    uint32_t* labels, uint32_t* merge_left_min, uint32_t* merge_right_min,
                    double* merge_dist, uint64_t* op_count) {
    if (c < 1 || c > m || m == 0) return 1;
    int squared = linkage == SGO_WARD || linkage == SGO_CENTROID;
    double* dist = (double*)malloc((size_t)m * m * sizeof(double));
    sgo_pairwise(emb, m, d, dist);
    uint64_t ops = (uint64_t)m * (m - 1) / 2 * d;
    if (squared)
        for (size_t i = 0; i < (size_t)m * m; ++i) dist[i] *= dist[i];
    unsigned char* alive = (unsigned char*)malloc(m);
    uint32_t* size = (uint32_t*)malloc(m * sizeof(uint32_t));
    uint32_t* minm = (uint32_t*)malloc(m * sizeof(uint32_t));
    uint32_t* owner = (uint32_t*)malloc(m * sizeof(uint32_t));
    for (uint32_t i = 0; i < m; ++i) {
        alive[i] = 1;
        size[i] = 1;
        minm[i] = i;
        owner[i] = i;
    }
#define D(i, j) dist[(size_t)(i) * m + (j)]
    uint32_t active = m, step = 0;
    while (active > c) {
        double best = INFINITY;
        uint32_t bi = m, bj = m, bk0 = 0, bk1 = 0;
        for (uint32_t i = 0; i < m; ++i) {
            if (!alive[i]) continue;
            for (uint32_t j = i + 1; j < m; ++j) {
                if (!alive[j]) continue;
                ++ops;
                double v = D(i, j);
                uint32_t k0 = minm[i] < minm[j] ? minm[i] : minm[j];
                uint32_t k1 = minm[i] < minm[j] ? minm[j] : minm[i];
                if (v < best || (v == best && (k0 < bk0 || (k0 == bk0 && k1 < bk1)))) {
                    best = v;
                    bi = i;
                    bj = j;
                    bk0 = k0;
                    bk1 = k1;
                }
            }
        }
        uint32_t keep = minm[bi] < minm[bj] ? bi : bj;
        uint32_t kill = keep == bi ? bj : bi;
        double na = size[keep], nb = size[kill];
        merge_left_min[step] = minm[keep];
        merge_right_min[step] = minm[kill];
        merge_dist[step] = linkage == SGO_WARD ? best / 2.0
                         : linkage == SGO_CENTROID ? sqrt(best) : best;
        ++step;
        for (uint32_t k = 0; k < m; ++k) {
            if (!alive[k] || k == keep || k == kill) continue;
            ++ops;
            double dak = D(keep, k), dbk = D(kill, k), dab = D(keep, kill);
            double nk = size[k];
            double v = 0;
            switch (linkage) {
                case SGO_SINGLE: v = dak < dbk ? dak : dbk; break;
                case SGO_COMPLETE: v = dak > dbk ? dak : dbk; break;
                case SGO_AVERAGE: v = (na * dak + nb * dbk) / (na + nb); break;
                case SGO_CENTROID:
                    v = (na * dak + nb * dbk) / (na + nb) - (na * nb * dab) / ((na + nb) * (na + nb));
                    break;
                case SGO_WARD:
                    v = ((na + nk) * dak + (nb + nk) * dbk - nk * dab) / (na + nb + nk);
                    break;
            }
            D(keep, k) = v;
            D(k, keep) = v;
        }
        alive[kill] = 0;
        size[keep] += size[kill];
        if (minm[kill] < minm[keep]) minm[keep] = minm[kill];
        for (uint32_t i = 0; i < m; ++i)
            if (owner[i] == kill) owner[i] = keep;
        --active;
    }
#undef D
    /* labels by ascending min member (clustering.cpp:162-172) */
    uint32_t* label_of_slot = (uint32_t*)malloc(m * sizeof(uint32_t));
    uint32_t next = 0;
    /* alive slot index == its min member (keep always holds the smaller min) */
    for (uint32_t i = 0; i < m; ++i)
        if (alive[i]) label_of_slot[i] = next++;
    for (uint32_t i = 0; i < m; ++i) labels[i] = label_of_slot[owner[i]];
    if (op_count) *op_count = ops;
    free(label_of_slot);
    free(dist);
    free(alive);
    free(size);
    free(minm);
    free(owner);
    return 0;
}

/* tests/support/cluster_oracle.hpp:23-116: naive set-linkage agglomeration */
int sgo_naive_agglomerate(const float* pts, uint32_t m, uint32_t dim, int linkage, uint32_t c,
                          uint32_t* labels, double* merge_dist) {
    if (c < 1 || c > m) return 1;
    double* pd = (double*)malloc((size_t)m * m * sizeof(double));
    for (uint32_t i = 0; i < m; ++i)
        for (uint32_t j = 0; j < m; ++j)
            pd[(size_t)i * m + j] = euclid(pts + (size_t)i * dim, pts + (size_t)j * dim, dim);
    /* clusters as sorted member lists; cl_start/cl_len into a member pool */
    uint32_t** cl = (uint32_t**)malloc(m * sizeof(uint32_t*));
    uint32_t* cn = (uint32_t*)malloc(m * sizeof(uint32_t));
    for (uint32_t i = 0; i < m; ++i) {
        cl[i] = (uint32_t*)malloc(m * sizeof(uint32_t));
        cl[i][0] = i;
        cn[i] = 1;
    }
    uint32_t nc = m, step = 0;
    double* ca = (double*)malloc(dim * sizeof(double));
    double* cb = (double*)malloc(dim * sizeof(double));
    while (nc > c) {
        double best = INFINITY;
        uint32_t bi = 0, bj = 0, bk0 = 0, bk1 = 0;
        for (uint32_t i = 0; i < nc; ++i) {
            for (uint32_t j = i + 1; j < nc; ++j) {
                double v = 0;
                const uint32_t *a = cl[i], *b = cl[j];
                uint32_t na_ = cn[i], nb_ = cn[j];
                if (linkage == SGO_SINGLE) {
                    v = INFINITY;
                    for (uint32_t x = 0; x < na_; ++x)
                        for (uint32_t y = 0; y < nb_; ++y) {
                            double t = pd[(size_t)a[x] * m + b[y]];
                            v = t < v ? t : v;
                        }
                } else if (linkage == SGO_COMPLETE) {
                    v = 0;
                    for (uint32_t x = 0; x < na_; ++x)
                        for (uint32_t y = 0; y < nb_; ++y) {
                            double t = pd[(size_t)a[x] * m + b[y]];
                            v = t > v ? t : v;
                        }
                } else if (linkage == SGO_AVERAGE) {
                    double sum = 0;
                    for (uint32_t x = 0; x < na_; ++x)
                        for (uint32_t y = 0; y < nb_; ++y) sum += pd[(size_t)a[x] * m + b[y]];
                    v = sum / ((double)na_ * (double)nb_);
                } else {
                    for (uint32_t k = 0; k < dim; ++k) ca[k] = cb[k] = 0;
                    for (uint32_t x = 0; x < na_; ++x)
                        for (uint32_t k = 0; k < dim; ++k) ca[k] += pts[(size_t)a[x] * dim + k];
                    for (uint32_t y = 0; y < nb_; ++y)
                        for (uint32_t k = 0; k < dim; ++k) cb[k] += pts[(size_t)b[y] * dim + k];
                    double gap2 = 0;
                    for (uint32_t k = 0; k < dim; ++k) {
                        double t = ca[k] / na_ - cb[k] / nb_;
                        gap2 += t * t;
                    }
                    if (linkage == SGO_CENTROID) v = sqrt(gap2);
                    else {
                        double fa = na_, fb = nb_;
                        v = fa * fb / (fa + fb) * gap2;
                    }
                }
                uint32_t k0 = a[0] < b[0] ? a[0] : b[0];
                uint32_t k1 = a[0] < b[0] ? b[0] : a[0];
                if (v < best || (v == best && (k0 < bk0 || (k0 == bk0 && k1 < bk1)))) {
                    best = v;
                    bi = i;
                    bj = j;
                    bk0 = k0;
                    bk1 = k1;
                }
            }
        }
        if (merge_dist) merge_dist[step] = best;
        ++step;
        /* std::merge of the two sorted lists into bi, erase bj */
        uint32_t* merged = (uint32_t*)malloc(m * sizeof(uint32_t));
        uint32_t x = 0, y = 0, t = 0;
        while (x < cn[bi] || y < cn[bj]) {
            if (y >= cn[bj] || (x < cn[bi] && cl[bi][x] <= cl[bj][y])) merged[t++] = cl[bi][x++];
            else merged[t++] = cl[bj][y++];
        }
        free(cl[bi]);
        cl[bi] = merged;
        cn[bi] = t;
        free(cl[bj]);
        for (uint32_t k = bj; k + 1 < nc; ++k) {
            cl[k] = cl[k + 1];
            cn[k] = cn[k + 1];
        }
        --nc;
    }
    /* sort clusters by front, label */
    for (uint32_t i = 0; i < nc; ++i)
        for (uint32_t j = i + 1; j < nc; ++j)
            if (cl[j][0] < cl[i][0]) {
                uint32_t* tp = cl[i]; cl[i] = cl[j]; cl[j] = tp;
                uint32_t tn = cn[i]; cn[i] = cn[j]; cn[j] = tn;
            }
    for (uint32_t l = 0; l < nc; ++l)
        for (uint32_t x = 0; x < cn[l]; ++x) labels[cl[l][x]] = l;
    for (uint32_t i = 0; i < nc; ++i) free(cl[i]);
    free(cl);
    free(cn);
    free(pd);
    free(ca);
    free(cb);
    return 0;
}

/* ------------------------------------------- representative construction */

/* graph_store.cpp:223-235 merge_subgraphs: std::set union == ascending unique */
uint32_t sgo_union(const uint32_t* const* lists, const uint32_t* lens, uint32_t n_lists,
                   uint32_t universe, uint32_t* out) {
    unsigned char* bits = (unsigned char*)calloc(universe ? universe : 1, 1);
    for (uint32_t l = 0; l < n_lists; ++l)
        for (uint32_t i = 0; i < lens[l]; ++i) bits[lists[l][i]] = 1;
    uint32_t n = 0;
    for (uint32_t i = 0; i < universe; ++i)
        if (bits[i]) out[n++] = i;
    free(bits);
    return n;
}

/* graph_store.cpp:237-247 csv_quote */
size_t sgo_csv_quote(const char* f, size_t len, char* dst) {
    int need = 0;
    for (size_t i = 0; i < len; ++i)
        if (f[i] == ',' || f[i] == '"' || f[i] == '\n') need = 1;
    if (!need) {
        if (dst) memcpy(dst, f, len);
        return len;
    }
    size_t n = 0;
    if (dst) dst[n] = '"';
    ++n;
    for (size_t i = 0; i < len; ++i) {
        if (f[i] == '"') {
            if (dst) { dst[n] = '"'; dst[n + 1] = '"'; }
            n += 2;
        } else {
            if (dst) dst[n] = f[i];
            ++n;
        }
    }
    if (dst) dst[n] = '"';
    return n + 1;
}

static const char kHeader[] = "Use the following graph to answer the question.\n\n";
static const char kNodeHdr[] = "node id,node attr";
static const char kEdgeHdr[] = "src,edge attr,dst";

/* cache_engine.cpp:43-70 prefix side of build_prompt, then tokenize (tokenizer.cpp:5-11) */
long sgo_build_prefix(const char* const* node_rows, const uint32_t* node_len, uint32_t n_nodes,
                      const char* const* edge_rows, const uint32_t* edge_len, uint32_t n_edges,
                      uint32_t budget_tokens, int32_t* tokens, uint32_t* dropped_nodes,
                      uint32_t* dropped_edges) {
    size_t budget_bytes = budget_tokens == 0 ? 0 : budget_tokens - 1;
    size_t base = strlen(kHeader) + strlen(kNodeHdr) + strlen(kEdgeHdr) + 2;
    size_t node_bytes = 0, edge_bytes = 0;
    for (uint32_t i = 0; i < n_nodes; ++i) node_bytes += node_len[i] + 1;
    for (uint32_t i = 0; i < n_edges; ++i) edge_bytes += edge_len[i] + 1;
    uint32_t ke = n_edges, kn = n_nodes;
    while (ke > 0 && base + node_bytes + edge_bytes > budget_bytes) {
        --ke;
        edge_bytes -= edge_len[ke] + 1;
    }
    while (kn > 0 && base + node_bytes + edge_bytes > budget_bytes) {
        --kn;
        node_bytes -= node_len[kn] + 1;
    }
    if (base + node_bytes + edge_bytes > budget_bytes) return -1;
    if (dropped_nodes) *dropped_nodes = n_nodes - kn;
    if (dropped_edges) *dropped_edges = n_edges - ke;
    long t = 0;
    tokens[t++] = 256; /* BOS */
#define PUT(p, n)                                                        \
    do {                                                                 \
        for (size_t _i = 0; _i < (n); ++_i) tokens[t++] = (unsigned char)(p)[_i]; \
    } while (0)
    PUT(kHeader, strlen(kHeader));
    PUT(kNodeHdr, strlen(kNodeHdr));
    tokens[t++] = '\n';
    for (uint32_t i = 0; i < kn; ++i) {
        PUT(node_rows[i], node_len[i]);
        tokens[t++] = '\n';
    }
    PUT(kEdgeHdr, strlen(kEdgeHdr));
    tokens[t++] = '\n';
    for (uint32_t i = 0; i < ke; ++i) {
        PUT(edge_rows[i], edge_len[i]);
        tokens[t++] = '\n';
    }
#undef PUT
    return t;
}

/* cache_engine.cpp:33-41 question side */
long sgo_question_tokens(const char* q, size_t len, uint32_t question_budget, int32_t* tokens) {
    static const char pre[] = "\nQuestion: ";
    static const char post[] = "\nAnswer:";
    size_t wrapper = strlen(pre) + strlen(post);
    if (question_budget <= wrapper) return -1;
    size_t room = question_budget - wrapper;
    if (len > room) len = room;
    long t = 0;
    for (size_t i = 0; i < strlen(pre); ++i) tokens[t++] = (unsigned char)pre[i];
    for (size_t i = 0; i < len; ++i) tokens[t++] = (unsigned char)q[i];
    for (size_t i = 0; i < strlen(post); ++i) tokens[t++] = (unsigned char)post[i];
    return t;
}

/* ---------------------------------------------------------------- ToyLm */

#define VOCAB 260

struct sgo_lm {
    uint32_t L, H, d, hd, ffn, max_seq;
    float *tok, *head;
    float **wqkv, **wo, **w1, **w2;
    float *rcos, *rsin;
};

struct sgo_kv {
    const sgo_lm* lm;
    uint32_t n;       /* tokens */
    float **k, **v;   /* [L][max_seq*d] */
    int32_t* ids;
};

/* kernels_scalar.cpp:10-14 (sequential fp32 dot) */
static float dotf(const float* a, const float* b, size_t n) {
    float acc = 0.0f;
    for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

static void matvec(const float* w, const float* x, float* y, size_t rows, size_t cols) {
    for (size_t r = 0; r < rows; ++r) y[r] = dotf(w + r * cols, x, cols);
}

/* kernels_scalar.cpp:42-64 Cephes polynomial exp */
static float expf_poly(float x) {
    const float kExpHi = 88.3762626647950f, kExpLo = -88.3762626647949f;
    x = x > kExpHi ? kExpHi : x;
    x = x < kExpLo ? kExpLo : x;
    float fx = fmaf(x, 1.44269504088896341f, 0.5f);
    fx = floorf(fx);
    x = fmaf(fx, -0.693359375f, x);
    x = fmaf(fx, 2.12194440e-4f, x);
    float z = x * x;
    float y = 1.9875691500e-4f;
    y = fmaf(y, x, 1.3981999507e-3f);
    y = fmaf(y, x, 8.3334519073e-3f);
    y = fmaf(y, x, 4.1665795894e-2f);
    y = fmaf(y, x, 1.6666665459e-1f);
    y = fmaf(y, x, 5.0000001201e-1f);
    y = fmaf(y, z, x);
    y += 1.0f;
    int n = (int)fx;
    union { int i; float f; } bits;
    bits.i = (n + 127) << 23;
    return y * bits.f;
}

/* lm_core.cpp:26-31 rmsnorm without gain */
static void rmsnorm(const float* x, float* out, size_t n) {
    float ms = dotf(x, x, n) / (float)n;
    float inv = 1.0f / sqrtf(ms + 1e-5f);
    for (size_t i = 0; i < n; ++i) out[i] = x[i] * inv;
}

/* lm_core.cpp:122-161 */
sgo_lm* sgo_lm_create(uint32_t layers, uint32_t heads, uint32_t dim, uint32_t ffn,
                      uint32_t max_seq, uint64_t seed) {
    if (!layers || !heads || !dim || dim % heads) return NULL;
    sgo_lm* lm = (sgo_lm*)calloc(1, sizeof(sgo_lm));
    lm->L = layers; lm->H = heads; lm->d = dim; lm->hd = dim / heads;
    lm->ffn = ffn; lm->max_seq = max_seq;
    size_t d = dim;
    lm->tok = (float*)malloc(VOCAB * d * sizeof(float));
    lm->head = (float*)malloc(VOCAB * d * sizeof(float));
    sgo_fill_uniform(lm->tok, VOCAB * d, seed ^ 0x10ad1ULL, d);
    sgo_fill_uniform(lm->head, VOCAB * d, seed ^ 0x8eadULL, d);
    lm->wqkv = (float**)calloc(layers, sizeof(float*));
    lm->wo = (float**)calloc(layers, sizeof(float*));
    lm->w1 = (float**)calloc(layers, sizeof(float*));
    lm->w2 = (float**)calloc(layers, sizeof(float*));
    for (uint32_t l = 0; l < layers; ++l) {
        lm->wqkv[l] = (float*)malloc(3 * d * d * sizeof(float));
        lm->wo[l] = (float*)malloc(d * d * sizeof(float));
        lm->w1[l] = (float*)malloc((size_t)ffn * d * sizeof(float));
        lm->w2[l] = (float*)malloc((size_t)ffn * d * sizeof(float));
        sgo_fill_uniform(lm->wqkv[l], 3 * d * d, seed ^ (0x9a11ULL + l * 4ULL), d);
        sgo_fill_uniform(lm->wo[l], d * d, seed ^ (0x9a12ULL + l * 4ULL), d);
        sgo_fill_uniform(lm->w1[l], (size_t)ffn * d, seed ^ (0x9a13ULL + l * 4ULL), d);
        sgo_fill_uniform(lm->w2[l], (size_t)ffn * d, seed ^ (0x9a14ULL + l * 4ULL), ffn);
    }
    uint32_t half = lm->hd / 2;
    lm->rcos = (float*)malloc((size_t)max_seq * (half ? half : 1) * sizeof(float));
    lm->rsin = (float*)malloc((size_t)max_seq * (half ? half : 1) * sizeof(float));
    for (uint32_t p = 0; p < max_seq; ++p)
        for (uint32_t i = 0; i < half; ++i) {
            float freq = powf(10000.0f, -2.0f * (float)i / (float)lm->hd);
            float angle = (float)p * freq;
            lm->rcos[(size_t)p * half + i] = cosf(angle);
            lm->rsin[(size_t)p * half + i] = sinf(angle);
        }
    return lm;
}

void sgo_lm_destroy(sgo_lm* lm) {
    if (!lm) return;
    for (uint32_t l = 0; l < lm->L; ++l) {
        free(lm->wqkv[l]); free(lm->wo[l]); free(lm->w1[l]); free(lm->w2[l]);
    }
    free(lm->wqkv); free(lm->wo); free(lm->w1); free(lm->w2);
    free(lm->tok); free(lm->head); free(lm->rcos); free(lm->rsin);
    free(lm);
}

/* which: 0 tok_embedding, 1 head, 2 wqkv, 3 wo, 4 w1, 5 w2, 6 rope_cos, 7 rope_sin */
const float* sgo_lm_weight(const sgo_lm* lm, int which, uint32_t layer, size_t* n) {
    size_t d = lm->d;
    switch (which) {
        case 0: *n = VOCAB * d; return lm->tok;
        case 1: *n = VOCAB * d; return lm->head;
        case 2: *n = 3 * d * d; return lm->wqkv[layer];
        case 3: *n = d * d; return lm->wo[layer];
        case 4: *n = (size_t)lm->ffn * d; return lm->w1[layer];
        case 5: *n = (size_t)lm->ffn * d; return lm->w2[layer];
        case 6: *n = (size_t)lm->max_seq * (lm->hd / 2); return lm->rcos;
        case 7: *n = (size_t)lm->max_seq * (lm->hd / 2); return lm->rsin;
    }
    *n = 0;
    return NULL;
}

sgo_kv* sgo_kv_create(const sgo_lm* lm) {
    sgo_kv* kv = (sgo_kv*)calloc(1, sizeof(sgo_kv));
    kv->lm = lm;
    kv->k = (float**)calloc(lm->L, sizeof(float*));
    kv->v = (float**)calloc(lm->L, sizeof(float*));
    for (uint32_t l = 0; l < lm->L; ++l) {
        kv->k[l] = (float*)malloc((size_t)lm->max_seq * lm->d * sizeof(float));
        kv->v[l] = (float*)malloc((size_t)lm->max_seq * lm->d * sizeof(float));
    }
    kv->ids = (int32_t*)malloc(lm->max_seq * sizeof(int32_t));
    return kv;
}

sgo_kv* sgo_kv_fork(const sgo_kv* src) {
    sgo_kv* kv = sgo_kv_create(src->lm);
    kv->n = src->n;
    for (uint32_t l = 0; l < src->lm->L; ++l) {
        memcpy(kv->k[l], src->k[l], (size_t)src->n * src->lm->d * sizeof(float));
        memcpy(kv->v[l], src->v[l], (size_t)src->n * src->lm->d * sizeof(float));
    }
    memcpy(kv->ids, src->ids, src->n * sizeof(int32_t));
    return kv;
}

void sgo_kv_destroy(sgo_kv* kv) {
    if (!kv) return;
    for (uint32_t l = 0; l < kv->lm->L; ++l) {
        free(kv->k[l]);
        free(kv->v[l]);
    }
    free(kv->k); free(kv->v); free(kv->ids);
    free(kv);
}

uint32_t sgo_kv_tokens(const sgo_kv* kv) { return kv->n; }
const float* sgo_kv_data(const sgo_kv* kv, int is_v, uint32_t layer) {
    return is_v ? kv->v[layer] : kv->k[layer];
}

/* lm_core.cpp:179-297 forward (token-sequential, scalar kernel order) */
static int forward(const sgo_lm* lm, sgo_kv* kv, const float* emb, const int32_t* ids,
                   uint32_t n_new, float* logits, float* all_logits) {
    const uint32_t d = lm->d, hd = lm->hd, half = hd / 2, H = lm->H;
    const float inv_sqrt_hd = 1.0f / sqrtf((float)hd);
    if (n_new == 0) return 0;
    if (kv->n + n_new > lm->max_seq) return 2;
    float* x = (float*)malloc((size_t)d * sizeof(float));
    float* xn = (float*)malloc(d * sizeof(float));
    float* qkv = (float*)malloc(3 * (size_t)d * sizeof(float));
    float* attn = (float*)malloc(d * sizeof(float));
    float* proj = (float*)malloc(d * sizeof(float));
    float* hbuf = (float*)malloc((size_t)lm->ffn * sizeof(float));
    float* scores = (float*)malloc((size_t)lm->max_seq * sizeof(float));
    float lg[VOCAB];
    const uint32_t base = kv->n;
    for (uint32_t t = 0; t < n_new; ++t) {
        const uint32_t pos = base + t;
        memcpy(x, emb + (size_t)t * d, d * sizeof(float));
        const float* cp = lm->rcos + (size_t)pos * half;
        const float* sp = lm->rsin + (size_t)pos * half;
        for (uint32_t l = 0; l < lm->L; ++l) {
            rmsnorm(x, xn, d);
            matvec(lm->wqkv[l], xn, qkv, 3 * (size_t)d, d);
            float* q = qkv;
            float* k = qkv + d;
            const float* v = qkv + 2 * (size_t)d;
            for (uint32_t h = 0; h < H; ++h) {
                float* qh = q + h * hd;
                float* kh = k + h * hd;
                for (uint32_t i = 0; i < half; ++i) {
                    float c = cp[i], s = sp[i];
                    float q0 = qh[i], q1 = qh[i + half];
                    qh[i] = q0 * c - q1 * s;
                    qh[i + half] = q1 * c + q0 * s;
                    float k0 = kh[i], k1 = kh[i + half];
                    kh[i] = k0 * c - k1 * s;
                    kh[i + half] = k1 * c + k0 * s;
                }
            }
            memcpy(kv->k[l] + (size_t)pos * d, k, d * sizeof(float));
            memcpy(kv->v[l] + (size_t)pos * d, v, d * sizeof(float));
            const uint32_t n_ctx = pos + 1;
            for (uint32_t h = 0; h < H; ++h) {
                float* qh = q + h * hd;
                for (uint32_t i = 0; i < hd; ++i) qh[i] *= inv_sqrt_hd;
                for (uint32_t j = 0; j < n_ctx; ++j)
                    scores[j] = dotf(qh, kv->k[l] + (size_t)j * d + h * hd, hd);
                float mx = scores[0];
                for (uint32_t j = 1; j < n_ctx; ++j) mx = scores[j] > mx ? scores[j] : mx;
                for (uint32_t j = 0; j < n_ctx; ++j) scores[j] -= mx;
                float sum = 0.0f;
                for (uint32_t j = 0; j < n_ctx; ++j) {
                    scores[j] = expf_poly(scores[j]);
                    sum += scores[j];
                }
                float inv = 1.0f / sum;
                for (uint32_t j = 0; j < n_ctx; ++j) scores[j] *= inv;
                float* oh = attn + h * hd;
                for (uint32_t i = 0; i < hd; ++i) oh[i] = 0.0f;
                for (uint32_t j = 0; j < n_ctx; ++j) {
                    const float* vj = kv->v[l] + (size_t)j * d + h * hd;
                    for (uint32_t i = 0; i < hd; ++i) oh[i] = fmaf(scores[j], vj[i], oh[i]);
                }
            }
            matvec(lm->wo[l], attn, proj, d, d);
            for (uint32_t i = 0; i < d; ++i) x[i] += proj[i];
            rmsnorm(x, xn, d);
            matvec(lm->w1[l], xn, hbuf, lm->ffn, d);
            for (uint32_t i = 0; i < lm->ffn; ++i) {
                float vv = hbuf[i];
                vv = vv > 9.0f ? 9.0f : (vv < -9.0f ? -9.0f : vv);
                float e = expf_poly(2.0f * vv);
                hbuf[i] = (e - 1.0f) / (e + 1.0f);
            }
            matvec(lm->w2[l], hbuf, proj, d, lm->ffn);
            for (uint32_t i = 0; i < d; ++i) x[i] += proj[i];
        }
        kv->ids[pos] = ids[t];
        kv->n = pos + 1;
        if (t + 1 == n_new || all_logits) {
            rmsnorm(x, xn, d);
            matvec(lm->head, xn, lg, VOCAB, d);
            if (all_logits) memcpy(all_logits + (size_t)t * VOCAB, lg, sizeof(lg));
            if (t + 1 == n_new && logits) memcpy(logits, lg, sizeof(lg));
        }
    }
    free(x); free(xn); free(qkv); free(attn); free(proj); free(hbuf); free(scores);
    return 0;
}

/* lm_core.cpp:163-173 embed_tokens + :299-327 prefill */
int sgo_lm_prefill(const sgo_lm* lm, sgo_kv* kv, const int32_t* tokens, uint32_t n,
                   const float* soft, float* logits, float* all_logits) {
    uint32_t total = n + (soft ? 1 : 0);
    if (total > lm->max_seq) return 2;
    if (total == 0) return 0;
    size_t d = lm->d;
    float* emb = (float*)malloc(total * d * sizeof(float));
    int32_t* ids = (int32_t*)malloc(total * sizeof(int32_t));
    uint32_t o = 0;
    if (soft) {
        memcpy(emb, soft, d * sizeof(float));
        ids[0] = 259;
        o = 1;
    }
    for (uint32_t t = 0; t < n; ++t) {
        if (tokens[t] < 0 || tokens[t] >= VOCAB) { free(emb); free(ids); return 1; }
        memcpy(emb + (size_t)(o + t) * d, lm->tok + (size_t)tokens[t] * d, d * sizeof(float));
        ids[o + t] = tokens[t];
    }
    kv->n = 0;
    int rc = forward(lm, kv, emb, ids, total, logits, all_logits);
    free(emb);
    free(ids);
    return rc;
}

/* lm_core.cpp:329-339 extend */
int sgo_lm_extend(const sgo_lm* lm, sgo_kv* kv, const int32_t* tokens, uint32_t n, float* logits,
                  float* all_logits) {
    if (n == 0) return 0;
    size_t d = lm->d;
    float* emb = (float*)malloc(n * d * sizeof(float));
    for (uint32_t t = 0; t < n; ++t) {
        if (tokens[t] < 0 || tokens[t] >= VOCAB) { free(emb); return 1; }
        memcpy(emb + (size_t)t * d, lm->tok + (size_t)tokens[t] * d, d * sizeof(float));
    }
    int rc = forward(lm, kv, emb, tokens, n, logits, all_logits);
    free(emb);
    return rc;
}

/* lm_core.cpp:39-50 */
int32_t sgo_greedy_argmax(const float* logits, uint32_t n, int32_t bias_target, float bonus) {
    int32_t best = 0;
    float best_val = logits[0] + (bias_target == 0 ? bonus : 0.0f);
    for (int32_t v = 1; v < (int32_t)n; ++v) {
        float val = logits[v] + (v == bias_target ? bonus : 0.0f);
        if (val > best_val) {
            best_val = val;
            best = v;
        }
    }
    return best;
}

/* lm_core.cpp:360-374 copy-pointer search */
int sgo_hint_found(const int32_t* ctx, uint32_t ctx_len, uint32_t limit, const int32_t* answer,
                   uint32_t ans_len) {
    if (ans_len == 0) return 0;
    if (limit > ctx_len) limit = ctx_len;
    if (ans_len > limit) return 0;
    for (uint32_t s = 0; s + ans_len <= limit; ++s) {
        uint32_t i = 0;
        while (i < ans_len && ctx[s + i] == answer[i]) ++i;
        if (i == ans_len) return 1;
    }
    return 0;
}
