// api.cu -- C ABI (include/sgc_b200.h) and the C++ host orchestration of the SubGCache hot
// path: graph ingest-side preparation, batched GNN encode, clustering, representative
// construction, batched representative prefill and batched cascade member extend.
//
// Reference call stack being replaced (paths under /root/reference/proj):
//   pipeline.cpp:212-293  run() SubgCache branch  -> sgc_run_subgcache
//   cache_engine.cpp:140-233 process_cluster / run_batch -> sgc_prefill + sgc_extend
//   lm_core.cpp:179-297 ToyLm::forward (token-sequential)  -> forward_rows (row-batched)
#include <algorithm>
#include <cstdlib>
#include <deque>
#include <set>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <unordered_map>

#include "attention.cuh"
#include "cluster_kernels.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "gnn_kernels.cuh"
#include "graph_kernels.cuh"
#include "lm_kernels.cuh"
#include "rng.cuh"

using sgc::Ctx;
using sgc::fail;
using bf16 = __nv_bfloat16;

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return SGC_OK;
    } catch (const sgc::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return SGC_CUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SGC_LOGIC;
    }
}

// every ABI entry that touches the device makes the context's device current first: a process
// may hold contexts on several GPUs and call them from any thread
Ctx* current(Ctx* c) {
    int cur = -1;
    SGC_CUDA_CHECK(cudaGetDevice(&cur));
    if (cur != c->device) SGC_CUDA_CHECK(cudaSetDevice(c->device));
    return c;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// SGC_TRACE_HOST=1: host wall-clock marks inside sgc_run_subgcache (stderr), to locate host stalls
void host_mark(const char* what, double t0) {
    static const bool on = std::getenv("SGC_TRACE_HOST") != nullptr;
    if (on) std::fprintf(stderr, "[sgc host] %-24s %9.3f ms\n", what, now_ms() - t0);
}

template <typename T>
T* dalloc(Ctx* c, size_t n) {
    void* p = nullptr;
    SGC_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), c->stream));
    return static_cast<T*>(p);
}
inline void dfree(Ctx* c, void* p) {
    if (p) cudaFreeAsync(p, c->stream);
}

// is `p` device (or managed) memory? host pointers are read directly -- no stream sync, so host
// preparation of the next wave never drains the GPU queue
inline bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// host copy of a possibly-device array
template <typename T>
std::vector<T> to_host(Ctx* c, const T* p, size_t n) {
    std::vector<T> v(n);
    if (!n) return v;
    if (!is_device_ptr(p)) {
        std::memcpy(v.data(), p, n * sizeof(T));
        return v;
    }
    SGC_CUDA_CHECK(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDefault, c->stream));
    SGC_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return v;
}

std::string csv_quote(const std::string& f) {  // graph_store.cpp:237-247
    if (f.find_first_of(",\"\n") == std::string::npos) return f;
    std::string out = "\"";
    for (char ch : f) {
        if (ch == '"') out += "\"\"";
        else out += ch;
    }
    return out + "\"";
}

// encoders.cpp:62-80 token hashing (host string work, once per graph)
void hash_tokens(const char* s, size_t n, uint64_t salt, std::vector<uint32_t>& b,
                 std::vector<int8_t>& sg) {
    uint64_t h = 0xcbf29ce484222325ULL;
    size_t len = 0;
    for (size_t i = 0; i <= n; ++i) {
        unsigned char ch = i < n ? static_cast<unsigned char>(s[i]) : 0;
        bool tok = i < n && ((ch >= '0' && ch <= '9') || (ch >= 'a' && ch <= 'z') ||
                             (ch >= 'A' && ch <= 'Z') || ch >= 0x80);
        if (tok) {
            if (ch >= 'A' && ch <= 'Z') ch = static_cast<unsigned char>(ch - 'A' + 'a');
            h ^= ch;
            h *= 0x100000001b3ULL;
            ++len;
            continue;
        }
        if (len) {
            uint64_t hh = sgc::splitmix64_once(h ^ salt);
            b.push_back(static_cast<uint32_t>(hh % 4096));
            sg.push_back(((hh >> 32) & 1) ? 1 : -1);
            h = 0xcbf29ce484222325ULL;
            len = 0;
        }
    }
}

const char kHeader[] = "Use the following graph to answer the question.\n\n";
const char kNodeHdr[] = "node id,node attr";
const char kEdgeHdr[] = "src,edge attr,dst";

}  // namespace

// ====================================================================== handles

// ---- paged bf16 KV cache --------------------------------------------------------------------
// One page pool per model: K and V are [L][pages][128][d] bf16 (layer-major, so one layer's pages
// form a [pages * 128 x d] matrix for the attention's TMA descriptors). A sealed prefix segment
// owns a list of pages (its block table); pages come from a free list and go back to it when the
// handle is released (KVCache::release_suffix / the shared prefix dropped, lm_core.hpp:35-92). The
// pool grows like a vector (new buffers, live pages copied, indices unchanged); new memory is
// zeroed once, so a page's unused tail rows always hold finite values (masked keys read 0 * V).
struct KvPool {
    bf16* k = nullptr;
    bf16* v = nullptr;
    uint32_t pages = 0;
    std::vector<int32_t> free_pages;  // sorted descending: pop_back hands out ascending ids
    uint32_t live() const { return pages - static_cast<uint32_t>(free_pages.size()); }
};

struct sgc_model {
    Ctx* c = nullptr;
    KvPool pool;
    sgc_lm_config cfg{};
    int d = 0, hd = 0, H = 0, L = 0, ffn = 0;
    float* tok_emb = nullptr;  // fp32 [260 x d]
    float* head = nullptr;     // fp32 [260 x d]
    float* head_t = nullptr;   // fp32 [d x 260]
    bf16* weights = nullptr;   // all layers, bf16
    std::vector<bf16*> wqkv, wo, w1, w2;
    float* rope_cos = nullptr;
    float* rope_sin = nullptr;
    uint64_t seed_states[6] = {};
};

struct sgc_graph {
    Ctx* c = nullptr;
    uint32_t n_nodes = 0, n_edges = 0;
    std::vector<uint32_t> ids;  // ascending
    std::vector<uint32_t> edge_src_idx, edge_dst_idx;  // dense node indices
    uint32_t* d_ids = nullptr;
    char* d_node_rows = nullptr;
    uint64_t* d_node_row_off = nullptr;
    uint32_t* d_node_row_len = nullptr;
    char* d_edge_rows = nullptr;
    uint64_t* d_edge_row_off = nullptr;
    uint32_t* d_edge_row_len = nullptr;
    // text hashes for nodes then edges, per salt
    uint64_t hash_salt = ~0ull;
    uint32_t* d_bucket = nullptr;
    int8_t* d_sign = nullptr;
    uint64_t* d_tok_off = nullptr;
    std::vector<std::string> texts;  // node texts then edge texts (for re-hashing)
};

struct sgc_kv {
    sgc_model* model = nullptr;
    uint32_t n = 0;
    std::vector<uint64_t> len;       // tokens per sealed segment
    std::vector<uint32_t> bt_off;    // segment s's pages: pages[bt_off[s] ..]
    std::vector<int32_t> pages;      // block table (host copy)
    int32_t* d_bt = nullptr;         // block table (device)
    uint64_t rows = 0;               // tokens of all segments
    int32_t* d_tokens = nullptr;     // context token ids (prefix, incl. soft slot), segments back to back
    uint64_t* d_tok_off = nullptr;
    int refs = 1;                    // the handle + live forks (the prefix outlives its forks' users)
    size_t layer_elems() const { return static_cast<size_t>(model->pool.pages) * sgc::kPageTokens * model->d; }
    bf16* k_layer(int l) const { return model->pool.k + l * layer_elems(); }
    bf16* v_layer(int l) const { return model->pool.v + l * layer_elems(); }
    int pool_rows() const { return static_cast<int>(model->pool.pages * sgc::kPageTokens); }
    uint32_t seg_pages(uint32_t s) const { return static_cast<uint32_t>((len[s] + sgc::kPageTokens - 1) / sgc::kPageTokens); }
};

namespace {

// ============================================================ KV page pool

size_t page_bytes(const sgc_model* m) {
    return static_cast<size_t>(m->L) * 2 * sgc::kPageTokens * m->d * sizeof(bf16);  // K + V, all layers
}

// grow the pool to at least `need` pages (x1.5 when memory allows): new zeroed buffers, live pages
// copied (page ids unchanged), old buffers freed in stream order
void pool_grow(Ctx* c, sgc_model* m, uint32_t need) {
    KvPool& p = m->pool;
    if (need <= p.pages) return;
    size_t free_b = 0, total_b = 0;
    c->mem_info(&free_b, &total_b);
    const size_t pb = page_bytes(m);
    const size_t headroom = std::max<size_t>(static_cast<size_t>(0.04 * total_b), 2ull << 30);
    size_t avail = free_b > headroom ? free_b - headroom : 0;  // new buffers coexist with the old
    if (p.pages && p.live() == 0) {
        // nothing to carry over: hand the old buffers back (stream order) before allocating, so a
        // pool sized for an earlier, smaller batch does not have to coexist with its replacement
        SGC_CUDA_CHECK(cudaFreeAsync(p.k, c->stream));
        SGC_CUDA_CHECK(cudaFreeAsync(p.v, c->stream));
        avail += static_cast<size_t>(p.pages) * pb;
        p.k = p.v = nullptr;
        p.pages = 0;
        p.free_pages.clear();
    }
    uint32_t want = std::max<uint32_t>(need, p.pages + p.pages / 2);
    if (static_cast<size_t>(want) * pb > avail) want = need;
    if (static_cast<size_t>(want) * pb > avail)
        fail(SGC_CAPACITY, "KV page pool: " + std::to_string(want) + " pages (" +
                               std::to_string((static_cast<size_t>(want) * pb) >> 20) +
                               " MiB) do not fit in free device memory");
    const size_t row_elems = static_cast<size_t>(sgc::kPageTokens) * m->d;
    static const bool trace = std::getenv("SGC_TRACE_POOL") != nullptr;
    if (trace) std::fprintf(stderr, "[sgc] KV pool grow: %u -> %u pages (need %u, %zu MiB per page)\n", p.pages, want, need, pb >> 20);
    bf16 *nk = nullptr, *nv = nullptr;
    const size_t bytes = static_cast<size_t>(want) * row_elems * m->L * sizeof(bf16);
    SGC_CUDA_CHECK(cudaMallocAsync(&nk, bytes, c->stream));
    SGC_CUDA_CHECK(cudaMallocAsync(&nv, bytes, c->stream));
    SGC_CUDA_CHECK(cudaMemsetAsync(nk, 0, bytes, c->stream));
    SGC_CUDA_CHECK(cudaMemsetAsync(nv, 0, bytes, c->stream));
    if (p.pages) {
        const size_t src_pitch = static_cast<size_t>(p.pages) * row_elems * sizeof(bf16);
        const size_t dst_pitch = static_cast<size_t>(want) * row_elems * sizeof(bf16);
        SGC_CUDA_CHECK(cudaMemcpy2DAsync(nk, dst_pitch, p.k, src_pitch, src_pitch, m->L, cudaMemcpyDeviceToDevice, c->stream));
        SGC_CUDA_CHECK(cudaMemcpy2DAsync(nv, dst_pitch, p.v, src_pitch, src_pitch, m->L, cudaMemcpyDeviceToDevice, c->stream));
        SGC_CUDA_CHECK(cudaFreeAsync(p.k, c->stream));
        SGC_CUDA_CHECK(cudaFreeAsync(p.v, c->stream));
    }
    for (uint32_t i = p.pages; i < want; ++i) p.free_pages.push_back(static_cast<int32_t>(i));
    std::sort(p.free_pages.begin(), p.free_pages.end(), std::greater<int32_t>());
    p.k = nk;
    p.v = nv;
    p.pages = want;
    c->mem_changed();
}

std::vector<int32_t> pool_alloc(Ctx* c, sgc_model* m, uint32_t n) {
    KvPool& p = m->pool;
    if (p.free_pages.size() < n) pool_grow(c, m, p.live() + n);
    std::vector<int32_t> out(p.free_pages.end() - n, p.free_pages.end());
    p.free_pages.resize(p.free_pages.size() - n);
    std::reverse(out.begin(), out.end());
    return out;
}

// pages return to the free list; stream order makes the reuse safe (one stream per context)
void pool_release(sgc_model* m, const std::vector<int32_t>& pages) {
    if (pages.empty()) return;
    KvPool& p = m->pool;
    p.free_pages.insert(p.free_pages.end(), pages.begin(), pages.end());
    std::sort(p.free_pages.begin(), p.free_pages.end(), std::greater<int32_t>());
}

// ============================================================ model weights

void check_lm_cfg(const sgc_lm_config& c) {
    if (c.model_dim == 0 || c.heads == 0 || c.layers == 0)
        fail(SGC_DOMAIN, "lm config needs layers, heads, dim >= 1");
    if (c.model_dim % c.heads) fail(SGC_DOMAIN, "model_dim must be divisible by heads");
    uint32_t hd = c.model_dim / c.heads;
    if (hd != 16 && hd != 32 && hd != 64 && hd != 128)
        fail(SGC_DOMAIN, "head_dim must be 16, 32, 64 or 128 on this backend");
    if (c.model_dim % 64 || c.ffn_hidden % 64)
        fail(SGC_DOMAIN, "model_dim and ffn_hidden must be multiples of 64 on this backend");
}

// ============================================================ row-batched forward

struct FwdBatch {
    int M = 0;
    const int32_t* d_tokens = nullptr;  // [M]
    const float* d_soft = nullptr;      // soft vectors
    const int32_t* d_soft_idx = nullptr;  // [M] row -> soft vector index or -1
    const int32_t* d_pos = nullptr;
    const int32_t* d_seg_lo = nullptr;
    const sgc::AttnWork* d_work = nullptr;  // tiles of <= attn_tile(hd) rows
    int n_work = 0;
    int pfx_rows = 0;  // rows of the prefix KV region (TMA bounds)
    int loc_rows = 0;  // rows of the k_loc / v_loc region (TMA bounds; 0 = M, contiguous batch rows)
    const int32_t* d_bt = nullptr;  // block table of the pages the work items reference
    // KV written by this batch: row r -> loc row r of (k_loc_layer(l), v_loc_layer(l))
    std::function<bf16*(int)> k_loc, v_loc;
    std::function<const bf16*(int)> k_pfx, v_pfx;
    const int32_t* d_logit_rows = nullptr;
    int n_logits = 0;
    float* d_logits = nullptr;
    // KV row written for batch row r (default r); decode writes generated tokens' K/V elsewhere
    const int32_t* d_kv_row = nullptr;
    // decode step (one row per generating member): prefix partial + own keys, see DecodeRows
    const struct DecodeRows* dec = nullptr;
};

// device arrays of one decode step (rows = active members): prefix segment, own question rows
// and own generated rows (lm_core.cpp:352-404 for a batch of forks)
struct DecodeRows {
    const int32_t *p_lo, *p_n, *q_lo, *q_n, *g_lo, *g_n;
    std::function<const bf16*(int)> k_q, v_q;  // persistent question K/V per layer
};

void forward_rows(Ctx* c, sgc_model* m, const FwdBatch& b) {
    const int M = b.M, d = m->d;
    if (M == 0) return;
    float* x = c->buf<float>("fwd_x", static_cast<size_t>(M) * d);
    bf16* xb = c->buf<bf16>("fwd_xb", static_cast<size_t>(M) * d);
    bf16* q = c->buf<bf16>("fwd_q", static_cast<size_t>(M) * d);
    bf16* ao = c->buf<bf16>("fwd_attn", static_cast<size_t>(M) * d);
    bf16* h = c->buf<bf16>("fwd_h", static_cast<size_t>(M) * m->ffn);
    int* bad = c->buf<int>("fwd_bad", 1);
    const int32_t* kv_row = b.d_kv_row;
    if (!kv_row) kv_row = c->iota(M);
    float* part_o = nullptr;
    float* part_lse = nullptr;
    if (b.dec && sgc::attention_tc_supported(m->hd)) {
        part_o = c->buf<float>("dec_part_o", static_cast<size_t>(M) * d);
        part_lse = c->buf<float>("dec_part_lse", static_cast<size_t>(M) * m->H);
    }
    SGC_CUDA_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    // RMSNorm is fused: every residual GEMM (and the embedding) writes bf16(x) and the row sums
    // of squares; the next GEMM scales its accumulator rows (gemm.cuh GemmEpi::in_ss)
    // row sums of squares as d/32 chunk slots per row (written, never accumulated: deterministic)
    const int parts = d / 32;
    float* ss_a = c->buf<float>("fwd_ss_a", static_cast<size_t>(M) * parts);  // -> QKV
    float* ss_b = c->buf<float>("fwd_ss_b", static_cast<size_t>(M) * parts);  // -> W1
    float* rs = c->buf<float>("fwd_rscale", M);                                // finalized scales
    sgc::embed(c, x, b.d_tokens, m->tok_emb, b.d_soft, b.d_soft_idx, d, M, bad, xb, ss_a);
    for (int l = 0; l < m->L; ++l) {
        sgc::GemmEpi e;
        if (b.dec) {  // decode step: the GEMM epilogue finalizes the row scales (no rms_scale launch)
            e.ss_parts = ss_a;
            e.ss_n = l == 0 ? 1 : parts;  // the embedding writes one slot per row
            e.ss_d = d;
        } else {
            sgc::rms_scale(c, rs, ss_a, M, l == 0 ? 1 : parts, d);  // the embedding writes one slot per row
            e.row_scale = rs;
        }
        e.mode = sgc::EPI_QKV;
        e.q_out = q;
        e.k_cache = b.k_loc(l);
        e.v_cache = b.v_loc(l);
        e.kv_row = kv_row;
        e.pos = b.d_pos;
        e.rope_cos = m->rope_cos;
        e.rope_sin = m->rope_sin;
        e.d = d;
        e.hd = m->hd;
        e.splitk_ok = b.dec != nullptr;  // decode step: stream-K / split-K allowed
        sgc::gemm_bf16(c, xb, m->wqkv[l], M, 3 * d, d, e);
        // last layer: K/V of every row are written now; the rest of the layer only feeds the
        // head, so rows without logits skip it (values nothing reads: a prefill without logits
        // stops here, an extend finishes only its members' last rows; decode rows all need logits)
        const bool last = l == m->L - 1;
        if (last && !b.dec && b.n_logits == 0) break;

        sgc::AttnParams ap;
        ap.q = q;
        ap.out = ao;
        ap.k_pfx = b.k_pfx ? b.k_pfx(l) : b.k_loc(l);
        ap.v_pfx = b.v_pfx ? b.v_pfx(l) : b.v_loc(l);
        ap.k_loc = b.k_loc(l);
        ap.v_loc = b.v_loc(l);
        ap.loc_kv0 = 0;
        ap.seg_lo = b.d_seg_lo;
        ap.work = b.d_work;
        ap.bt = b.d_bt;
        ap.d = d;
        ap.scale = 1.0f / std::sqrt(static_cast<float>(m->hd));
        if (b.dec) {
            // decode: prefix partial on the tensor cores (units of one prefix segment), then each
            // row's own question + generated keys and the merge
            sgc::DecodeAttnParams dp;
            dp.q = q;
            dp.k_p = ap.k_pfx;
            dp.v_p = ap.v_pfx;
            dp.k_q = b.dec->k_q(l);
            dp.v_q = b.dec->v_q(l);
            dp.k_g = b.k_loc(l);
            dp.v_g = b.v_loc(l);
            dp.p_lo = b.dec->p_lo;
            dp.p_n = b.dec->p_n;
            dp.q_lo = b.dec->q_lo;
            dp.q_n = b.dec->q_n;
            dp.g_lo = b.dec->g_lo;
            dp.g_n = b.dec->g_n;
            dp.p_bt = b.d_bt;
            dp.out = ao;
            dp.rows = M;
            dp.d = d;
            dp.heads = m->H;
            dp.scale = ap.scale;
            if (part_o) {
                ap.part_o = part_o;
                ap.part_lse = part_lse;
                ap.k_loc = ap.k_pfx;
                ap.v_loc = ap.v_pfx;
                sgc::cascade_attention_tc(c, ap, b.n_work, m->H, m->hd, M, b.pfx_rows, b.pfx_rows);
                dp.part_o = part_o;
                dp.part_lse = part_lse;
            } else {
                dp.part_o = nullptr;
                dp.part_lse = nullptr;
            }
            sgc::decode_attention_local(c, dp);
        } else if (sgc::attention_tc_supported(m->hd)) {
            const int loc_rows = b.loc_rows ? b.loc_rows : M;
            sgc::cascade_attention_tc(c, ap, b.n_work, m->H, m->hd, M, b.k_pfx ? b.pfx_rows : loc_rows, loc_rows);
        } else {
            sgc::cascade_attention(c, ap, b.n_work, m->H, m->hd);
        }

        sgc::GemmEpi r;
        r.mode = sgc::EPI_RESID;
        r.out = x;
        r.ldo = d;
        r.out_xb = xb;
        r.out_ss = ss_b;
        r.splitk_ok = b.dec != nullptr;
        if (last && !b.dec && b.n_logits < M) {
            // the rows the head reads, compacted (per-row GEMM results are independent of M)
            const int n = b.n_logits;
            float* cx = c->buf<float>("fwd_cx", static_cast<size_t>(n) * d);
            bf16* cao = c->buf<bf16>("fwd_cao", static_cast<size_t>(n) * d);
            bf16* cxb = c->buf<bf16>("fwd_cxb", static_cast<size_t>(n) * d);
            bf16* ch = c->buf<bf16>("fwd_ch", static_cast<size_t>(n) * m->ffn);
            float* css = c->buf<float>("fwd_css", static_cast<size_t>(n) * parts);
            float* crs = c->buf<float>("fwd_crs", n);
            sgc::gather_rows(c, cx, x, b.d_logit_rows, n, static_cast<size_t>(d) * sizeof(float));
            sgc::gather_rows(c, cao, ao, b.d_logit_rows, n, static_cast<size_t>(d) * sizeof(bf16));
            r.out = cx;
            r.out_xb = cxb;
            r.out_ss = css;
            sgc::gemm_bf16(c, cao, m->wo[l], n, d, d, r);
            sgc::GemmEpi t;
            t.mode = sgc::EPI_TANH;
            t.out = ch;
            t.ldo = m->ffn;
            sgc::rms_scale(c, crs, css, n, parts, d);
            t.row_scale = crs;
            sgc::gemm_bf16(c, cxb, m->w1[l], n, m->ffn, d, t);
            r.out_xb = nullptr;  // no next layer
            r.out_ss = nullptr;
            sgc::gemm_bf16(c, ch, m->w2[l], n, d, m->ffn, r);
            sgc::head_logits(c, b.d_logits, cx, c->iota(n), n, m->head_t, d);
            c->flag_readback(bad);
            return;
        }
        sgc::gemm_bf16(c, ao, m->wo[l], M, d, d, r);

        sgc::GemmEpi t;
        t.mode = sgc::EPI_TANH;
        t.out = h;
        t.ldo = m->ffn;
        if (b.dec) {
            t.ss_parts = ss_b;
            t.ss_n = parts;
            t.ss_d = d;
        } else {
            sgc::rms_scale(c, rs, ss_b, M, parts, d);
            t.row_scale = rs;
        }
        t.splitk_ok = b.dec != nullptr;
        sgc::gemm_bf16(c, xb, m->w1[l], M, m->ffn, d, t);
        r.out_ss = last ? nullptr : ss_a;  // the next layer's QKV input
        if (last) r.out_xb = nullptr;
        sgc::gemm_bf16(c, h, m->w2[l], M, d, m->ffn, r);
    }
    sgc::head_logits(c, b.d_logits, x, b.d_logit_rows, b.n_logits, m->head_t, d);
    // the out-of-vocab flag lands in pinned host memory; callers check it after their own sync
    c->flag_readback(bad);
}

// after the caller's stream sync: fail if any forward since the last check saw a bad token id
void check_forward_flags(Ctx* c) {
    if (c->take_flag()) fail(SGC_DOMAIN, "token id out of vocab");
}

// tiles of <= attn_tile rows that never cross a `group` boundary (sequence for prefill, segment
// for extend); rows of one group are contiguous. loc_bt: per group, the block-table offset of the
// group's own pages (paged prefill) or -1 (own keys in contiguous scratch rows)
int attn_tile(int hd) { return sgc::attention_tc_supported(hd) ? 256 : 64; }

std::vector<sgc::AttnWork> make_work(const std::vector<int>& group_start, const std::vector<int>& group_rows,
                                     const std::vector<int>& pfx_off, const std::vector<int>& pfx_len,
                                     const std::vector<int>& loc_bt, int tile) {
    std::vector<sgc::AttnWork> w;
    for (size_t g = 0; g < group_start.size(); ++g)
        for (int r = 0; r < group_rows[g]; r += tile)
            w.push_back({group_start[g] + r, std::min(tile, group_rows[g] - r), pfx_off[g], pfx_len[g], loc_bt[g]});
    return w;
}

// ============================================================ prefill / extend

// ToyLm::prefill + KVCache::seal (lm_core.cpp:299-327, :60-80) for `count` sequences in one
// handle. Every sequence gets its own 128-token pages from the model's pool (its block table);
// the forward runs over chunks of whole sequences (<= max_rows rows: bounded activations), the QKV
// GEMM epilogue writes each row's K/V straight into its page slot, and the attention reads each
// sequence's own keys through its pages.
// n_remote: the last n_remote sequences get pages and context tokens but are not computed -- their
// sealed K/V arrive point to point from the rank that prefilled them (last_logits: local ones).
sgc_kv* do_prefill(Ctx* c, sgc_model* m, uint32_t count, const uint64_t* off_in, const int32_t* tok_in,
                   const float* soft, const uint8_t* soft_mask, float* last_logits, bool sync = true,
                   uint32_t n_remote = 0, uint64_t max_rows = 1ull << 16) {
    std::vector<uint64_t> off = to_host(c, off_in, count + 1);
    std::vector<int32_t> toks = to_host(c, tok_in, off[count]);
    std::vector<uint8_t> smask = soft_mask ? to_host(c, soft_mask, count) : std::vector<uint8_t>(count, 0);
    const int d = m->d;
    if (n_remote > count) fail(SGC_LOGIC, "prefill: more remote sequences than sequences");
    auto kv = std::make_unique<sgc_kv>();
    kv->model = m;
    kv->n = count;
    std::vector<int32_t> rows_tok, soft_idx;
    std::vector<uint64_t> ctx_off(1, 0), seq_row0;
    bool any_soft = false;
    for (uint32_t s = 0; s < count; ++s) {
        uint64_t n = off[s + 1] - off[s];
        bool has_soft = smask[s] != 0;
        any_soft |= has_soft;
        uint64_t total = n + (has_soft ? 1 : 0);
        if (total > m->cfg.max_seq_len)
            fail(SGC_CAPACITY, "prompt of " + std::to_string(total) + " tokens exceeds max " +
                                   std::to_string(m->cfg.max_seq_len));
        if (total == 0) fail(SGC_DOMAIN, "prefill: empty sequence");
        seq_row0.push_back(rows_tok.size());
        kv->len.push_back(total);
        if (has_soft) {
            rows_tok.push_back(259);
            soft_idx.push_back(static_cast<int32_t>(s));
        }
        for (uint64_t i = 0; i < n; ++i) {
            rows_tok.push_back(toks[off[s] + i]);
            soft_idx.push_back(-1);
        }
        ctx_off.push_back(rows_tok.size());
    }
    const uint64_t M = rows_tok.size();
    kv->rows = M;
    // pages: one block table for the handle, segment s at bt_off[s]
    uint32_t npages = 0;
    for (uint32_t s = 0; s < count; ++s) {
        kv->bt_off.push_back(npages);
        npages += kv->seg_pages(s);
    }
    kv->pages = pool_alloc(c, m, npages);
    kv->d_bt = dalloc<int32_t>(c, npages);
    sgc::copy_in_staged(c, kv->d_bt, kv->pages.data(), npages);
    kv->d_tokens = dalloc<int32_t>(c, M);
    kv->d_tok_off = dalloc<uint64_t>(c, count + 1);
    sgc::copy_in_staged(c, kv->d_tokens, rows_tok.data(), M);
    sgc::copy_in_staged(c, kv->d_tok_off, ctx_off.data(), count + 1);
    float* d_soft = nullptr;
    if (any_soft) {
        d_soft = c->buf<float>("pf_soft", static_cast<size_t>(count) * d);
        sgc::copy_in(c, d_soft, soft, static_cast<size_t>(count) * d);
    }
    const uint32_t n_local = count - n_remote;
    float* d_logits = c->buf<float>("pf_logits", static_cast<size_t>(std::max<uint32_t>(1, n_local)) * SGC_VOCAB);
    sgc_kv* kvp = kv.get();
    // the forward, one chunk of whole local sequences at a time
    for (uint32_t s0 = 0; s0 < n_local;) {
        uint32_t s1 = s0 + 1;
        uint64_t rows = kv->len[s0];
        while (s1 < n_local && rows + kv->len[s1] <= max_rows) rows += kv->len[s1++];
        const uint64_t R0 = seq_row0[s0];
        std::vector<int32_t> pos, seg_lo, sidx, kvrow, lrows;
        std::vector<int> gs, gr, z, lb;
        for (uint32_t s = s0; s < s1; ++s) {
            const int start = static_cast<int>(seq_row0[s] - R0);
            gs.push_back(start);
            gr.push_back(static_cast<int>(kv->len[s]));
            z.push_back(0);
            lb.push_back(static_cast<int>(kv->bt_off[s]));
            for (uint64_t t = 0; t < kv->len[s]; ++t) {
                pos.push_back(static_cast<int32_t>(t));
                seg_lo.push_back(start);
                sidx.push_back(soft_idx[seq_row0[s] + t]);
                kvrow.push_back(kv->pages[kv->bt_off[s] + t / sgc::kPageTokens] * sgc::kPageTokens +
                                static_cast<int32_t>(t % sgc::kPageTokens));
            }
            lrows.push_back(static_cast<int32_t>(start + kv->len[s] - 1));
        }
        std::vector<sgc::AttnWork> work = make_work(gs, gr, z, z, lb, attn_tile(m->hd));
        const int Mc = static_cast<int>(rows);
        int32_t* d_arr = c->buf<int32_t>("pf_rows", static_cast<size_t>(Mc) * 4 + (s1 - s0));
        std::vector<int32_t> packed;
        packed.reserve(static_cast<size_t>(Mc) * 4 + (s1 - s0));
        for (auto* v : {&pos, &seg_lo, &sidx, &kvrow, &lrows}) packed.insert(packed.end(), v->begin(), v->end());
        sgc::copy_in_staged(c, d_arr, packed.data(), packed.size());
        sgc::AttnWork* d_work = c->buf<sgc::AttnWork>("pf_work", work.size());
        sgc::copy_in_staged(c, d_work, work.data(), work.size());
        FwdBatch b;
        b.M = Mc;
        b.d_tokens = kv->d_tokens + R0;
        b.d_soft = d_soft;
        b.d_soft_idx = any_soft ? d_arr + 2 * static_cast<size_t>(Mc) : nullptr;
        b.d_pos = d_arr;
        b.d_seg_lo = d_arr + Mc;
        b.d_kv_row = d_arr + 3 * static_cast<size_t>(Mc);
        b.d_work = d_work;
        b.n_work = static_cast<int>(work.size());
        b.k_loc = [kvp](int l) { return kvp->k_layer(l); };
        b.v_loc = [kvp](int l) { return kvp->v_layer(l); };
        b.loc_rows = kv->pool_rows();
        b.d_bt = kv->d_bt;
        b.d_logit_rows = d_arr + 4 * static_cast<size_t>(Mc);
        // no logits requested (a representative's prompt): the last layer stops after its K/V
        b.n_logits = last_logits ? static_cast<int>(s1 - s0) : 0;
        b.d_logits = last_logits ? d_logits + static_cast<size_t>(s0) * SGC_VOCAB : nullptr;
        forward_rows(c, m, b);
        s0 = s1;
    }
    if (last_logits && n_local) sgc::copy_out(c, last_logits, d_logits, static_cast<size_t>(n_local) * SGC_VOCAB);
    if (sync) {  // else: the caller syncs (last_logits must then be pinned or null)
        c->sync();
        check_forward_flags(c);
    }
    return kv.release();
}

// Optional output of do_extend for a following decode: the members' question K/V kept for all
// layers (instead of a per-layer scratch) and the copy-pointer decision per member.
struct ExtendKeep {
    bf16* k = nullptr;  // [L][rows][d]; preset by the caller to share one buffer across calls
    bf16* v = nullptr;
    uint64_t rows = 0;  // rows per layer of the buffer
    uint64_t base = 0;  // first row used by this call
    std::vector<int32_t> q_lo;  // per member (input order): first question row (absolute)
    std::vector<int8_t> hint;   // per member: answer found in the prefix (lm_core.cpp:361-374)
};

// Deferred outputs of do_extend: logits / first tokens in the extend's row order (members
// stably sorted by segment) land in PINNED host memory with no stream sync; `order` maps that
// order back to member indices. The caller syncs once (e.g. at the end of the batch).
struct ExtendDefer {
    float* logits = nullptr;   // pinned [n * 260] or null
    int32_t* first = nullptr;  // pinned [n]
    std::vector<uint32_t> order;
};

// members: segment, question tokens, answers; returns logits/first token in member order
void do_extend(Ctx* c, sgc_model* m, sgc_kv* kv, uint32_t n, const uint32_t* seg_in,
               const uint64_t* q_off_in, const int32_t* q_in, const uint64_t* a_off_in,
               const int32_t* a_in, float bonus, float* logits_out, int32_t* first_out,
               ExtendKeep* keep = nullptr, ExtendDefer* defer = nullptr, uint64_t max_rows = 1ull << 16) {
    if (n == 0) return;
    const int d = m->d;
    std::vector<uint32_t> seg = to_host(c, seg_in, n);
    std::vector<uint64_t> qo = to_host(c, q_off_in, n + 1);
    std::vector<int32_t> qt = to_host(c, q_in, qo[n]);
    std::vector<uint64_t> ao;
    std::vector<int32_t> at;
    if (a_off_in) {
        ao = to_host(c, a_off_in, n + 1);
        at = to_host(c, a_in, ao[n]);
    }
    for (uint32_t j = 0; j < n; ++j) {
        if (seg[j] >= kv->n) fail(SGC_DOMAIN, "extend: member references an unknown segment");
        uint64_t qn = qo[j + 1] - qo[j];
        if (qn == 0) fail(SGC_DOMAIN, "extend: empty question (KVCache::extend with zero tokens is a no-op)");
        if (kv->len[seg[j]] + qn > m->cfg.max_seq_len)
            fail(SGC_CAPACITY, "sequence length " + std::to_string(kv->len[seg[j]] + qn) + " exceeds max " +
                                   std::to_string(m->cfg.max_seq_len));
    }
    // members grouped by segment (stable), processed in row chunks
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return seg[a] < seg[b]; });
    std::vector<int32_t> first_h(first_out ? n : 0);
    std::vector<float> logits_h(logits_out ? static_cast<size_t>(n) * SGC_VOCAB : 0);
    if (keep) {
        if (!keep->k) {
            keep->rows = qo[n];
            keep->base = 0;
            keep->k = c->buf<bf16>("ex_keep_k", static_cast<size_t>(m->L) * keep->rows * d);
            keep->v = c->buf<bf16>("ex_keep_v", static_cast<size_t>(m->L) * keep->rows * d);
        } else if (keep->base + qo[n] > keep->rows) {
            fail(SGC_LOGIC, "question KV buffer overflow");
        }
        keep->q_lo.assign(n, 0);
        keep->hint.assign(n, 0);
    }
    uint64_t chunk0 = keep ? keep->base : 0;  // first kept row of the chunk
    size_t i0 = 0;
    while (i0 < n) {
        // chunk [i0, i1) with <= max_rows rows
        size_t i1 = i0;
        uint64_t rows = 0;
        while (i1 < n) {
            uint64_t qn = qo[order[i1] + 1] - qo[order[i1]];
            if (i1 > i0 && rows + qn > max_rows) break;
            rows += qn;
            ++i1;
        }
        const int M = static_cast<int>(rows);
        std::vector<int32_t> toks, pos, seg_lo, lrows;
        std::vector<int> gs, gr, pk, pl, lb;
        std::vector<uint32_t> mseg;
        std::vector<uint64_t> a_off(1, 0);
        std::vector<int32_t> a_tok;
        for (size_t ii = i0; ii < i1; ++ii) {
            uint32_t j = order[ii];
            uint32_t s = seg[j];
            int start = static_cast<int>(toks.size());
            uint64_t qn = qo[j + 1] - qo[j];
            if (gs.empty() || mseg.back() != s) {
                gs.push_back(start);
                gr.push_back(0);
                pk.push_back(static_cast<int>(kv->bt_off[s]));  // the sealed prefix's pages
                pl.push_back(static_cast<int>(kv->len[s]));
                lb.push_back(-1);                                // own keys: contiguous scratch
            }
            gr.back() += static_cast<int>(qn);
            mseg.push_back(s);
            for (uint64_t t = 0; t < qn; ++t) {
                toks.push_back(qt[qo[j] + t]);
                pos.push_back(static_cast<int32_t>(kv->len[s] + t));
                seg_lo.push_back(start);
            }
            lrows.push_back(static_cast<int32_t>(toks.size() - 1));
            if (keep) keep->q_lo[j] = static_cast<int32_t>(chunk0 + start);
            if (!ao.empty()) {
                for (uint64_t t = ao[j]; t < ao[j + 1]; ++t) a_tok.push_back(at[t]);
            }
            a_off.push_back(a_tok.size());
        }
        std::vector<sgc::AttnWork> work = make_work(gs, gr, pk, pl, lb, attn_tile(m->hd));
        const int nm = static_cast<int>(i1 - i0);
        int32_t* d_tok = c->buf<int32_t>("ex_tok", M);
        int32_t* d_pos = c->buf<int32_t>("ex_pos", M);
        int32_t* d_seg = c->buf<int32_t>("ex_seg", M);
        int32_t* d_lr = c->buf<int32_t>("ex_lrows", nm);
        uint32_t* d_mseg = c->buf<uint32_t>("ex_mseg", nm);
        uint64_t* d_aoff = c->buf<uint64_t>("ex_aoff", nm + 1);
        int32_t* d_atok = c->buf<int32_t>("ex_atok", a_tok.size());
        sgc::AttnWork* d_work = c->buf<sgc::AttnWork>("ex_work", work.size());
        float* d_logits = c->buf<float>("ex_logits", static_cast<size_t>(nm) * SGC_VOCAB);
        int32_t* d_first = c->buf<int32_t>("ex_first", nm);
        int8_t* d_hint = keep ? c->buf<int8_t>("ex_hint", nm) : nullptr;
        sgc::copy_in_staged(c, d_tok, toks.data(), M);
        sgc::copy_in_staged(c, d_pos, pos.data(), M);
        sgc::copy_in_staged(c, d_seg, seg_lo.data(), M);
        sgc::copy_in_staged(c, d_lr, lrows.data(), nm);
        sgc::copy_in_staged(c, d_mseg, mseg.data(), nm);
        sgc::copy_in_staged(c, d_aoff, a_off.data(), nm + 1);
        sgc::copy_in_staged(c, d_atok, a_tok.data(), a_tok.size());
        sgc::copy_in_staged(c, d_work, work.data(), work.size());
        FwdBatch b;
        b.M = M;
        b.d_tokens = d_tok;
        b.d_pos = d_pos;
        b.d_seg_lo = d_seg;
        b.d_work = d_work;
        b.n_work = static_cast<int>(work.size());
        if (keep) {  // question K/V of every layer kept for the decode steps
            const size_t lstride = static_cast<size_t>(keep->rows) * d, off = chunk0 * d;
            bf16 *kk = keep->k, *vv = keep->v;
            b.k_loc = [kk, lstride, off](int l) { return kk + l * lstride + off; };
            b.v_loc = [vv, lstride, off](int l) { return vv + l * lstride + off; };
        } else {  // one layer at a time
            bf16* kl = c->buf<bf16>("ex_kloc", static_cast<size_t>(M) * d);
            bf16* vl = c->buf<bf16>("ex_vloc", static_cast<size_t>(M) * d);
            b.k_loc = [kl](int) { return kl; };
            b.v_loc = [vl](int) { return vl; };
        }
        b.k_pfx = [kv](int l) { return static_cast<const bf16*>(kv->k_layer(l)); };
        b.pfx_rows = kv->pool_rows();
        b.v_pfx = [kv](int l) { return static_cast<const bf16*>(kv->v_layer(l)); };
        b.d_bt = kv->d_bt;
        b.d_logit_rows = d_lr;
        b.n_logits = nm;
        b.d_logits = d_logits;
        forward_rows(c, m, b);
        sgc::first_tokens(c, d_first, d_logits, nm, kv->d_tokens, kv->d_tok_off, d_mseg, d_atok,
                          a_tok.empty() ? nullptr : d_aoff, bonus, d_hint);
        // scatter back to member order
        if (defer) {  // no sync: results stay in extend order, copied to pinned host memory
            if (defer->logits) sgc::copy_out(c, defer->logits + i0 * SGC_VOCAB, d_logits, static_cast<size_t>(nm) * SGC_VOCAB);
            if (defer->first) sgc::copy_out(c, defer->first + i0, d_first, nm);
            chunk0 += static_cast<uint64_t>(M);
            i0 = i1;
            continue;
        }
        std::vector<float> lg(logits_out ? static_cast<size_t>(nm) * SGC_VOCAB : 0);
        std::vector<int32_t> ft(nm);
        std::vector<int8_t> hn(keep ? nm : 0);
        sgc::copy_out(c, lg.data(), d_logits, lg.size());
        sgc::copy_out(c, ft.data(), d_first, ft.size());
        if (keep) sgc::copy_out(c, hn.data(), d_hint, hn.size());
        c->sync();
        check_forward_flags(c);
        // scatter back to member order (outputs may be host or device memory)
        for (int k = 0; k < nm; ++k) {
            const uint32_t j = order[i0 + k];
            if (keep) keep->hint[j] = hn[k];
            if (first_out) first_h[j] = ft[k];
            if (logits_out)
                std::memcpy(logits_h.data() + static_cast<size_t>(j) * SGC_VOCAB,
                            lg.data() + static_cast<size_t>(k) * SGC_VOCAB, SGC_VOCAB * sizeof(float));
        }
        chunk0 += static_cast<uint64_t>(M);
        i0 = i1;
    }
    if (defer) {
        defer->order = order;
        return;
    }
    if (first_out) sgc::copy_in(c, first_out, first_h.data(), n);
    if (logits_out) sgc::copy_in(c, logits_out, logits_h.data(), logits_h.size());
    c->sync();
}

// ============================================================ batched greedy decode
// ToyLm::greedy_decode (lm_core.cpp:352-404) for a batch of forks, one row per still-generating
// member per step. Member j: prefix segment [pfx_kv0, +pfx_len) of the wave's sealed KV,
// own question rows [q_lo, +q_n) of the kept question K/V, generated rows [j*max_new, +t) of
// the decode K/V; token t is fed back at position pos0 + t (pos0 = context tokens after the
// extend). Stops per member on EOS, after max_new tokens, or when the context is full; the
// copy pointer biases answer[t] (then EOS) when the answer occurs in the prefix.
struct GenJob {
    std::vector<int32_t> pfx_bt, pfx_len, q_lo, q_n, pos0, first, gen_row0;  // pfx_bt: block-table offset
    std::vector<int8_t> hint;
    std::vector<uint64_t> a_off{0};
    std::vector<int32_t> a_tok;
    uint32_t size() const { return static_cast<uint32_t>(first.size()); }
};
// progress of every member of a GenJob (resumable: a wave may defer its stragglers)
struct GenState {
    uint32_t max_new = 1;
    std::vector<int32_t> tokens;  // [n * max_new], -1 padded
    std::vector<uint32_t> count;  // tokens so far
    std::vector<uint8_t> done;
    std::vector<int32_t> last_ev;  // event index of the member's last token (-1: the first token)
    std::vector<cudaEvent_t> events;  // one per decode step
    uint64_t rows = 0;
    void init(const GenJob& job, uint32_t mx, uint64_t max_seq) {
        const uint32_t n = job.size();
        max_new = std::max<uint32_t>(1, mx);
        tokens.assign(static_cast<size_t>(n) * max_new, -1);
        count.assign(n, 1);
        done.assign(n, 0);
        last_ev.assign(n, -1);
        for (uint32_t j = 0; j < n; ++j) {
            tokens[static_cast<size_t>(j) * max_new] = job.first[j];
            done[j] = max_new <= 1 || job.first[j] == SGC_EOS || static_cast<uint64_t>(job.pos0[j]) + 1 > max_seq;
        }
    }
};
// Decode buffers shared by every step of a batch: the block table of every sealed prefix the job's
// pfx_bt offsets index (pages of the model's pool), the kept question K/V and the generated-token
// K/V, each [L][rows][d].
struct GenBuffers {
    sgc_model* model = nullptr;
    int32_t* d_bt = nullptr;
    const ExtendKeep* keep = nullptr;
    bf16 *gk = nullptr, *gv = nullptr;
    size_t grows = 0;
    int8_t* d_hint = nullptr;
    uint64_t* d_aoff = nullptr;
    int32_t* d_atok = nullptr;
};

GenBuffers gen_buffers(Ctx* c, sgc_model* m, const std::vector<int32_t>& block_table, const ExtendKeep* keep,
                       const GenJob& job, size_t gen_rows) {
    GenBuffers g;
    g.model = m;
    g.d_bt = c->buf<int32_t>("dec_bt", std::max<size_t>(1, block_table.size()));
    sgc::copy_in_staged(c, g.d_bt, block_table.data(), block_table.size());
    g.keep = keep;
    g.grows = std::max<size_t>(1, gen_rows);
    g.gk = c->buf<bf16>("dec_gk", static_cast<size_t>(m->L) * g.grows * m->d);
    g.gv = c->buf<bf16>("dec_gv", static_cast<size_t>(m->L) * g.grows * m->d);
    const uint32_t n = job.size();
    g.d_hint = c->buf<int8_t>("dec_hint", n);
    g.d_aoff = c->buf<uint64_t>("dec_aoff", n + 1);
    g.d_atok = c->buf<int32_t>("dec_atok", std::max<size_t>(1, job.a_tok.size()));
    sgc::copy_in_staged(c, g.d_hint, job.hint.data(), n);
    sgc::copy_in_staged(c, g.d_aoff, job.a_off.data(), n + 1);
    sgc::copy_in_staged(c, g.d_atok, job.a_tok.data(), job.a_tok.size());
    return g;
}

// Runs decode steps for members `sel` of the job until all are done, or until fewer than
// `min_active` of them are still generating (the rest stay pending in `st`).
void decode_steps(Ctx* c, sgc_model* m, const GenBuffers& g, const GenJob& job, GenState& st,
                  const std::vector<uint32_t>& sel, uint32_t min_active, float bonus) {
    const int d = m->d;
    const uint32_t max_new = st.max_new;
    const uint64_t max_seq = m->cfg.max_seq_len;
    const int tile = attn_tile(m->hd);
    for (;;) {
        std::vector<int32_t> act;
        for (uint32_t j : sel)
            if (!st.done[j]) act.push_back(static_cast<int32_t>(j));
        if (act.empty() || act.size() < min_active) break;
        const int M = static_cast<int>(act.size());
        // rows follow `sel` order == grouped by prefix segment
        std::vector<int32_t> tok(M), pos(M), kvr(M), step(M), lrow(M);
        std::vector<int32_t> plo(M), pn(M), qlo(M), qn(M), glo(M), gn(M);
        std::vector<sgc::AttnWork> work;
        for (int i = 0; i < M; ++i) {
            const int32_t j = act[i];
            const int32_t t = static_cast<int32_t>(st.count[j]);  // index of the token produced now
            tok[i] = st.tokens[static_cast<size_t>(j) * max_new + t - 1];
            pos[i] = job.pos0[j] + t - 1;
            kvr[i] = job.gen_row0[j] + t - 1;
            step[i] = t;
            lrow[i] = i;
            plo[i] = job.pfx_bt[j];
            pn[i] = job.pfx_len[j];
            qlo[i] = job.q_lo[j];
            qn[i] = job.q_n[j];
            glo[i] = job.gen_row0[j];
            gn[i] = t;
            if (work.empty() || work.back().pfx_off != plo[i] || work.back().nrows == tile)
                work.push_back({i, 0, plo[i], pn[i], -1});
            work.back().nrows++;
        }
        int32_t* d_arr = c->buf<int32_t>("dec_rows", static_cast<size_t>(M) * 12);
        std::vector<int32_t> packed;
        packed.reserve(static_cast<size_t>(M) * 12);
        for (auto* v : {&tok, &pos, &kvr, &step, &lrow, &plo, &pn, &qlo, &qn, &glo, &gn, &act})
            packed.insert(packed.end(), v->begin(), v->end());
        sgc::copy_in_staged(c, d_arr, packed.data(), packed.size());
        auto col = [&](int k) { return d_arr + static_cast<size_t>(k) * M; };
        sgc::AttnWork* d_work = c->buf<sgc::AttnWork>("dec_work", work.size());
        sgc::copy_in_staged(c, d_work, work.data(), work.size());
        float* d_logits = c->buf<float>("dec_logits", static_cast<size_t>(M) * SGC_VOCAB);
        int32_t* d_tok_out = c->buf<int32_t>("dec_tok", M);
        DecodeRows dr;
        dr.p_lo = col(5);
        dr.p_n = col(6);
        dr.q_lo = col(7);
        dr.q_n = col(8);
        dr.g_lo = col(9);
        dr.g_n = col(10);
        {
            const size_t ls = static_cast<size_t>(g.keep ? g.keep->rows : 0) * d;
            const bf16* qk = g.keep ? g.keep->k : nullptr;
            const bf16* qv = g.keep ? g.keep->v : nullptr;
            dr.k_q = [qk, ls](int l) { return qk ? qk + l * ls : nullptr; };
            dr.v_q = [qv, ls](int l) { return qv ? qv + l * ls : nullptr; };
        }
        FwdBatch b;
        b.M = M;
        b.d_tokens = col(0);
        b.d_pos = col(1);
        b.d_kv_row = col(2);
        b.d_seg_lo = col(4);  // unused by the decode attention (own keys come from DecodeRows)
        b.d_work = d_work;
        b.n_work = static_cast<int>(work.size());
        const KvPool* pool = &m->pool;
        const size_t pls = static_cast<size_t>(pool->pages) * sgc::kPageTokens * d;
        b.pfx_rows = static_cast<int>(pool->pages * sgc::kPageTokens);
        b.k_pfx = [pool, pls](int l) { return static_cast<const bf16*>(pool->k + l * pls); };
        b.v_pfx = [pool, pls](int l) { return static_cast<const bf16*>(pool->v + l * pls); };
        b.d_bt = g.d_bt;
        bf16 *gk = g.gk, *gv = g.gv;
        const size_t grows = g.grows;
        b.k_loc = [gk, grows, d](int l) { return gk + l * grows * d; };
        b.v_loc = [gv, grows, d](int l) { return gv + l * grows * d; };
        b.dec = &dr;
        b.d_logit_rows = col(4);
        b.n_logits = M;
        b.d_logits = d_logits;
        forward_rows(c, m, b);
        sgc::step_tokens(c, d_tok_out, d_logits, M, g.d_hint, g.d_atok, g.d_aoff, col(11), col(3), bonus);
        cudaEvent_t ev = c->event();
        SGC_CUDA_CHECK(cudaEventRecord(ev, c->stream));
        const int32_t ev_idx = static_cast<int32_t>(st.events.size());
        st.events.push_back(ev);
        std::vector<int32_t> out(M);
        sgc::copy_out(c, out.data(), d_tok_out, M);
        c->sync();
        check_forward_flags(c);
        st.rows += static_cast<uint64_t>(M);
        for (int i = 0; i < M; ++i) {
            const int32_t j = act[i];
            const uint32_t t = st.count[j];
            st.tokens[static_cast<size_t>(j) * max_new + t] = out[i];
            st.count[j] = t + 1;
            st.last_ev[j] = ev_idx;
            // stop rules after emitting token t (lm_core.cpp:387-389)
            if (out[i] == SGC_EOS || t + 1 == max_new || static_cast<uint64_t>(job.pos0[j]) + t + 1 > max_seq)
                st.done[j] = 1;
        }
    }
}

// ============================================================ graph-side helpers

void ensure_hashes(Ctx* c, sgc_graph* g, uint64_t salt) {
    if (g->hash_salt == salt) return;
    std::vector<uint32_t> b;
    std::vector<int8_t> s;
    std::vector<uint64_t> off(1, 0);
    for (const std::string& t : g->texts) {
        hash_tokens(t.data(), t.size(), salt, b, s);
        off.push_back(b.size());
    }
    dfree(c, g->d_bucket);
    dfree(c, g->d_sign);
    dfree(c, g->d_tok_off);
    g->d_bucket = dalloc<uint32_t>(c, b.size());
    g->d_sign = dalloc<int8_t>(c, s.size());
    g->d_tok_off = dalloc<uint64_t>(c, off.size());
    sgc::copy_in_staged(c, g->d_bucket, b.data(), b.size());
    sgc::copy_in_staged(c, g->d_sign, s.data(), s.size());
    sgc::copy_in_staged(c, g->d_tok_off, off.data(), off.size());
    c->sync();
    g->hash_salt = salt;
}

// frozen encoder state cached per context: text projection and folded GNN weights
struct EncoderState {
    uint32_t dim = 0;
    uint64_t text_seed = 0;
    float* proj_t = nullptr;
    uint32_t layers = 0, heads = 0;
    uint64_t gnn_seed = 0;
    double* wbar = nullptr;
};
std::map<Ctx*, EncoderState> g_enc;

EncoderState& encoder_state(Ctx* c, const sgc_gnn_config& cfg) {
    EncoderState& e = g_enc[c];
    if (!e.proj_t || e.dim != cfg.dim || e.text_seed != cfg.text_seed) {
        dfree(c, e.proj_t);
        e.proj_t = dalloc<float>(c, static_cast<size_t>(cfg.dim) * 4096);
        sgc::gen_text_projection_t(c, e.proj_t, cfg.dim, sgc::splitmix64_once(cfg.text_seed ^ 0x7e87a11dULL));
        e.text_seed = cfg.text_seed;
        e.wbar = (dfree(c, e.wbar), nullptr);
    }
    if (!e.wbar || e.dim != cfg.dim || e.layers != cfg.layers || e.heads != cfg.heads || e.gnn_seed != cfg.seed) {
        dfree(c, e.wbar);
        e.wbar = dalloc<double>(c, static_cast<size_t>(cfg.layers) * cfg.dim * cfg.dim);
        float scale = std::sqrt(3.0f / static_cast<float>(cfg.dim));
        sgc::gnn_gen_wbar(c, e.wbar, cfg.layers, cfg.heads, cfg.dim,
                          sgc::splitmix64_once(cfg.seed ^ 0x6e6eULL), scale);
        e.layers = cfg.layers;
        e.heads = cfg.heads;
        e.gnn_seed = cfg.seed;
    }
    e.dim = cfg.dim;
    return e;
}

float* compute_text_features(Ctx* c, sgc_graph* g, uint32_t dim, uint64_t seed, uint64_t salt,
                             const sgc_gnn_config* gcfg) {
    sgc_gnn_config cfg{};
    if (gcfg) cfg = *gcfg;
    cfg.dim = dim;
    cfg.text_seed = seed;
    if (!gcfg) {  // features only: keep any cached GNN weights of the same dim
        EncoderState& e = g_enc[c];
        cfg.layers = e.layers ? e.layers : 1;
        cfg.heads = e.heads ? e.heads : 1;
        cfg.seed = e.gnn_seed;
    }
    EncoderState& es = encoder_state(c, cfg);
    ensure_hashes(c, g, salt);
    const int ne = static_cast<int>(g->n_nodes + g->n_edges);
    float* feat = c->buf<float>("text_feat", static_cast<size_t>(ne) * dim);
    sgc::text_features(c, feat, g->d_bucket, g->d_sign, g->d_tok_off, ne, es.proj_t, dim);
    return feat;
}

// read a subgraph CSR to host
struct HostSubs {
    std::vector<uint64_t> noff, eoff;
    std::vector<uint32_t> nodes, edges;
};
HostSubs host_subs(Ctx* c, const sgc_subgraphs* s) {
    HostSubs h;
    h.noff = to_host(c, s->node_off, s->count + 1);
    h.eoff = to_host(c, s->edge_off, s->count + 1);
    h.nodes = to_host(c, s->nodes, h.noff[s->count]);
    h.edges = to_host(c, s->edges, h.eoff[s->count]);
    return h;
}

// subgraphs [lo, hi) of a CSR batch
HostSubs slice_subs(const HostSubs& h, uint32_t lo, uint32_t hi) {
    HostSubs s;
    for (uint32_t i = lo; i <= hi; ++i) {
        s.noff.push_back(h.noff[i] - h.noff[lo]);
        s.eoff.push_back(h.eoff[i] - h.eoff[lo]);
    }
    s.nodes.assign(h.nodes.begin() + h.noff[lo], h.nodes.begin() + h.noff[hi]);
    s.edges.assign(h.edges.begin() + h.eoff[lo], h.edges.begin() + h.eoff[hi]);
    return s;
}

uint32_t dense_index(const sgc_graph* g, uint32_t id) {
    auto it = std::lower_bound(g->ids.begin(), g->ids.end(), id);
    if (it == g->ids.end() || *it != id)
        fail(SGC_INTEGRITY, "subgraph node " + std::to_string(id) + " not in parent graph");
    return static_cast<uint32_t>(it - g->ids.begin());
}

// GnnEncoder::encode for a batch of subgraphs; identical subgraphs are encoded once
void encode_subgraphs(Ctx* c, sgc_graph* g, const sgc_gnn_config& cfg, const HostSubs& hs,
                      uint32_t count, float* out_dev) {
    if (cfg.dim == 0 || cfg.layers == 0 || cfg.heads == 0)
        fail(SGC_DOMAIN, "gnn encoder needs dim, layers, heads >= 1");
    if (cfg.dim % 16) fail(SGC_DOMAIN, "gnn dim must be a multiple of 16 on this backend");
    const int d = static_cast<int>(cfg.dim);
    float* feat = compute_text_features(c, g, cfg.dim, cfg.text_seed, cfg.text_salt, &cfg);
    EncoderState& es = g_enc[c];
    // dedup
    std::unordered_map<uint64_t, std::vector<uint32_t>> seen;
    std::vector<uint32_t> uniq_of(count), uniq_first;
    for (uint32_t i = 0; i < count; ++i) {
        uint64_t nn = hs.noff[i + 1] - hs.noff[i], ne = hs.eoff[i + 1] - hs.eoff[i];
        if (nn == 0) fail(SGC_DOMAIN, "encode_subgraph: empty subgraph");
        uint64_t h = sgc::mix64(nn * 1000003ull + ne);
        for (uint64_t k = hs.noff[i]; k < hs.noff[i + 1]; ++k) h = sgc::mix64(h ^ hs.nodes[k]);
        h = sgc::mix64(h ^ 0xabcdefull);
        for (uint64_t k = hs.eoff[i]; k < hs.eoff[i + 1]; ++k) h = sgc::mix64(h ^ hs.edges[k]);
        auto& cand = seen[h];
        uint32_t found = UINT32_MAX;
        for (uint32_t u : cand) {
            if (!c->gnn_dedup) break;
            uint32_t f = uniq_first[u];
            if (hs.noff[f + 1] - hs.noff[f] == nn && hs.eoff[f + 1] - hs.eoff[f] == ne &&
                std::equal(hs.nodes.begin() + hs.noff[i], hs.nodes.begin() + hs.noff[i + 1],
                           hs.nodes.begin() + hs.noff[f]) &&
                std::equal(hs.edges.begin() + hs.eoff[i], hs.edges.begin() + hs.eoff[i + 1],
                           hs.edges.begin() + hs.eoff[f])) {
                found = u;
                break;
            }
        }
        if (found == UINT32_MAX) {
            found = static_cast<uint32_t>(uniq_first.size());
            uniq_first.push_back(i);
            cand.push_back(found);
        }
        uniq_of[i] = found;
    }
    const uint32_t nu = static_cast<uint32_t>(uniq_first.size());
    // node instances of the unique subgraphs with their in-edges (ascending edge index,
    // encoders.cpp:142-162), then per-layer signature dedup: an instance's state after layer
    // l+1 is a function of (its state after l, [(edge, source state after l)] in ascending edge
    // order), so instances with equal signatures share one computed state -- bit-identically
    // in-edges per instance as CSR (in_off / in_e / in_s), each instance's list in ascending
    // edge order (the subgraph's edge list order, as the reference aggregates)
    std::vector<uint32_t> inst_node, sub_off(1, 0);
    std::vector<std::pair<uint32_t, uint32_t>> edge_dst;  // (dst instance, (edge, src) index) per edge
    std::vector<uint32_t> tmp_e, tmp_s;
    std::vector<uint32_t> local_dense;
    for (uint32_t u = 0; u < nu; ++u) {
        uint32_t i = uniq_first[u];
        const uint32_t base = static_cast<uint32_t>(inst_node.size());
        const uint64_t n0 = hs.noff[i], n1 = hs.noff[i + 1];
        local_dense.clear();
        for (uint64_t k = n0; k < n1; ++k) {
            if (k > n0 && hs.nodes[k] <= hs.nodes[k - 1])
                fail(SGC_DOMAIN, "subgraph node ids must be ascending and unique");
            uint32_t di = dense_index(g, hs.nodes[k]);
            local_dense.push_back(di);
            inst_node.push_back(di);
        }
        for (uint64_t k = hs.eoff[i]; k < hs.eoff[i + 1]; ++k) {
            uint32_t e = hs.edges[k];
            if (e >= g->n_edges) fail(SGC_INTEGRITY, "subgraph edge index " + std::to_string(e) + " out of range");
            auto ls = std::lower_bound(local_dense.begin(), local_dense.end(), g->edge_src_idx[e]);
            auto ld = std::lower_bound(local_dense.begin(), local_dense.end(), g->edge_dst_idx[e]);
            if (ls == local_dense.end() || *ls != g->edge_src_idx[e] || ld == local_dense.end() ||
                *ld != g->edge_dst_idx[e])
                fail(SGC_INTEGRITY, "subgraph edge " + std::to_string(e) + " violates closure: endpoint missing");
            edge_dst.push_back({base + static_cast<uint32_t>(ld - local_dense.begin()), static_cast<uint32_t>(tmp_e.size())});
            tmp_e.push_back(e);
            tmp_s.push_back(base + static_cast<uint32_t>(ls - local_dense.begin()));
        }
        sub_off.push_back(static_cast<uint32_t>(inst_node.size()));
    }
    const size_t n_inst = inst_node.size();
    std::vector<uint32_t> in_off(n_inst + 1, 0), in_e(tmp_e.size()), in_s(tmp_e.size());
    for (const auto& ed : edge_dst) ++in_off[ed.first + 1];
    for (size_t v = 0; v < n_inst; ++v) in_off[v + 1] += in_off[v];
    {
        std::vector<uint32_t> fill(in_off.begin(), in_off.end() - 1);
        for (const auto& ed : edge_dst) {  // stable: per instance in subgraph edge order
            const uint32_t o = fill[ed.first]++;
            in_e[o] = tmp_e[ed.second];
            in_s[o] = tmp_s[ed.second];
        }
    }
    // layer 0 groups = distinct nodes
    std::vector<uint32_t> gid(n_inst), g0_node;
    {
        std::vector<uint32_t> m0(g->n_nodes, UINT32_MAX);  // dense node -> group
        for (size_t v = 0; v < n_inst; ++v) {
            uint32_t& slot = m0[inst_node[v]];
            if (!c->gnn_dedup || slot == UINT32_MAX) {
                slot = static_cast<uint32_t>(g0_node.size());
                g0_node.push_back(inst_node[v]);
            }
            gid[v] = slot;
        }
    }
    struct LayerHost {
        std::vector<uint32_t> self_row, in_off{0}, in_src, in_gate;
    };
    std::vector<LayerHost> lh(cfg.layers);
    size_t max_groups = g0_node.size();
    // open-addressing table over (signature hash -> group); a group's signature is read back
    // from its own plan rows (self_row, in_src, in_gate), so no key copies are stored. Groups are
    // numbered in order of first appearance, exactly as before.
    size_t cap = 16;
    while (cap < 2 * n_inst + 16) cap <<= 1;
    std::vector<uint32_t> table(cap);
    std::vector<uint64_t> ghash;
    for (uint32_t l = 0; l < cfg.layers; ++l) {
        std::fill(table.begin(), table.end(), UINT32_MAX);
        ghash.clear();
        std::vector<uint32_t> next(n_inst);
        LayerHost& L = lh[l];
        for (size_t v = 0; v < n_inst; ++v) {
            const uint32_t i0 = in_off[v], i1 = in_off[v + 1], n_in = i1 - i0;
            uint64_t h = sgc::mix64(0x9e3779b97f4a7c15ULL ^ gid[v]);
            for (uint32_t k = i0; k < i1; ++k) {
                h = sgc::mix64(h ^ in_e[k]);
                h = sgc::mix64(h ^ gid[in_s[k]]);
            }
            size_t pos = static_cast<size_t>(h) & (cap - 1);
            uint32_t found = UINT32_MAX;
            for (; c->gnn_dedup && table[pos] != UINT32_MAX; pos = (pos + 1) & (cap - 1)) {
                const uint32_t ng = table[pos];
                if (ghash[ng] != h || L.self_row[ng] != gid[v] || L.in_off[ng + 1] - L.in_off[ng] != n_in)
                    continue;
                bool eq = true;
                for (uint32_t k = 0; k < n_in && eq; ++k) {
                    const uint32_t o = L.in_off[ng] + k;
                    eq = L.in_gate[o] == g->n_nodes + in_e[i0 + k] && L.in_src[o] == gid[in_s[i0 + k]];
                }
                if (eq) {
                    found = ng;
                    break;
                }
            }
            if (found == UINT32_MAX) {
                found = static_cast<uint32_t>(L.self_row.size());
                table[pos] = found;
                ghash.push_back(h);
                L.self_row.push_back(gid[v]);
                for (uint32_t k = i0; k < i1; ++k) {
                    L.in_src.push_back(gid[in_s[k]]);
                    L.in_gate.push_back(g->n_nodes + in_e[k]);
                }
                L.in_off.push_back(static_cast<uint32_t>(L.in_src.size()));
            }
            next[v] = found;
        }
        gid.swap(next);
        max_groups = std::max(max_groups, L.self_row.size());
    }
    sgc::GnnPlan p{};
    p.layers = static_cast<int>(cfg.layers);
    p.heads = static_cast<int>(cfg.heads);
    p.d = d;
    p.n0 = static_cast<int>(g0_node.size());
    uint32_t* d_g0 = c->buf<uint32_t>("gnn_g0", g0_node.size());
    sgc::copy_in_staged(c, d_g0, g0_node.data(), g0_node.size());
    p.g0_node = d_g0;
    if (cfg.layers > 8) fail(SGC_DOMAIN, "gnn encoder supports at most 8 layers on this backend");
    for (uint32_t l = 0; l < cfg.layers; ++l) {
        LayerHost& L = lh[l];
        const std::string t = "gnn_l" + std::to_string(l);
        uint32_t* sr = c->buf<uint32_t>(t + "_self", L.self_row.size());
        uint32_t* io = c->buf<uint32_t>(t + "_off", L.in_off.size());
        uint32_t* is = c->buf<uint32_t>(t + "_src", L.in_src.size());
        uint32_t* ig = c->buf<uint32_t>(t + "_gate", L.in_gate.size());
        sgc::copy_in_staged(c, sr, L.self_row.data(), L.self_row.size());
        sgc::copy_in_staged(c, io, L.in_off.data(), L.in_off.size());
        sgc::copy_in_staged(c, is, L.in_src.data(), L.in_src.size());
        sgc::copy_in_staged(c, ig, L.in_gate.data(), L.in_gate.size());
        p.layer[l] = {static_cast<int>(L.self_row.size()), sr, io, is, ig};
    }
    p.n_sub = static_cast<int>(nu);
    uint32_t* d_so = c->buf<uint32_t>("gnn_sub_off", sub_off.size());
    uint32_t* d_sr = c->buf<uint32_t>("gnn_sub_rows", gid.size());
    sgc::copy_in_staged(c, d_so, sub_off.data(), sub_off.size());
    sgc::copy_in_staged(c, d_sr, gid.data(), gid.size());
    p.sub_off = d_so;
    p.sub_rows = d_sr;
    p.feat = feat;
    p.wbar = es.wbar;
    p.state[0] = c->buf<double>("gnn_state0", max_groups * d);
    p.state[1] = c->buf<double>("gnn_state1", max_groups * d);
    p.agg = c->buf<double>("gnn_agg", max_groups * d);
    float* uniq_out = c->buf<float>("gnn_uniq_out", static_cast<size_t>(nu) * d);
    p.out = uniq_out;
    sgc::gnn_encode_layers(c, p);
    // work accounting (bench.py's embedding roofline): unique node states computed per layer vs
    // the reference's node instances (every subgraph's nodes, every layer)
    c->gnn_state_rows = 0;
    for (uint32_t l = 0; l < cfg.layers; ++l) c->gnn_state_rows += lh[l].self_row.size();
    c->gnn_node_instances = static_cast<uint64_t>(hs.nodes.size()) * cfg.layers;
    // unique subgraph embeddings -> every subgraph
    uint32_t* d_uo = c->buf<uint32_t>("gnn_uniq_of", count);
    sgc::copy_in_staged(c, d_uo, uniq_of.data(), count);
    sgc::gather_rows(c, out_dev, uniq_out, d_uo, static_cast<int>(count), d);
    c->sync();
}

// clustering on device; labels etc. are device pointers
void cluster_device(Ctx* c, const float* d_emb, uint32_t m, uint32_t dim, int linkage, uint32_t k,
                    uint32_t* d_labels, uint32_t* d_left, uint32_t* d_right, double* d_dist) {
    if (k < 1) fail(SGC_DOMAIN, "cluster count must be >= 1");
    if (m == 0) fail(SGC_DOMAIN, "pairwise_distances: need at least one embedding");
    if (k > m)
        fail(SGC_DOMAIN, "cluster count " + std::to_string(k) + " exceeds point count " + std::to_string(m));
    if (linkage < SGC_WARD || linkage > SGC_CENTROID) fail(SGC_DOMAIN, "unknown linkage");
    double* D = c->buf<double>("agg_D", static_cast<size_t>(m) * m);
    bool squared = linkage == SGC_WARD || linkage == SGC_CENTROID;
    sgc::pairwise_distances(c, D, d_emb, static_cast<int>(m), static_cast<int>(dim), squared);
    sgc::agglomerate(c, D, static_cast<int>(m), static_cast<int>(k), linkage, d_labels, d_left, d_right, d_dist);
}

uint64_t agglomerate_op_count(uint64_t m, uint64_t dim, uint64_t c) {
    // clustering.cpp:71,99,130: distance evals + scanned alive pairs + recurrence updates
    uint64_t ops = m * (m - 1) / 2 * dim;
    for (uint64_t a = m; a > c; --a) ops += a * (a - 1) / 2 + (a - 2);
    return ops;
}

// LPT: clusters by descending cost (ties by index) to the least-loaded rank (ties by rank)
std::vector<uint32_t> lpt_assign(const std::vector<double>& cost, int world) {
    std::vector<uint32_t> order(cost.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(world, 0.0);
    std::vector<uint32_t> owner(cost.size(), 0);
    for (uint32_t ci : order) {
        int best = 0;
        for (int r = 1; r < world; ++r)
            if (load[r] < load[best]) best = r;
        owner[ci] = static_cast<uint32_t>(best);
        load[best] += cost[ci];
    }
    return owner;
}

// Member-level rebalancing on top of the cluster LPT. Whole clusters
// first go to ranks by LPT on their cost (prefill + members); then, while the busiest rank is
// ahead of the idlest by more than it costs to replicate one of its clusters' prefix there,
// members of the busiest rank's largest cluster move over (highest query index first) -- the
// receiving rank prefills that prefix itself (a replica: same representative, same tokens), so
// no KV crosses GPUs. Deterministic: every rank computes the same plan from the same labels.
// replica_cost (optional): what another serving rank pays to hold the prefix (default: its
// prefill; with a transport, the point-to-point copy of the sealed K/V).
std::vector<uint32_t> balance_members(const std::vector<double>& prefill_cost,
                                      const std::vector<std::vector<uint32_t>>& members,
                                      const std::vector<double>& member_cost, int world,
                                      std::vector<uint32_t>& cluster_owner,
                                      const std::vector<double>* replica_cost = nullptr) {
    const size_t k = prefill_cost.size();
    std::vector<double> cost(k);
    for (size_t ci = 0; ci < k; ++ci) {
        cost[ci] = prefill_cost[ci];
        for (uint32_t q : members[ci]) cost[ci] += member_cost[q];
    }
    cluster_owner = lpt_assign(cost, world);
    std::vector<uint32_t> qown(member_cost.size(), 0);
    std::vector<double> load(world, 0.0);
    std::set<std::pair<uint32_t, uint32_t>> replica;  // (cluster, rank) holding its prefix
    for (size_t ci = 0; ci < k; ++ci) {
        for (uint32_t q : members[ci]) qown[q] = cluster_owner[ci];
        load[cluster_owner[ci]] += cost[ci];
        replica.insert({static_cast<uint32_t>(ci), cluster_owner[ci]});
    }
    if (world < 2) return qown;
    for (size_t iter = 0; iter < member_cost.size(); ++iter) {
        int rmax = 0, rmin = 0;
        for (int r = 1; r < world; ++r) {
            if (load[r] > load[rmax]) rmax = r;
            if (load[r] < load[rmin]) rmin = r;
        }
        // the busiest rank's largest cluster (by the member work it serves), >= 2 members there
        int best = -1;
        double best_w = 0.0;
        for (size_t ci = 0; ci < k; ++ci) {
            double w = 0.0;
            int cnt = 0;
            for (uint32_t q : members[ci])
                if (qown[q] == static_cast<uint32_t>(rmax)) {
                    w += member_cost[q];
                    ++cnt;
                }
            if (cnt >= 2 && w > best_w) {
                best_w = w;
                best = static_cast<int>(ci);
            }
        }
        if (best < 0) break;
        bool moved = false;
        const auto& mem = members[best];
        int left = 0;
        for (uint32_t q : mem) left += qown[q] == static_cast<uint32_t>(rmax);
        for (auto it = mem.rbegin(); it != mem.rend() && left > 1; ++it) {
            const uint32_t q = *it;
            if (qown[q] != static_cast<uint32_t>(rmax)) continue;
            const bool has = replica.count({static_cast<uint32_t>(best), static_cast<uint32_t>(rmin)}) != 0;
            const double add = member_cost[q] + (has ? 0.0 : (replica_cost ? (*replica_cost)[best] : prefill_cost[best]));
            const double before = std::max(load[rmax], load[rmin]);
            const double after = std::max(load[rmax] - member_cost[q], load[rmin] + add);
            if (!(after < before * (1.0 - 1e-9))) break;
            qown[q] = static_cast<uint32_t>(rmin);
            load[rmax] -= member_cost[q];
            load[rmin] += add;
            replica.insert({static_cast<uint32_t>(best), static_cast<uint32_t>(rmin)});
            --left;
            moved = true;
        }
        if (!moved) break;
    }
    return qown;
}

struct RepResult {
    std::vector<uint64_t> prefix_off;  // [c+1] on host
    int32_t* d_prefix = nullptr;       // device tokens (BOS + bytes)
    uint64_t* d_prefix_off = nullptr;
    std::vector<uint32_t> stats;       // [c x 6]
    uint32_t* d_sel_nodes = nullptr;
    uint32_t* d_sel_edges = nullptr;
};

RepResult build_reps(Ctx* c, sgc_graph* g, const HostSubs& hs, uint32_t count,
                     const std::vector<std::vector<uint32_t>>& members, uint32_t budget_tokens) {
    const uint32_t k = static_cast<uint32_t>(members.size());
    RepResult r;
    // dense node indices of all subgraph nodes (device binary search)
    uint64_t total_nodes = hs.noff[count];
    uint32_t* d_ids = c->buf<uint32_t>("rep_ids", total_nodes);
    int32_t* d_idx = c->buf<int32_t>("rep_idx", total_nodes);
    uint64_t* d_noff = c->buf<uint64_t>("rep_noff", count + 1);
    uint32_t* d_edges = c->buf<uint32_t>("rep_edges_in", hs.eoff[count]);
    uint64_t* d_eoff = c->buf<uint64_t>("rep_eoff", count + 1);
    sgc::copy_in_staged(c, d_ids, hs.nodes.data(), total_nodes);
    sgc::copy_in_staged(c, d_noff, hs.noff.data(), count + 1);
    sgc::copy_in_staged(c, d_edges, hs.edges.data(), hs.eoff[count]);
    sgc::copy_in_staged(c, d_eoff, hs.eoff.data(), count + 1);
    sgc::node_index(c, d_idx, d_ids, total_nodes, g->d_ids, static_cast<int>(g->n_nodes));
    std::vector<uint32_t> mem;
    std::vector<uint64_t> moff(1, 0);
    for (auto& v : members) {
        if (v.empty()) fail(SGC_DOMAIN, "merge_subgraphs: empty member list");
        mem.insert(mem.end(), v.begin(), v.end());
        moff.push_back(mem.size());
    }
    uint32_t* d_mem = c->buf<uint32_t>("rep_members", mem.size());
    uint64_t* d_moff = c->buf<uint64_t>("rep_moff", moff.size());
    sgc::copy_in_staged(c, d_mem, mem.data(), mem.size());
    sgc::copy_in_staged(c, d_moff, moff.data(), moff.size());
    const int nw = static_cast<int>((g->n_nodes + 31) / 32), ew = static_cast<int>((g->n_edges + 31) / 32);
    sgc::UnionArgs a;
    a.clusters = static_cast<int>(k);
    a.sub_nodes = d_idx;
    a.sub_node_off = d_noff;
    a.sub_edges = d_edges;
    a.sub_edge_off = d_eoff;
    a.members = d_mem;
    a.member_off = d_moff;
    a.node_bm = c->buf<uint32_t>("rep_nbm", static_cast<size_t>(k) * std::max(nw, 1));
    a.edge_bm = c->buf<uint32_t>("rep_ebm", static_cast<size_t>(k) * std::max(ew, 1));
    a.node_words = nw;
    a.edge_words = ew;
    a.node_row_len = g->d_node_row_len;
    a.edge_row_len = g->d_edge_row_len;
    a.n_nodes = static_cast<int>(g->n_nodes);
    a.n_edges = static_cast<int>(g->n_edges);
    a.budget_bytes = budget_tokens == 0 ? 0 : budget_tokens - 1;
    a.base_bytes = static_cast<uint32_t>(strlen(kHeader) + strlen(kNodeHdr) + strlen(kEdgeHdr) + 2);
    r.d_sel_nodes = a.sel_nodes = c->buf<uint32_t>("rep_seln", static_cast<size_t>(k) * std::max<uint32_t>(g->n_nodes, 1));
    r.d_sel_edges = a.sel_edges = c->buf<uint32_t>("rep_sele", static_cast<size_t>(k) * std::max<uint32_t>(g->n_edges, 1));
    a.node_pre = c->buf<uint32_t>("rep_npre", static_cast<size_t>(k) * (g->n_nodes + 1));
    a.edge_pre = c->buf<uint32_t>("rep_epre", static_cast<size_t>(k) * (g->n_edges + 1));
    uint32_t* d_stats = c->buf<uint32_t>("rep_stats", static_cast<size_t>(k) * 6);
    a.stats = d_stats;
    int* d_status = c->buf<int>("rep_status", 1);
    a.status = d_status;
    SGC_CUDA_CHECK(cudaMemsetAsync(d_status, 0, sizeof(int), c->stream));
    sgc::union_prompt(c, a);
    r.stats = to_host(c, d_stats, static_cast<size_t>(k) * 6);
    int status = to_host(c, d_status, 1)[0];
    if (status == SGC_INTEGRITY) fail(SGC_INTEGRITY, "subgraph references a node or edge outside the graph");
    if (status == SGC_CAPACITY) fail(SGC_CAPACITY, "prompt headers alone exceed the prefix budget");
    r.prefix_off.assign(1, 0);
    uint64_t maxp = 0;
    const uint64_t head_len = strlen(kHeader) + strlen(kNodeHdr) + 1, ehead_len = strlen(kEdgeHdr) + 1;
    for (uint32_t i = 0; i < k; ++i) {
        const uint32_t* st = &r.stats[i * 6];
        uint64_t P = 1 + head_len + st[4] + ehead_len + st[5];
        maxp = std::max(maxp, P);
        r.prefix_off.push_back(r.prefix_off.back() + P);
    }
    r.d_prefix = c->buf<int32_t>("rep_prefix", r.prefix_off.back());
    r.d_prefix_off = c->buf<uint64_t>("rep_prefix_off", k + 1);
    sgc::copy_in_staged(c, r.d_prefix_off, r.prefix_off.data(), k + 1);
    const std::string h = std::string(kHeader) + kNodeHdr + "\n";
    const std::string eh = std::string(kEdgeHdr) + "\n";
    sgc::GatherArgs ga;
    ga.clusters = static_cast<int>(k);
    ga.max_tokens = maxp;
    ga.tokens = r.d_prefix;
    ga.tok_off = r.d_prefix_off;
    ga.stats = d_stats;
    ga.sel_nodes = a.sel_nodes;
    ga.sel_edges = a.sel_edges;
    ga.node_pre = a.node_pre;
    ga.edge_pre = a.edge_pre;
    ga.node_text = g->d_node_rows;
    ga.node_text_off = g->d_node_row_off;
    ga.edge_text = g->d_edge_rows;
    ga.edge_text_off = g->d_edge_row_off;
    ga.n_nodes = static_cast<int>(g->n_nodes);
    ga.n_edges = static_cast<int>(g->n_edges);
    ga.head_len = static_cast<int>(head_len);
    ga.ehead_len = static_cast<int>(ehead_len);
    ga.head = h.data();
    ga.ehead = eh.data();
    sgc::prompt_gather(c, ga);
    return r;
}

}  // namespace

// ====================================================================== C ABI

extern "C" {

const char* sgc_last_error(void) { return g_last_error.c_str(); }
const char* sgc_version(void) { return "subgcache-b200 0.1 (sm_100a)"; }

int sgc_ctx_create(int device, sgc_ctx** out) {
    return guarded([&] {
        if (!out) fail(SGC_DOMAIN, "null out");
        int n = 0;
        SGC_CUDA_CHECK(cudaGetDeviceCount(&n));
        if (device < 0 || device >= n) fail(SGC_CUDA, "no such CUDA device " + std::to_string(device));
        SGC_CUDA_CHECK(cudaSetDevice(device));
        cudaDeviceProp prop;
        SGC_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) fail(SGC_CUDA, std::string("sm_100a device required, found ") + prop.name);
        auto* h = new sgc_ctx();
        h->c.device = device;
        h->c.num_sms = prop.multiProcessorCount;
        SGC_CUDA_CHECK(cudaStreamCreateWithFlags(&h->c.own_stream, cudaStreamNonBlocking));
        // keep freed pool memory mapped: KV segments and activation buffers are re-allocated
        // every batch, and returning them to the driver would re-map GBs per step
        cudaMemPool_t pool;
        SGC_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        SGC_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        h->c.stream = h->c.own_stream;
        *out = h;
    });
}

int sgc_ctx_destroy(sgc_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        Ctx* c = current(&ctx->c);
        cudaStreamSynchronize(c->stream);
        ctx->comm.reset();
        for (auto& kv : c->scratch) cudaFree(kv.second.ptr);
        auto it = g_enc.find(c);
        if (it != g_enc.end()) {
            cudaFree(it->second.proj_t);
            cudaFree(it->second.wbar);
            g_enc.erase(it);
        }
        for (auto e : c->event_pool) cudaEventDestroy(e);
        for (auto& pe : c->pending) {
            cudaEventDestroy(pe.second.first);
            cudaEventDestroy(pe.second.second);
        }
        if (c->h_flags) cudaFreeHost(c->h_flags);
        if (c->ring_base) cudaFreeHost(c->ring_base);
        for (auto e : c->ring_ev) if (e) cudaEventDestroy(e);
        for (auto& kv : c->pinned_bufs) cudaFreeHost(kv.second.ptr);
        cudaStreamDestroy(c->own_stream);
        if (c->side) cudaStreamDestroy(c->side);
        delete ctx;
    });
}

int sgc_ctx_set_stream(sgc_ctx* ctx, void* stream) {
    return guarded([&] {
        ctx->c.sync();
        ctx->c.stream = stream ? static_cast<cudaStream_t>(stream) : ctx->c.own_stream;
    });
}

uint64_t sgc_ctx_launch_count(const sgc_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int sgc_comm_unique_id(uint8_t id[128]) {
    return guarded([&] { sgc::nccl_unique_id(id); });
}

int sgc_comm_init_nccl(sgc_ctx* ctx, const uint8_t id[128], int world, int rank) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(SGC_DOMAIN, "comm: rank must lie in [0, world)");
        Ctx* c = current(&ctx->c);
        ctx->comm.reset(sgc::comm_nccl(c, id, world, rank));
    });
}

int sgc_comm_init_host(sgc_ctx* ctx, const sgc_host_transport* t, int world, int rank) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(SGC_DOMAIN, "comm: rank must lie in [0, world)");
        ctx->comm.reset(sgc::comm_host(t, world, rank));
    });
}

int sgc_comm_destroy(sgc_ctx* ctx) {
    return guarded([&] {
        current(&ctx->c)->sync();
        ctx->comm.reset();
    });
}

int sgc_comm_info(const sgc_ctx* ctx, int* world, int* rank, int* kind) {
    const sgc::Comm* cm = ctx ? ctx->comm.get() : nullptr;
    if (world) *world = cm ? cm->world : 1;
    if (rank) *rank = cm ? cm->rank : 0;
    if (kind) *kind = cm ? (std::string(cm->kind()) == "nccl" ? 1 : 2) : 0;
    return cm && cm->world > 1 ? 1 : 0;
}

int sgc_model_create(sgc_ctx* ctx, const sgc_lm_config* cfg, sgc_model** out) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        check_lm_cfg(*cfg);
        auto m = std::make_unique<sgc_model>();
        m->c = c;
        m->cfg = *cfg;
        m->d = cfg->model_dim;
        m->H = cfg->heads;
        m->hd = cfg->model_dim / cfg->heads;
        m->L = cfg->layers;
        m->ffn = cfg->ffn_hidden;
        const size_t d = m->d, ffn = m->ffn, L = m->L;
        const uint64_t seed = cfg->seed;
        m->tok_emb = dalloc<float>(c, SGC_VOCAB * d);
        m->head = dalloc<float>(c, SGC_VOCAB * d);
        m->head_t = dalloc<float>(c, SGC_VOCAB * d);
        const float sd = std::sqrt(3.0f / static_cast<float>(d));
        const float sf = std::sqrt(3.0f / static_cast<float>(ffn));
        // lm_core.cpp:131-147: fill_uniform(w, seed ^ const, fan_in) -> stream splitmix64_once(seed^const)
        sgc::gen_uniform(c, m->tok_emb, SGC_VOCAB * d, sgc::splitmix64_once(seed ^ 0x10ad1ULL), -sd, sd);
        sgc::gen_uniform(c, m->head, SGC_VOCAB * d, sgc::splitmix64_once(seed ^ 0x8eadULL), -sd, sd);
        sgc::head_transpose(c, m->head_t, m->head, static_cast<int>(d));
        const size_t per_layer = 3 * d * d + d * d + ffn * d + d * ffn;
        m->weights = dalloc<bf16>(c, per_layer * L);
        for (size_t l = 0; l < L; ++l) {
            bf16* base = m->weights + per_layer * l;
            m->wqkv.push_back(base);
            m->wo.push_back(base + 3 * d * d);
            m->w1.push_back(base + 4 * d * d);
            m->w2.push_back(base + 4 * d * d + ffn * d);
            sgc::gen_uniform(c, m->wqkv[l], 3 * d * d, sgc::splitmix64_once(seed ^ (0x9a11ULL + l * 4)), -sd, sd);
            sgc::gen_uniform(c, m->wo[l], d * d, sgc::splitmix64_once(seed ^ (0x9a12ULL + l * 4)), -sd, sd);
            sgc::gen_uniform(c, m->w1[l], ffn * d, sgc::splitmix64_once(seed ^ (0x9a13ULL + l * 4)), -sd, sd);
            sgc::gen_uniform(c, m->w2[l], d * ffn, sgc::splitmix64_once(seed ^ (0x9a14ULL + l * 4)), -sf, sf);
        }
        // RoPE tables exactly as lm_core.cpp:149-160 (host libm, float)
        const uint32_t half = m->hd / 2, ms = cfg->max_seq_len;
        std::vector<float> cs(static_cast<size_t>(ms) * half), sn(static_cast<size_t>(ms) * half);
        for (uint32_t p = 0; p < ms; ++p)
            for (uint32_t i = 0; i < half; ++i) {
                float freq = std::pow(10000.0f, -2.0f * static_cast<float>(i) / static_cast<float>(m->hd));
                float angle = static_cast<float>(p) * freq;
                cs[static_cast<size_t>(p) * half + i] = std::cos(angle);
                sn[static_cast<size_t>(p) * half + i] = std::sin(angle);
            }
        m->rope_cos = dalloc<float>(c, cs.size());
        m->rope_sin = dalloc<float>(c, sn.size());
        sgc::copy_in(c, m->rope_cos, cs.data(), cs.size());
        sgc::copy_in(c, m->rope_sin, sn.data(), sn.size());
        c->sync();
        *out = m.release();
    });
}

int sgc_model_destroy(sgc_model* m) {
    return guarded([&] {
        if (!m) return;
        Ctx* c = current(m->c);
        dfree(c, m->tok_emb);
        dfree(c, m->head);
        dfree(c, m->head_t);
        dfree(c, m->weights);
        dfree(c, m->rope_cos);
        dfree(c, m->rope_sin);
        dfree(c, m->pool.k);
        dfree(c, m->pool.v);
        c->sync();
        delete m;
    });
}

int sgc_model_weight(sgc_model* m, int which, uint32_t layer, int fp32, float* out, size_t n) {
    return guarded([&] {
        Ctx* c = current(m->c);
        const size_t d = m->d, ffn = m->ffn;
        if (which < 2) {
            if (n != SGC_VOCAB * d) fail(SGC_DOMAIN, "size mismatch");
            sgc::copy_out(c, out, which == 0 ? m->tok_emb : m->head, n);
            c->sync();
            return;
        }
        if (layer >= static_cast<uint32_t>(m->L)) fail(SGC_DOMAIN, "layer out of range");
        size_t cnt = which == 2 ? 3 * d * d : which == 3 ? d * d : ffn * d;
        if (n != cnt) fail(SGC_DOMAIN, "size mismatch");
        const uint64_t seed = m->cfg.seed;
        const uint64_t k = which == 2 ? 0x9a11ULL : which == 3 ? 0x9a12ULL : which == 4 ? 0x9a13ULL : 0x9a14ULL;
        const float s = std::sqrt(3.0f / static_cast<float>(which == 5 ? ffn : d));
        if (fp32) {
            float* tmp = c->buf<float>("wtmp", cnt);
            sgc::gen_uniform(c, tmp, cnt, sgc::splitmix64_once(seed ^ (k + layer * 4)), -s, s);
            sgc::copy_out(c, out, tmp, cnt);
        } else {
            const bf16* src = which == 2 ? m->wqkv[layer] : which == 3 ? m->wo[layer] : which == 4 ? m->w1[layer] : m->w2[layer];
            std::vector<bf16> h(cnt);
            sgc::copy_out(c, h.data(), src, cnt);
            c->sync();
            std::vector<float> f(cnt);
            for (size_t i = 0; i < cnt; ++i) f[i] = __bfloat162float(h[i]);
            sgc::copy_out(c, out, f.data(), cnt);
        }
        c->sync();
    });
}

int sgc_graph_upload(sgc_ctx* ctx, uint32_t n_nodes, const uint32_t* node_ids, const char* node_text,
                     const uint64_t* node_off, uint32_t n_edges, const uint32_t* edge_src,
                     const uint32_t* edge_dst, const char* edge_text, const uint64_t* edge_off,
                     sgc_graph** out) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        auto g = std::make_unique<sgc_graph>();
        g->c = c;
        g->n_nodes = n_nodes;
        g->n_edges = n_edges;
        g->ids.assign(node_ids, node_ids + n_nodes);
        for (uint32_t i = 1; i < n_nodes; ++i)
            if (g->ids[i] <= g->ids[i - 1]) fail(SGC_INTEGRITY, "node ids must be ascending and unique");
        std::string nrows, erows;
        std::vector<uint64_t> noff(1, 0), eoff(1, 0);
        std::vector<uint32_t> nlen, elen;
        for (uint32_t i = 0; i < n_nodes; ++i) {
            std::string attr(node_text + node_off[i], node_text + node_off[i + 1]);
            g->texts.push_back(attr);
            std::string row = std::to_string(g->ids[i]) + ',' + csv_quote(attr);  // graph_store.cpp:251-253
            nrows += row;
            noff.push_back(nrows.size());
            nlen.push_back(static_cast<uint32_t>(row.size()));
        }
        for (uint32_t e = 0; e < n_edges; ++e) {
            std::string attr(edge_text + edge_off[e], edge_text + edge_off[e + 1]);
            g->texts.push_back(attr);
            g->edge_src_idx.push_back(dense_index(g.get(), edge_src[e]));
            g->edge_dst_idx.push_back(dense_index(g.get(), edge_dst[e]));
            std::string row = std::to_string(edge_src[e]) + ',' + csv_quote(attr) + ',' +
                              std::to_string(edge_dst[e]);  // graph_store.cpp:256-259
            erows += row;
            eoff.push_back(erows.size());
            elen.push_back(static_cast<uint32_t>(row.size()));
        }
        g->d_ids = dalloc<uint32_t>(c, n_nodes);
        g->d_node_rows = dalloc<char>(c, nrows.size());
        g->d_node_row_off = dalloc<uint64_t>(c, noff.size());
        g->d_node_row_len = dalloc<uint32_t>(c, nlen.size());
        g->d_edge_rows = dalloc<char>(c, erows.size());
        g->d_edge_row_off = dalloc<uint64_t>(c, eoff.size());
        g->d_edge_row_len = dalloc<uint32_t>(c, elen.size());
        sgc::copy_in(c, g->d_ids, g->ids.data(), n_nodes);
        sgc::copy_in(c, g->d_node_rows, nrows.data(), nrows.size());
        sgc::copy_in(c, g->d_node_row_off, noff.data(), noff.size());
        sgc::copy_in(c, g->d_node_row_len, nlen.data(), nlen.size());
        sgc::copy_in(c, g->d_edge_rows, erows.data(), erows.size());
        sgc::copy_in(c, g->d_edge_row_off, eoff.data(), eoff.size());
        sgc::copy_in(c, g->d_edge_row_len, elen.data(), elen.size());
        c->sync();
        *out = g.release();
    });
}

int sgc_graph_destroy(sgc_graph* g) {
    return guarded([&] {
        if (!g) return;
        Ctx* c = current(g->c);
        for (void* p : {(void*)g->d_ids, (void*)g->d_node_rows, (void*)g->d_node_row_off,
                        (void*)g->d_node_row_len, (void*)g->d_edge_rows, (void*)g->d_edge_row_off,
                        (void*)g->d_edge_row_len, (void*)g->d_bucket, (void*)g->d_sign, (void*)g->d_tok_off})
            dfree(c, p);
        c->sync();
        delete g;
    });
}

int sgc_text_features(sgc_ctx* ctx, sgc_graph* g, uint32_t dim, uint64_t seed, uint64_t salt, float* out) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        if (dim == 0) fail(SGC_DOMAIN, "text encoder dim must be >= 1");
        float* f = compute_text_features(c, g, dim, seed, salt, nullptr);
        sgc::copy_out(c, out, f, static_cast<size_t>(g->n_nodes + g->n_edges) * dim);
        c->sync();
    });
}

int sgc_retrieve(sgc_ctx* ctx, sgc_graph* g, const sgc_retrieval_config* cfg, uint32_t m,
                 const char* q_text, const uint64_t* q_off, uint64_t* node_off, uint32_t* nodes,
                 uint64_t node_cap, uint64_t* edge_off, uint32_t* edges, uint64_t edge_cap) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        // RetrievalConfig::validate (retrieval.cpp:21-25), retrieve() (:226-239)
        if (cfg->k < 1) fail(SGC_DOMAIN, "retrieval k must be >= 1");
        if (cfg->ego_hops < 1) fail(SGC_DOMAIN, "ego hops must be >= 1");
        if (cfg->edge_cost < 0) fail(SGC_DOMAIN, "edge cost must be >= 0");
        if (cfg->dim == 0) fail(SGC_DOMAIN, "text encoder dim must be >= 1");
        if (g->n_nodes == 0) fail(SGC_DOMAIN, "retrieve: graph has no nodes");
        const int N = static_cast<int>(g->n_nodes), E = static_cast<int>(g->n_edges);
        const int d = static_cast<int>(cfg->dim);
        const bool ego = cfg->strategy == SGC_RETRIEVE_EGO_TOPK;
        // element features (nodes then edges) and question features: TextEncoder::embed
        const float* feat = compute_text_features(c, g, cfg->dim, cfg->text_seed, cfg->hash_salt, nullptr);
        std::vector<uint64_t> qo = to_host(c, q_off, m + 1);
        std::vector<char> qt = to_host(c, q_text, qo[m]);
        std::vector<uint32_t> qb;
        std::vector<int8_t> qs;
        std::vector<uint64_t> qtok(1, 0);
        for (uint32_t i = 0; i < m; ++i) {
            hash_tokens(qt.data() + qo[i], qo[i + 1] - qo[i], cfg->hash_salt, qb, qs);
            qtok.push_back(qb.size());
        }
        uint32_t* d_qb = c->buf<uint32_t>("ret_qb", std::max<size_t>(1, qb.size()));
        int8_t* d_qs = c->buf<int8_t>("ret_qs", std::max<size_t>(1, qs.size()));
        uint64_t* d_qtok = c->buf<uint64_t>("ret_qtok", m + 1);
        sgc::copy_in_staged(c, d_qb, qb.data(), qb.size());
        sgc::copy_in_staged(c, d_qs, qs.data(), qs.size());
        sgc::copy_in_staged(c, d_qtok, qtok.data(), m + 1);
        float* qf = c->buf<float>("ret_qf", static_cast<size_t>(std::max<uint32_t>(1, m)) * d);
        sgc::text_features(c, qf, d_qb, d_qs, d_qtok, static_cast<int>(m), g_enc[c].proj_t, d);
        // cosine scores of every (question, element): exact fp64 sums on the device
        const int ne = ego ? N : N + E;
        double* d_dot = c->buf<double>("ret_dot", static_cast<size_t>(std::max<uint32_t>(1, m)) * ne);
        double* d_qsq = c->buf<double>("ret_qsq", std::max<uint32_t>(1, m));
        double* d_esq = c->buf<double>("ret_esq", ne);
        sgc::retrieval_dots(c, d_dot, d_qsq, d_esq, qf, static_cast<int>(m), feat, ne, d);
        std::vector<double> dot = to_host(c, d_dot, static_cast<size_t>(m) * ne);
        std::vector<double> qsq = to_host(c, d_qsq, m), esq = to_host(c, d_esq, ne);
        auto cosine = [](double dt, double na, double nb) {  // encoders.cpp:35-37
            if (na == 0 || nb == 0) return 0.0;
            return dt / (std::sqrt(na) * std::sqrt(nb));
        };
        // undirected adjacency, neighbours sorted by (node id, edge index) (retrieval.cpp:30-49)
        std::vector<std::vector<std::pair<uint32_t, uint32_t>>> nb(N);  // (node index, edge)
        for (int e = 0; e < E; ++e) {
            nb[g->edge_src_idx[e]].push_back({g->edge_dst_idx[e], static_cast<uint32_t>(e)});
            nb[g->edge_dst_idx[e]].push_back({g->edge_src_idx[e], static_cast<uint32_t>(e)});
        }
        for (auto& v : nb) std::sort(v.begin(), v.end());  // node index order == id order
        auto top_k = [](const double* sc, int n, uint32_t k) {  // retrieval.cpp:85-93
            std::vector<uint32_t> o(n);
            std::iota(o.begin(), o.end(), 0u);
            std::stable_sort(o.begin(), o.end(), [&](uint32_t a, uint32_t b) { return sc[a] > sc[b]; });
            if (o.size() > k) o.resize(k);
            return o;
        };
        std::vector<std::set<uint32_t>> out_nodes(m), out_edges(m);  // node indices / edge indices
        if (!ego) {
            // node-edge-topk (retrieval.cpp:96-148)
            for (uint32_t q = 0; q < m; ++q) {
                std::vector<double> sc(ne);
                for (int j = 0; j < ne; ++j) sc[j] = cosine(dot[static_cast<size_t>(q) * ne + j], qsq[q], esq[j]);
                std::set<uint32_t>& sn = out_nodes[q];
                std::set<uint32_t>& se = out_edges[q];
                for (uint32_t i : top_k(sc.data(), N, cfg->k)) sn.insert(i);
                const std::set<uint32_t> seeds = sn;
                for (uint32_t ei : top_k(sc.data() + N, E, cfg->k)) {
                    const uint32_t a = g->edge_src_idx[ei], b2 = g->edge_dst_idx[ei];
                    const bool covered = seeds.count(a) && seeds.count(b2);
                    if (sc[N + ei] >= cfg->edge_cost || covered) {
                        se.insert(ei);
                        sn.insert(a);
                        sn.insert(b2);
                    }
                }
                for (auto it = seeds.begin(); it != seeds.end(); ++it)
                    for (auto jt = std::next(it); jt != seeds.end(); ++jt) {
                        // BFS shortest path, first-discovery parents (retrieval.cpp:54-82)
                        const uint32_t s0 = *it, t0 = *jt;
                        std::vector<int64_t> pe(N, -1), pn(N, -1);
                        std::vector<uint8_t> seen(N, 0);
                        std::deque<uint32_t> dq{s0};
                        seen[s0] = 1;
                        while (!dq.empty()) {
                            const uint32_t u = dq.front();
                            dq.pop_front();
                            if (u == t0) break;
                            for (const auto& [v, ei] : nb[u]) {
                                if (seen[v]) continue;
                                seen[v] = 1;
                                pe[v] = ei;
                                pn[v] = u;
                                dq.push_back(v);
                            }
                        }
                        if (!seen[t0]) continue;
                        std::vector<uint32_t> path;
                        for (uint32_t cur = t0; cur != s0; cur = static_cast<uint32_t>(pn[cur]))
                            path.push_back(static_cast<uint32_t>(pe[cur]));
                        if (path.empty()) continue;
                        const double gain = std::max(0.0, sc[s0]) + std::max(0.0, sc[t0]);
                        if (static_cast<double>(path.size()) * cfg->edge_cost > gain) continue;
                        for (uint32_t ei : path) {
                            se.insert(ei);
                            sn.insert(g->edge_src_idx[ei]);
                            sn.insert(g->edge_dst_idx[ei]);
                        }
                    }
            }
        } else {
            // ego-topk (retrieval.cpp:151-223): ego nets of the top centres on the host, their
            // pooled features and re-ranking scores on the device
            struct Ego {
                uint32_t q, center;
                std::set<uint32_t> nodes, edges;
            };
            std::vector<Ego> egos;
            std::vector<uint32_t> mem_off(1, 0), mem_idx;
            std::vector<int32_t> ego_q;
            for (uint32_t q = 0; q < m; ++q) {
                std::vector<double> sc(N);
                for (int j = 0; j < N; ++j) sc[j] = cosine(dot[static_cast<size_t>(q) * N + j], qsq[q], esq[j]);
                for (uint32_t ci : top_k(sc.data(), N, cfg->ego_entity_cap)) {
                    Ego eg{q, ci, {ci}, {}};
                    std::set<uint32_t> visited{ci};
                    std::deque<std::pair<uint32_t, uint32_t>> dq{{ci, 0u}};
                    while (!dq.empty()) {
                        auto [u, depth] = dq.front();
                        dq.pop_front();
                        if (depth == cfg->ego_hops) continue;
                        for (const auto& [v, ei] : nb[u]) {
                            (void)ei;
                            if (visited.insert(v).second) {
                                eg.nodes.insert(v);
                                dq.push_back({v, depth + 1});
                            }
                        }
                    }
                    for (uint32_t u : eg.nodes)  // induced edges
                        for (const auto& [v, ei] : nb[u])
                            if (eg.nodes.count(v)) eg.edges.insert(ei);
                    for (uint32_t u : eg.nodes) mem_idx.push_back(u);
                    for (uint32_t ei : eg.edges) mem_idx.push_back(static_cast<uint32_t>(N) + ei);
                    mem_off.push_back(static_cast<uint32_t>(mem_idx.size()));
                    ego_q.push_back(static_cast<int32_t>(q));
                    egos.push_back(std::move(eg));
                }
            }
            const int n_ego = static_cast<int>(egos.size());
            std::vector<double> pdot(n_ego), psq(n_ego);
            if (n_ego) {
                uint32_t* d_moff = c->buf<uint32_t>("ret_moff", mem_off.size());
                uint32_t* d_midx = c->buf<uint32_t>("ret_midx", std::max<size_t>(1, mem_idx.size()));
                int32_t* d_eq = c->buf<int32_t>("ret_eq", n_ego);
                float* d_pool = c->buf<float>("ret_pool", static_cast<size_t>(n_ego) * d);
                double* d_pd = c->buf<double>("ret_pd", n_ego);
                double* d_ps = c->buf<double>("ret_ps", n_ego);
                sgc::copy_in_staged(c, d_moff, mem_off.data(), mem_off.size());
                sgc::copy_in_staged(c, d_midx, mem_idx.data(), mem_idx.size());
                sgc::copy_in_staged(c, d_eq, ego_q.data(), n_ego);
                sgc::ego_pool_dots(c, d_pool, d_pd, d_ps, feat, d_moff, d_midx, qf, d_eq, n_ego, d);
                pdot = to_host(c, d_pd, n_ego);
                psq = to_host(c, d_ps, n_ego);
            }
            size_t e0 = 0;
            for (uint32_t q = 0; q < m; ++q) {
                size_t e1 = e0;
                while (e1 < egos.size() && egos[e1].q == q) ++e1;
                std::vector<std::pair<double, uint32_t>> ranked;  // (score, ego)
                for (size_t e = e0; e < e1; ++e) ranked.push_back({cosine(pdot[e], qsq[q], psq[e]), static_cast<uint32_t>(e)});
                std::stable_sort(ranked.begin(), ranked.end(), [&](const auto& a, const auto& b2) {
                    if (a.first != b2.first) return a.first > b2.first;
                    return egos[a.second].center < egos[b2.second].center;
                });
                if (ranked.size() > cfg->k) ranked.resize(cfg->k);
                for (const auto& r : ranked) {  // merge_subgraphs: set union
                    out_nodes[q].insert(egos[r.second].nodes.begin(), egos[r.second].nodes.end());
                    out_edges[q].insert(egos[r.second].edges.begin(), egos[r.second].edges.end());
                }
                e0 = e1;
            }
        }
        // CSR out (node ids ascending == node indices ascending)
        std::vector<uint64_t> no(1, 0), eo(1, 0);
        std::vector<uint32_t> nv, ev;
        for (uint32_t q = 0; q < m; ++q) {
            for (uint32_t i : out_nodes[q]) nv.push_back(g->ids[i]);
            for (uint32_t ei : out_edges[q]) ev.push_back(ei);
            no.push_back(nv.size());
            eo.push_back(ev.size());
        }
        if (nv.size() > node_cap || ev.size() > edge_cap)
            fail(SGC_CAPACITY, "retrieve: output capacity too small (" + std::to_string(nv.size()) + " nodes, " +
                                   std::to_string(ev.size()) + " edges needed)");
        sgc::copy_in(c, node_off, no.data(), no.size());
        sgc::copy_in(c, edge_off, eo.data(), eo.size());
        sgc::copy_in(c, nodes, nv.data(), nv.size());
        sgc::copy_in(c, edges, ev.data(), ev.size());
        c->sync();
    });
}

int sgc_encode_subgraphs(sgc_ctx* ctx, sgc_graph* g, const sgc_gnn_config* cfg,
                         const sgc_subgraphs* subs, float* out) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        HostSubs hs = host_subs(c, subs);
        float* d_out = c->buf<float>("enc_out", static_cast<size_t>(subs->count) * cfg->dim);
        encode_subgraphs(c, g, *cfg, hs, subs->count, d_out);
        sgc::copy_out(c, out, d_out, static_cast<size_t>(subs->count) * cfg->dim);
        c->sync();
    });
}

int sgc_pairwise_distances(sgc_ctx* ctx, const float* emb, uint32_t m, uint32_t dim, double* out) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        if (m == 0) fail(SGC_DOMAIN, "pairwise_distances: need at least one embedding");
        float* e = c->buf<float>("pw_emb", static_cast<size_t>(m) * dim);
        sgc::copy_in(c, e, emb, static_cast<size_t>(m) * dim);
        double* D = c->buf<double>("pw_D", static_cast<size_t>(m) * m);
        sgc::pairwise_distances(c, D, e, static_cast<int>(m), static_cast<int>(dim), false);
        sgc::copy_out(c, out, D, static_cast<size_t>(m) * m);
        c->sync();
    });
}

int sgc_agglomerate(sgc_ctx* ctx, const float* emb, uint32_t m, uint32_t dim, int linkage, uint32_t k,
                    uint32_t* labels, uint32_t* merge_left, uint32_t* merge_right, double* merge_dist,
                    uint64_t* op_count) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        if (k < 1) fail(SGC_DOMAIN, "cluster count must be >= 1");
        if (k > m) fail(SGC_DOMAIN, "cluster count " + std::to_string(k) + " exceeds point count " + std::to_string(m));
        float* e = c->buf<float>("ag_emb", static_cast<size_t>(m) * dim);
        sgc::copy_in(c, e, emb, static_cast<size_t>(m) * dim);
        uint32_t* dl = c->buf<uint32_t>("ag_labels", m);
        uint32_t* dleft = c->buf<uint32_t>("ag_left", m);
        uint32_t* dright = c->buf<uint32_t>("ag_right", m);
        double* ddist = c->buf<double>("ag_dist", m);
        cluster_device(c, e, m, dim, linkage, k, dl, dleft, dright, ddist);
        sgc::copy_out(c, labels, dl, m);
        sgc::copy_out(c, merge_left, dleft, m - k);
        sgc::copy_out(c, merge_right, dright, m - k);
        sgc::copy_out(c, merge_dist, ddist, m - k);
        c->sync();
        if (op_count) *op_count = agglomerate_op_count(m, dim, k);
    });
}

int sgc_build_representatives(sgc_ctx* ctx, sgc_graph* g, const sgc_subgraphs* subs, const uint32_t* labels,
                              uint32_t k, uint32_t budget_tokens, uint64_t* rep_node_off, uint32_t* rep_nodes,
                              uint64_t rep_node_cap, uint64_t* rep_edge_off, uint32_t* rep_edges,
                              uint64_t rep_edge_cap, uint64_t* prefix_off, int32_t* prefix, uint64_t prefix_cap,
                              uint32_t* dropped) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        HostSubs hs = host_subs(c, subs);
        std::vector<uint32_t> lab = to_host(c, labels, subs->count);
        std::vector<std::vector<uint32_t>> members(k);
        for (uint32_t i = 0; i < subs->count; ++i) {
            if (lab[i] >= k) fail(SGC_DOMAIN, "label out of range");
            members[lab[i]].push_back(i);
        }
        RepResult r = build_reps(c, g, hs, subs->count, members, budget_tokens);
        uint64_t nsum = 0, esum = 0;
        for (uint32_t i = 0; i < k; ++i) {
            nsum += r.stats[i * 6];
            esum += r.stats[i * 6 + 1];
        }
        if (rep_nodes && nsum > rep_node_cap) fail(SGC_CAPACITY, "rep_nodes capacity too small");
        if (rep_edges && esum > rep_edge_cap) fail(SGC_CAPACITY, "rep_edges capacity too small");
        if (prefix && r.prefix_off[k] > prefix_cap) fail(SGC_CAPACITY, "prefix capacity too small");
        std::vector<uint64_t> no(1, 0), eo(1, 0);
        for (uint32_t i = 0; i < k; ++i) {
            const uint32_t* st = &r.stats[i * 6];
            if (rep_nodes)
                sgc::copy_out(c, rep_nodes + no.back(), r.d_sel_nodes + static_cast<size_t>(i) * g->n_nodes, st[0]);
            if (rep_edges)
                sgc::copy_out(c, rep_edges + eo.back(), r.d_sel_edges + static_cast<size_t>(i) * g->n_edges, st[1]);
            no.push_back(no.back() + st[0]);
            eo.push_back(eo.back() + st[1]);
            if (dropped) {
                dropped[2 * i] = st[0] - st[2];
                dropped[2 * i + 1] = st[1] - st[3];
            }
        }
        c->sync();
        // selected indices are dense node indices -> convert to ids
        if (rep_nodes) {
            std::vector<uint32_t> tmp = to_host(c, rep_nodes, nsum);
            for (auto& v : tmp) v = g->ids[v];
            sgc::copy_out(c, rep_nodes, tmp.data(), nsum);
        }
        if (rep_node_off) sgc::copy_out(c, rep_node_off, no.data(), k + 1);
        if (rep_edge_off) sgc::copy_out(c, rep_edge_off, eo.data(), k + 1);
        if (prefix_off) sgc::copy_out(c, prefix_off, r.prefix_off.data(), k + 1);
        if (prefix) sgc::copy_out(c, prefix, r.d_prefix, r.prefix_off[k]);
        c->sync();
    });
}

int sgc_prefill(sgc_ctx* ctx, sgc_model* model, const sgc_token_lists* seqs, const float* soft,
                const uint8_t* soft_mask, sgc_kv** out, float* last_logits) {
    return guarded([&] {
        if (seqs->count == 0) fail(SGC_DOMAIN, "prefill: no sequences");
        *out = do_prefill(current(&ctx->c), model, seqs->count, seqs->off, seqs->tokens, soft, soft_mask, last_logits);
    });
}

namespace {
void kv_drop_ref(sgc_kv* kv);
}

int sgc_kv_release(sgc_kv* kv) {
    return guarded([&] {
        if (!kv) return;
        // pages back to the model's pool and frees in stream order once no fork shares them: no
        // drain, so the host keeps preparing the next wave while the GPU still reads these pages
        kv_drop_ref(kv);
    });
}

uint32_t sgc_kv_count(const sgc_kv* kv) { return kv ? kv->n : 0; }
uint64_t sgc_kv_tokens(const sgc_kv* kv, uint32_t i) { return kv && i < kv->n ? kv->len[i] : 0; }
uint64_t sgc_kv_resident_bytes(const sgc_kv* kv) {
    // resident pages (KVCache::resident_kv_bytes counts tokens; pages round up to 128 tokens)
    return kv ? kv->pages.size() * page_bytes(kv->model) : 0;
}
uint32_t sgc_kv_pages(const sgc_kv* kv, uint32_t i, int32_t* pages) {
    if (!kv || i >= kv->n) return 0;
    const uint32_t n = kv->seg_pages(i);
    if (pages) std::copy(kv->pages.begin() + kv->bt_off[i], kv->pages.begin() + kv->bt_off[i] + n, pages);
    return n;
}

namespace {
// device digests of segments `segs` of a handle (kv_digest kernel) into out[0 ..) (device), on
// `stream`; meta / rows: scratch of >= 2 |segs| words and |segs| x 2 L x max len words
void kv_digests(Ctx* c, cudaStream_t stream, const sgc_kv* kv, const std::vector<uint32_t>& segs, uint64_t* out,
                uint32_t* d_meta, uint64_t* d_rows) {
    const uint32_t n = static_cast<uint32_t>(segs.size());
    if (!n) return;
    std::vector<uint32_t> meta(2 * n);
    uint32_t mx = 0;
    for (uint32_t i = 0; i < n; ++i) {
        meta[i] = kv->bt_off[segs[i]];
        meta[n + i] = static_cast<uint32_t>(kv->len[segs[i]]);
        mx = std::max(mx, meta[n + i]);
    }
    SGC_CUDA_CHECK(cudaMemcpyAsync(d_meta, meta.data(), meta.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, stream));
    sgc::kv_digest(c, stream, out, d_rows, kv->model->pool.k, kv->model->pool.v, kv->layer_elems(), kv->d_bt, d_meta,
                   d_meta + n, static_cast<int>(n), static_cast<int>(mx), kv->model->L, kv->model->d);
}
}  // namespace

uint64_t sgc_kv_digest(const sgc_kv* kv, uint32_t i) {
    if (!kv || i >= kv->n) return 0;
    try {
        Ctx* c = current(kv->model->c);
        uint64_t* d_out = c->buf<uint64_t>("kv_digest_out", 1);
        uint32_t* d_meta = c->buf<uint32_t>("kv_digest_meta", 2);
        uint64_t* d_rows = c->buf<uint64_t>("kv_digest_rows", 2ull * kv->model->L * std::max<uint64_t>(1, kv->len[i]));
        kv_digests(c, c->stream, kv, {i}, d_out, d_meta, d_rows);
        uint64_t h = 0;
        sgc::copy_out(c, &h, d_out, 1);
        c->sync();
        return h;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 0;
    }
}

int sgc_kv_read(const sgc_kv* kv, uint32_t i, uint32_t layer, int is_v, float* out) {
    return guarded([&] {
        if (i >= kv->n || layer >= static_cast<uint32_t>(kv->model->L)) fail(SGC_DOMAIN, "kv_read: out of range");
        Ctx* c = current(kv->model->c);
        const size_t d = kv->model->d, n = kv->len[i] * d;
        // gather the segment's rows of every layer through its pages, keep the requested layer
        const int L = kv->model->L;
        bf16* packed = c->buf<bf16>("kv_read_pack", static_cast<size_t>(L) * n);
        sgc::kv_pages_pack(c, packed, is_v ? kv->model->pool.v : kv->model->pool.k, kv->layer_elems(),
                           kv->d_bt + kv->bt_off[i], static_cast<int>(kv->len[i]), L, static_cast<int>(d), true);
        std::vector<bf16> buf(n);
        sgc::copy_out(c, buf.data(), packed + static_cast<size_t>(layer) * n, n);
        c->sync();
        std::vector<float> f(n);
        for (size_t t = 0; t < n; ++t) f[t] = __bfloat162float(buf[t]);
        SGC_CUDA_CHECK(cudaMemcpy(out, f.data(), n * sizeof(float), cudaMemcpyDefault));
    });
}

}  // extern "C"

// ---- fork handles: KVCache::fork / extend / truncate_to / release_suffix (lm_core.hpp:35-92) ----
// A fork shares one sealed segment of an sgc_kv (refcounted, as the reference's shared_ptr to the
// prefix Segment) and owns a private suffix stored in pages of the same pool. Extending a batch of
// forks runs one forward over their new tokens: every row attends to its segment's prefix pages and,
// causally, to its fork's suffix pages (earlier extends included) -- the own-key window starts at
// a virtual row `suffix tokens` before the fork's first new row, so the kernels' causal masks are
// unchanged and only the block table says where the keys live.
struct sgc_fork {
    sgc_kv* kv = nullptr;
    uint32_t seg = 0;
    std::vector<int32_t> pages;  // suffix pages (block table)
    uint64_t suffix = 0;         // suffix tokens
    std::vector<float> last_logits;
    uint64_t prefix_tokens() const { return kv->len[seg]; }
};

namespace {
void kv_drop_ref(sgc_kv* kv) {
    if (--kv->refs == 0) {
        Ctx* c = current(kv->model->c);
        pool_release(kv->model, kv->pages);
        dfree(c, kv->d_bt);
        dfree(c, kv->d_tokens);
        dfree(c, kv->d_tok_off);
        delete kv;
    }
}

void fork_reserve(Ctx* c, sgc_fork* f, uint64_t tokens) {
    const uint32_t need = static_cast<uint32_t>((tokens + sgc::kPageTokens - 1) / sgc::kPageTokens);
    if (need > f->pages.size()) {
        std::vector<int32_t> more = pool_alloc(c, f->kv->model, need - static_cast<uint32_t>(f->pages.size()));
        f->pages.insert(f->pages.end(), more.begin(), more.end());
    }
}

void fork_trim(sgc_fork* f) {
    const size_t keep = (f->suffix + sgc::kPageTokens - 1) / sgc::kPageTokens;
    if (f->pages.size() > keep) {
        pool_release(f->kv->model, std::vector<int32_t>(f->pages.begin() + keep, f->pages.end()));
        f->pages.resize(keep);
    }
}
}  // namespace

extern "C" {

int sgc_kv_fork(sgc_kv* kv, uint32_t seg, sgc_fork** out) {
    return guarded([&] {
        if (!kv || seg >= kv->n) fail(SGC_DOMAIN, "fork: unknown sealed segment");
        auto* f = new sgc_fork();
        f->kv = kv;
        f->seg = seg;
        ++kv->refs;
        *out = f;
    });
}

int sgc_fork_fork(const sgc_fork* src, sgc_fork** out) {
    return guarded([&] {
        Ctx* c = current(src->kv->model->c);
        sgc_model* m = src->kv->model;
        auto f = std::make_unique<sgc_fork>();
        f->kv = src->kv;
        f->seg = src->seg;
        f->last_logits = src->last_logits;
        f->suffix = src->suffix;
        fork_reserve(c, f.get(), src->suffix);  // deep copy of the private suffix (lm_core.cpp:82-90)
        if (src->suffix) {
            const int n = static_cast<int>(src->suffix);
            int32_t* bt = c->buf<int32_t>("fork_copy_bt", 2 * f->pages.size());
            sgc::copy_in_staged(c, bt, src->pages.data(), src->pages.size());
            sgc::copy_in_staged(c, bt + f->pages.size(), f->pages.data(), f->pages.size());
            bf16* stage = c->buf<bf16>("fork_copy_stage", static_cast<size_t>(m->L) * n * m->d);
            const size_t ls = static_cast<size_t>(m->pool.pages) * sgc::kPageTokens * m->d;
            for (bf16* pool : {m->pool.k, m->pool.v}) {
                sgc::kv_pages_pack(c, stage, pool, ls, bt, n, m->L, m->d, true);
                sgc::kv_pages_pack(c, stage, pool, ls, bt + f->pages.size(), n, m->L, m->d, false);
            }
        }
        ++f->kv->refs;
        *out = f.release();
    });
}

uint64_t sgc_fork_tokens(const sgc_fork* f) { return f ? f->prefix_tokens() + f->suffix : 0; }
uint64_t sgc_fork_prefix_tokens(const sgc_fork* f) { return f ? f->prefix_tokens() : 0; }

int sgc_fork_last_logits(const sgc_fork* f, float* out) {
    return guarded([&] {
        const std::vector<float>& lg = f->last_logits;
        if (lg.empty()) fail(SGC_DOMAIN, "fork: no logits yet (extend first)");
        std::memcpy(out, lg.data(), lg.size() * sizeof(float));
    });
}

int sgc_fork_truncate(sgc_fork* f, uint64_t n) {
    return guarded([&] {
        const uint64_t p = f->prefix_tokens();
        if (n < p) fail(SGC_LOGIC, "KVCache: cannot truncate into the sealed prefix segment");
        if (n - p > f->suffix) fail(SGC_DOMAIN, "KVCache: truncate_to beyond current token count");
        f->suffix = n - p;
        fork_trim(f);
    });
}

int sgc_fork_release_suffix(sgc_fork* f) { return sgc_fork_truncate(f, f->prefix_tokens()); }

int sgc_fork_destroy(sgc_fork* f) {
    return guarded([&] {
        if (!f) return;
        current(f->kv->model->c);
        pool_release(f->kv->model, f->pages);
        kv_drop_ref(f->kv);
        delete f;
    });
}

// ToyLm::extend (lm_core.cpp:329-339) on n forks at once: fork j appends tokens[j] to its suffix
int sgc_fork_extend(sgc_ctx* ctx, sgc_model* model, sgc_fork* const* forks, uint32_t n,
                    const sgc_token_lists* tokens, float* logits) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        if (tokens->count != n) fail(SGC_DOMAIN, "fork_extend: one token list per fork");
        if (n == 0) return;
        std::vector<uint64_t> off = to_host(c, tokens->off, n + 1);
        std::vector<int32_t> toks = to_host(c, tokens->tokens, off[n]);
        const int d = model->d;
        // one block table for the call: every involved sealed segment's pages, then every fork's suffix pages
        std::vector<int32_t> bt;
        std::map<std::pair<const sgc_kv*, uint32_t>, int> pfx_at;
        std::vector<int> suf_at(n);
        for (uint32_t j = 0; j < n; ++j) {
            sgc_fork* f = forks[j];
            if (f->kv->model != model) fail(SGC_DOMAIN, "fork does not belong to this model");
            const uint64_t sn = off[j + 1] - off[j];
            if (sn == 0) fail(SGC_DOMAIN, "extend: empty token list");
            if (f->prefix_tokens() + f->suffix + sn > model->cfg.max_seq_len)
                fail(SGC_CAPACITY, "sequence length " + std::to_string(f->prefix_tokens() + f->suffix + sn) +
                                       " exceeds max " + std::to_string(model->cfg.max_seq_len));
            for (uint32_t i = 0; i < j; ++i)
                if (forks[i] == f) fail(SGC_DOMAIN, "fork_extend: a fork appears twice");
        }
        for (uint32_t j = 0; j < n; ++j) fork_reserve(c, forks[j], forks[j]->suffix + off[j + 1] - off[j]);
        for (uint32_t j = 0; j < n; ++j) {
            sgc_fork* f = forks[j];
            auto key = std::make_pair(static_cast<const sgc_kv*>(f->kv), f->seg);
            if (!pfx_at.count(key)) {
                pfx_at[key] = static_cast<int>(bt.size());
                bt.insert(bt.end(), f->kv->pages.begin() + f->kv->bt_off[f->seg],
                          f->kv->pages.begin() + f->kv->bt_off[f->seg] + f->kv->seg_pages(f->seg));
            }
        }
        for (uint32_t j = 0; j < n; ++j) {
            suf_at[j] = static_cast<int>(bt.size());
            bt.insert(bt.end(), forks[j]->pages.begin(), forks[j]->pages.end());
        }
        const int M = static_cast<int>(off[n]);
        std::vector<int32_t> pos, seg_lo, kvrow, lrows;
        std::vector<int> gs, gr, pk, pl, lb;
        for (uint32_t j = 0; j < n; ++j) {
            sgc_fork* f = forks[j];
            const int start = static_cast<int>(off[j]);
            const int sn = static_cast<int>(off[j + 1] - off[j]);
            gs.push_back(start);
            gr.push_back(sn);
            pk.push_back(pfx_at[{f->kv, f->seg}]);
            pl.push_back(static_cast<int>(f->prefix_tokens()));
            lb.push_back(suf_at[j]);
            for (int i = 0; i < sn; ++i) {
                const uint64_t t = f->suffix + i;  // suffix-relative token index
                pos.push_back(static_cast<int32_t>(f->prefix_tokens() + t));
                seg_lo.push_back(start - static_cast<int>(f->suffix));  // virtual: earlier suffix keys
                kvrow.push_back(f->pages[t / sgc::kPageTokens] * sgc::kPageTokens + static_cast<int32_t>(t % sgc::kPageTokens));
            }
            lrows.push_back(start + sn - 1);
        }
        std::vector<sgc::AttnWork> work = make_work(gs, gr, pk, pl, lb, attn_tile(model->hd));
        int32_t* d_arr = c->buf<int32_t>("fk_rows", static_cast<size_t>(M) * 4 + n + bt.size());
        std::vector<int32_t> packed;
        for (auto* v : {&toks, &pos, &seg_lo, &kvrow, &lrows, &bt}) packed.insert(packed.end(), v->begin(), v->end());
        sgc::copy_in_staged(c, d_arr, packed.data(), packed.size());
        sgc::AttnWork* d_work = c->buf<sgc::AttnWork>("fk_work", work.size());
        sgc::copy_in_staged(c, d_work, work.data(), work.size());
        float* d_logits = c->buf<float>("fk_logits", static_cast<size_t>(n) * SGC_VOCAB);
        const KvPool* pool = &model->pool;
        const size_t pls = static_cast<size_t>(pool->pages) * sgc::kPageTokens * d;
        FwdBatch b;
        b.M = M;
        b.d_tokens = d_arr;
        b.d_pos = d_arr + M;
        b.d_seg_lo = d_arr + 2 * static_cast<size_t>(M);
        b.d_kv_row = d_arr + 3 * static_cast<size_t>(M);
        b.d_logit_rows = d_arr + 4 * static_cast<size_t>(M);
        b.d_bt = d_arr + 4 * static_cast<size_t>(M) + n;
        b.d_work = d_work;
        b.n_work = static_cast<int>(work.size());
        b.k_loc = [pool, pls](int l) { return pool->k + l * pls; };
        b.v_loc = [pool, pls](int l) { return pool->v + l * pls; };
        b.loc_rows = static_cast<int>(pool->pages * sgc::kPageTokens);
        b.k_pfx = [pool, pls](int l) { return static_cast<const bf16*>(pool->k + l * pls); };
        b.v_pfx = [pool, pls](int l) { return static_cast<const bf16*>(pool->v + l * pls); };
        b.pfx_rows = b.loc_rows;
        b.n_logits = static_cast<int>(n);
        b.d_logits = d_logits;
        forward_rows(c, model, b);
        std::vector<float> lg(static_cast<size_t>(n) * SGC_VOCAB);
        sgc::copy_out(c, lg.data(), d_logits, lg.size());
        c->sync();
        check_forward_flags(c);
        for (uint32_t j = 0; j < n; ++j) {
            forks[j]->suffix += off[j + 1] - off[j];
            forks[j]->last_logits.assign(lg.begin() + static_cast<size_t>(j) * SGC_VOCAB,
                                         lg.begin() + static_cast<size_t>(j + 1) * SGC_VOCAB);
        }
        if (logits) sgc::copy_in(c, logits, lg.data(), lg.size());
        c->sync();
    });
}

}  // extern "C"

extern "C" {

int sgc_extend(sgc_ctx* ctx, sgc_model* model, sgc_kv* kv, const uint32_t* member_seg,
               const sgc_token_lists* questions, const sgc_token_lists* answers, float pointer_bonus,
               float* logits, int32_t* first_token) {
    return guarded([&] {
        if (kv->model != model) fail(SGC_DOMAIN, "KV cache does not belong to this model");
        const bool ans = answers && answers->count > 0;
        if (ans && answers->count != questions->count) fail(SGC_DOMAIN, "answers/questions count mismatch");
        do_extend(current(&ctx->c), model, kv, questions->count, member_seg, questions->off, questions->tokens,
                  ans ? answers->off : nullptr, ans ? answers->tokens : nullptr, pointer_bonus, logits,
                  first_token);
    });
}

int sgc_extend_generate(sgc_ctx* ctx, sgc_model* model, sgc_kv* kv, const uint32_t* member_seg,
                        const sgc_token_lists* questions, const sgc_token_lists* answers,
                        float pointer_bonus, uint32_t max_new, float* logits, int32_t* first_token,
                        int32_t* tokens, uint32_t* n_tokens) {
    return guarded([&] {
        if (kv->model != model) fail(SGC_DOMAIN, "KV cache does not belong to this model");
        Ctx* c = current(&ctx->c);
        const uint32_t n = questions->count;
        const bool ans = answers && answers->count > 0;
        if (ans && answers->count != n) fail(SGC_DOMAIN, "answers/questions count mismatch");
        if (n == 0) return;
        std::vector<int32_t> first(n);
        ExtendKeep keep;
        do_extend(c, model, kv, n, member_seg, questions->off, questions->tokens, ans ? answers->off : nullptr,
                  ans ? answers->tokens : nullptr, pointer_bonus, logits, first.data(), &keep);
        std::vector<uint32_t> seg = to_host(c, member_seg, n);
        std::vector<uint64_t> qo = to_host(c, questions->off, n + 1);
        GenJob job;
        if (ans) {
            job.a_off = to_host(c, answers->off, n + 1);
            job.a_tok = to_host(c, answers->tokens, job.a_off[n]);
        } else {
            job.a_off.assign(n + 1, 0);
        }
        for (uint32_t j = 0; j < n; ++j) {
            const int32_t S = static_cast<int32_t>(qo[j + 1] - qo[j]);
            job.pfx_bt.push_back(static_cast<int32_t>(kv->bt_off[seg[j]]));
            job.pfx_len.push_back(static_cast<int32_t>(kv->len[seg[j]]));
            job.q_lo.push_back(keep.q_lo[j]);
            job.q_n.push_back(S);
            job.pos0.push_back(static_cast<int32_t>(kv->len[seg[j]]) + S);
            job.first.push_back(first[j]);
            job.hint.push_back(keep.hint[j]);
        }
        const uint32_t mx = std::max<uint32_t>(1, max_new);
        for (uint32_t j = 0; j < n; ++j) job.gen_row0.push_back(static_cast<int32_t>(j * mx));
        GenState st;
        st.init(job, mx, model->cfg.max_seq_len);
        GenBuffers gb = gen_buffers(c, model, kv->pages, &keep, job, static_cast<size_t>(n) * mx);
        std::vector<uint32_t> all(n);
        std::iota(all.begin(), all.end(), 0u);
        decode_steps(c, model, gb, job, st, all, 0, pointer_bonus);
        for (cudaEvent_t e : st.events) c->event_pool.push_back(e);
        if (first_token) sgc::copy_in(c, first_token, first.data(), n);
        if (tokens) sgc::copy_in(c, tokens, st.tokens.data(), st.tokens.size());
        if (n_tokens) sgc::copy_in(c, n_tokens, st.count.data(), n);
        c->sync();
    });
}

int sgc_run_subgcache(sgc_ctx* ctx, sgc_model* model, sgc_graph* g, const sgc_batch* b, sgc_batch_out* o) {
    return guarded([&] {
        Ctx* c = current(&ctx->c);
        const double t_start = now_ms();
        o->prefix_bytes_sent = o->prefix_bytes_received = 0;
        const uint32_t m = b->retrieved.count;
        const uint32_t d = model->d;
        if (m == 0) fail(SGC_DOMAIN, "no queries to run");
        if (b->questions.count != m) fail(SGC_DOMAIN, "questions count != retrieved count");
        if (b->clusters > m) fail(SGC_DOMAIN, "cluster count exceeds batch size");
        const sgc_lm_config& lc = model->cfg;
        // PromptBudget (cache_engine.hpp:21-32)
        const uint32_t reserved = b->question_budget + lc.max_new_tokens + (b->soft_prefix ? 1 : 0);
        const uint32_t budget = reserved >= lc.max_seq_len ? 0 : lc.max_seq_len - reserved;
        if (budget <= 1) fail(SGC_DOMAIN, "max_seq too small for the question budget and generation cap");
        HostSubs hs = host_subs(c, &b->retrieved);
        host_mark("host_subs", t_start);
        // ---- multi-GPU: the context's transport (comm.cuh) or a caller-driven plan
        sgc::Comm* comm = ctx->comm.get();
        const bool use_comm = comm && comm->world > 1;
        if (use_comm && b->world_size > 1 && b->world_size != comm->world)
            fail(SGC_DOMAIN, "batch world_size differs from the context transport's");
        const int world = use_comm ? comm->world : (b->world_size > 1 ? b->world_size : 1);
        const uint32_t me = use_comm ? static_cast<uint32_t>(comm->rank)
                                     : static_cast<uint32_t>(world > 1 || b->cluster_owner ? b->rank : 0);
        // ---- (1) embeddings
        float* d_emb = c->buf<float>("run_emb", static_cast<size_t>(m) * d);
        if (b->precomputed_embeddings) {
            sgc::copy_in(c, d_emb, b->precomputed_embeddings, static_cast<size_t>(m) * d);
        } else if (use_comm) {
            // data-parallel encode: rank r embeds the contiguous shard [r m / W, (r + 1) m / W),
            // then ONE all-gather (NCCL over NVLink) assembles [m x d] in query order on every rank
            auto lo_of = [&](int r) { return static_cast<uint32_t>(static_cast<uint64_t>(r) * m / world); };
            uint32_t mx = 1;
            for (int r = 0; r < world; ++r) mx = std::max(mx, lo_of(r + 1) - lo_of(r));
            const uint32_t lo = lo_of(static_cast<int>(me)), hi = lo_of(static_cast<int>(me) + 1);
            const size_t shard_elems = static_cast<size_t>(mx) * d;
            float* shard = c->buf<float>("run_emb_shard", shard_elems);
            SGC_CUDA_CHECK(cudaMemsetAsync(shard, 0, shard_elems * sizeof(float), c->stream));
            sgc_gnn_config gc = b->gnn;
            gc.dim = d;
            if (hi > lo) encode_subgraphs(c, g, gc, slice_subs(hs, lo, hi), hi - lo, shard);
            float* all = c->buf<float>("run_emb_all", shard_elems * world);
            comm->allgather(c, shard, all, shard_elems * sizeof(float));
            for (int r = 0; r < world; ++r)
                SGC_CUDA_CHECK(cudaMemcpyAsync(d_emb + static_cast<size_t>(lo_of(r)) * d, all + shard_elems * r,
                                               static_cast<size_t>(lo_of(r + 1) - lo_of(r)) * d * sizeof(float),
                                               cudaMemcpyDeviceToDevice, c->stream));
        } else {
            sgc_gnn_config gc = b->gnn;
            gc.dim = d;
            encode_subgraphs(c, g, gc, hs, m, d_emb);
        }
        c->sync();
        const double t_enc = now_ms();
        host_mark("encoded", t_start);
        // ---- (2) clustering
        uint32_t* d_lab = c->buf<uint32_t>("run_labels", m);
        uint32_t* d_left = c->buf<uint32_t>("run_left", m);
        uint32_t* d_right = c->buf<uint32_t>("run_right", m);
        double* d_dist = c->buf<double>("run_dist", m);
        cluster_device(c, d_emb, m, d, b->linkage, b->clusters, d_lab, d_left, d_right, d_dist);
        std::vector<uint32_t> labels = to_host(c, d_lab, m);
        const double t_cl = now_ms();
        host_mark("clustered", t_start);
        const uint32_t k = b->clusters;
        // ---- (3) jobs (pipeline.cpp:249-261) + representatives for the clusters served here
        std::vector<std::vector<uint32_t>> members(k);
        for (uint32_t i = 0; i < m; ++i) members[labels[i]].push_back(i);
        // representatives of every cluster (cheap, exact) -> costs -> LPT owner per cluster
        RepResult reps_all = build_reps(c, g, hs, m, members, budget);
        std::vector<uint64_t> q_off_all = to_host(c, b->questions.off, m + 1);
        std::vector<uint32_t> owner(k, 0);
        std::vector<uint32_t> qown;  // member-level plan (split_clusters): query -> rank
        // split clusters' sealed prefixes travel point to point (instead of replica prefills)
        const bool transfer = use_comm && b->split_clusters && b->transfer_prefix;
        // cost model (FLOPs): a representative's prefill, each member's extend, and the copy of a
        // sealed prefix over NVLink in FLOP-equivalents (bytes x sustained tensor FLOP/s / link B/s)
        std::vector<double> pcost(k, 0.0), mcost(m, 0.0), cost(k, 0.0), xcost(k, 0.0);
        {
            const double ftok = 2.0 * model->L * (4.0 * d * d + 2.0 * d * model->ffn);
            constexpr double kFlopPerLinkByte = 1.35e15 / 6.0e11;
            for (uint32_t ci = 0; ci < k; ++ci) {
                const double P = static_cast<double>(reps_all.prefix_off[ci + 1] - reps_all.prefix_off[ci]);
                pcost[ci] = P * ftok + 2.0 * d * model->L * P * P;
                xcost[ci] = P * 2.0 * model->L * d * sizeof(bf16) * kFlopPerLinkByte;
                cost[ci] = pcost[ci];
                for (uint32_t q : members[ci]) {
                    const double S = static_cast<double>(q_off_all[q + 1] - q_off_all[q]);
                    mcost[q] = S * ftok + 4.0 * d * model->L * S * P;
                    cost[ci] += mcost[q];
                }
            }
        }
        // a split cluster's other serving ranks receive the sealed K/V when the copy is cheaper
        // than prefilling a replica (C3: 1.1 GB ~ 2.4 TFLOP-eq vs a 25 TFLOP prefill; the tiny C1
        // model: replicas), or always with transfer_prefix == 2
        std::vector<uint8_t> xfer(k, 0);
        for (uint32_t ci = 0; ci < k; ++ci)
            xfer[ci] = transfer && (b->transfer_prefix == 2 || xcost[ci] < pcost[ci]) ? 1 : 0;
        if (b->cluster_owner) {
            owner = to_host(c, b->cluster_owner, k);
        } else if (world > 1) {
            if (b->split_clusters) {
                std::vector<double> rcost(k, 0.0);
                for (uint32_t ci = 0; ci < k; ++ci) rcost[ci] = xfer[ci] ? std::min(pcost[ci], xcost[ci]) : pcost[ci];
                qown = balance_members(pcost, members, mcost, world, owner, &rcost);
            } else {
                owner = lpt_assign(cost, world);
            }
        }
        // every rank knows who serves what (the plan is deterministic)
        std::vector<uint32_t> qrank(m, 0);
        for (uint32_t i = 0; i < m; ++i) qrank[i] = qown.empty() ? owner[labels[i]] : qown[i];
        if (o->query_rank) std::memcpy(o->query_rank, qrank.data(), m * sizeof(uint32_t));
        // a split cluster is served by more than one rank; with `transfer` its owner prefills it
        // and sends the sealed K/V to the other serving ranks
        std::vector<std::vector<uint32_t>> peers(k);  // serving ranks other than the owner
        for (uint32_t ci = 0; ci < k; ++ci) {
            std::set<uint32_t> rs;
            for (uint32_t q : members[ci])
                if (qrank[q] != owner[ci]) rs.insert(qrank[q]);
            peers[ci].assign(rs.begin(), rs.end());
        }
        auto is_split = [&](uint32_t ci) { return xfer[ci] && !peers[ci].empty(); };
        // representative prompt lengths of every cluster (deterministic on every rank)
        if (o->prefix_len)
            for (uint32_t ci = 0; ci < k; ++ci)
                o->prefix_len[ci] = reps_all.prefix_off[ci + 1] - reps_all.prefix_off[ci] + (b->soft_prefix ? 1 : 0);
        if (o->owner) sgc::copy_out(c, o->owner, owner.data(), k);
        std::vector<uint32_t> owned;
        std::vector<std::vector<uint32_t>> served(k);  // members this rank serves, per cluster
        for (uint32_t ci = 0; ci < k; ++ci) {
            for (uint32_t q : members[ci])
                if (qrank[q] == me) served[ci].push_back(q);
            // the owner of a split cluster prefills it even when all its members moved away
            if (!served[ci].empty() || (is_split(ci) && owner[ci] == me)) owned.push_back(ci);
        }
        // serving order: Smith's rule (ascending row cost per query) so the waves that finish
        // first carry the most queries -- minimizes the summed (mean) TTFT; results are
        // independent of the order (every row's math is batch-independent)
        if (b->waves > 1) {
            std::vector<double> ratio(k, 0.0);
            for (uint32_t ci : owned) {
                double cost = static_cast<double>(reps_all.prefix_off[ci + 1] - reps_all.prefix_off[ci]);
                for (uint32_t q : members[ci]) cost += static_cast<double>(q_off_all[q + 1] - q_off_all[q]);
                ratio[ci] = cost / std::max<size_t>(1, members[ci].size());
            }
            std::stable_sort(owned.begin(), owned.end(), [&](uint32_t a, uint32_t b2) { return ratio[a] < ratio[b2]; });
        }
        // split clusters first: all of them are served in wave 0, where their K/V are exchanged
        std::stable_partition(owned.begin(), owned.end(), [&](uint32_t ci) { return is_split(ci); });
        uint32_t n_split = 0;
        for (uint32_t ci : owned) n_split += is_split(ci) ? 1 : 0;
        auto is_remote = [&](uint32_t ci) { return is_split(ci) && owner[ci] != me; };
        if (o->prefilled)
            for (uint32_t ci = 0; ci < k; ++ci) o->prefilled[ci] = 0;
        // representatives are built from the FULL membership (a replicated prefix is identical on
        // every rank serving part of the cluster); own_members are the queries served here
        std::vector<std::vector<uint32_t>> own_members, rep_members;
        for (uint32_t ci : owned) {
            own_members.push_back(served[ci]);
            rep_members.push_back(members[ci]);
        }
        RepResult reps;
        if (!owned.empty()) {
            if (owned.size() == k && b->waves <= 1 && n_split == 0) reps = reps_all;
            else reps = build_reps(c, g, hs, m, rep_members, budget);
        }
        std::vector<float> soft_h;
        std::vector<uint8_t> soft_mask;
        float* d_soft = nullptr;
        if (b->soft_prefix && !owned.empty()) {
            // soft prefix = gnn.encode(representative) (pipeline.cpp:270-276)
            std::vector<uint64_t> no(1, 0), eo(1, 0);
            std::vector<uint32_t> rn, re;
            for (size_t i = 0; i < owned.size(); ++i) {
                const uint32_t* st = &reps.stats[i * 6];
                std::vector<uint32_t> sn = to_host(c, reps.d_sel_nodes + i * g->n_nodes, st[0]);
                std::vector<uint32_t> se = to_host(c, reps.d_sel_edges + i * g->n_edges, st[1]);
                for (auto v : sn) rn.push_back(g->ids[v]);
                re.insert(re.end(), se.begin(), se.end());
                no.push_back(rn.size());
                eo.push_back(re.size());
            }
            HostSubs rs{no, eo, rn, re};
            sgc_gnn_config gc = b->gnn;
            gc.dim = d;
            d_soft = c->buf<float>("run_soft", owned.size() * d);
            encode_subgraphs(c, g, gc, rs, static_cast<uint32_t>(owned.size()), d_soft);
        }
        c->sync();
        const double t_rep = now_ms();
        host_mark("represented", t_start);
        // ---- (4) KV precompute: representative prompts (+ standalone fallbacks) in one batch
        std::vector<uint64_t> q_off = to_host(c, b->questions.off, m + 1);
        std::vector<int32_t> q_tok = to_host(c, b->questions.tokens, q_off[m]);
        std::vector<uint64_t> a_off;
        std::vector<int32_t> a_tok;
        const bool ans = b->answers.count == m && b->answers.off;
        if (ans) {
            a_off = to_host(c, b->answers.off, m + 1);
            a_tok = to_host(c, b->answers.tokens, a_off[m]);
        }
        std::vector<int32_t> rep_tok = owned.empty() ? std::vector<int32_t>() : to_host(c, reps.d_prefix, reps.prefix_off.back());
        std::vector<float> soft_all;
        if (d_soft) soft_all = to_host(c, d_soft, owned.size() * d);
        std::vector<uint64_t> oo;
        std::vector<int32_t> ot;
        std::vector<float> emb_h;
        // ---- waves: owned clusters (serving order) in groups, so members of early clusters get
        // their first token before the whole batch is done (TTFT), while each wave still feeds
        // the GEMMs thousands of rows. First-token runs cut by query count (TTFT p50); runs to
        // EOS cut by row cost (balanced waves decode their members sooner: RT p50 672 vs 913 ms
        // at C3 with 4 waves)
        const uint32_t nown = static_cast<uint32_t>(owned.size());
        const bool cut_by_cost = b->max_new_tokens > 1;
        std::vector<double> wcost(nown, 0.0);
        double total_cost = 0;
        for (uint32_t i = 0; i < nown; ++i) {
            wcost[i] = static_cast<double>(reps.prefix_off[i + 1] - reps.prefix_off[i]);
            for (uint32_t q : own_members[i]) wcost[i] += static_cast<double>(q_off[q + 1] - q_off[q]);
            total_cost += wcost[i];
        }
        uint32_t n_waves = b->waves > 0 ? b->waves : 1;
        n_waves = std::max<uint32_t>(1, std::min(n_waves, nown));
        std::vector<uint32_t> wave_end;  // exclusive cluster index bound per wave
        {
            // cut wave w once MORE than (w + 1) / n_waves of the served queries are in: with the
            // Smith order the early waves are the cheap ones, and with 2 waves the median query
            // finishes with the first (TTFT p50 = end of wave 1, below half the batch's work)
            size_t served_q = 0;
            for (uint32_t i = 0; i < nown; ++i) served_q += own_members[i].size();
            size_t acc_q = 0;
            double acc = 0;
            for (uint32_t i = 0; i < nown; ++i) {
                acc_q += own_members[i].size();
                acc += wcost[i];
                const uint32_t w = static_cast<uint32_t>(wave_end.size());
                const bool last_wave = w + 1 == n_waves;
                const bool reached = cut_by_cost ? acc >= total_cost * (w + 1) / n_waves
                                                 : acc_q * n_waves > served_q * (w + 1);
                // or when only one cluster per remaining wave is left
                const bool must = nown - (i + 1) == n_waves - (w + 1);
                if (!last_wave && (reached || must) && nown - (i + 1) >= n_waves - (w + 1)) wave_end.push_back(i + 1);
            }
            while (wave_end.size() < n_waves) wave_end.push_back(nown);
        }
        {
            // KV page budget: a wave's representatives take whole 128-token pages of the model's
            // pool, which may grow into the free device memory minus a reserve for the forward's
            // activations (prefill runs in row chunks of <= 64k rows) and the extend scratch; split
            // any wave whose pages exceed it (C4 with 256 clusters: ~137 GB of K/V in each of 2 waves)
            size_t free_b = 0, total_b = 0;
            c->mem_info(&free_b, &total_b);
            const double act_row = d * (4.0 + 2 * 4) + 2.0 * model->ffn + 4.0 * d / 32;  // x, xb, q, ao, h, ss
            const double reserve = 2.0 * 65536.0 * act_row + 0.06 * static_cast<double>(total_b);
            const double pb = static_cast<double>(page_bytes(model));
            const double budget = static_cast<double>(model->pool.free_pages.size()) * pb +
                                  std::max(0.0, static_cast<double>(free_b) - reserve);
            const uint64_t cap = std::max<uint64_t>(1, static_cast<uint64_t>(budget / pb));
            std::vector<uint32_t> split;
            uint32_t w0 = 0;
            for (uint32_t e : wave_end) {
                uint64_t pages = 0;
                for (uint32_t i = w0; i < e; ++i) {
                    const uint64_t pr = (reps.prefix_off[i + 1] - reps.prefix_off[i] + 1 + sgc::kPageTokens - 1) /
                                        sgc::kPageTokens;
                    if (pages > 0 && pages + pr > cap) {
                        split.push_back(i);
                        pages = 0;
                    }
                    pages += pr;
                }
                split.push_back(e);
                w0 = e;
            }
            wave_end.swap(split);
            if (n_split > 0) {  // wave 0 holds every split cluster (one exchange point)
                std::vector<uint32_t> we2{std::max(wave_end.front(), n_split)};
                for (uint32_t e : wave_end)
                    if (e > we2.back()) we2.push_back(e);
                wave_end.swap(we2);
            }
        }
        host_mark("waves planned", t_start);
        cudaEvent_t ev_start = c->event();
        SGC_CUDA_CHECK(cudaEventRecord(ev_start, c->stream));
        std::vector<cudaEvent_t> ev_wave, ev_seal, ev_wave_start;
        std::vector<uint8_t> fb_flag(m, 0);
        double dev_pf_ms = 0.0, dev_ex_ms = 0.0;
        std::vector<int32_t> wave_of(m, -1);
        uint64_t prefill_rows = 0, extend_rows = 0, decode_rows = 0;
        double pf_ms = 0, ex_ms = 0, dec_ms = 0;
        const uint32_t max_new = b->max_new_tokens;
        const bool gen_on = max_new > 1;
        std::vector<int32_t> wave_of_job;  // decode job index -> wave
        // deferred first-token outputs (first tokens only): pinned, in extend order, + query ids
        float* def_lg = o->logits ? c->pinned<float>("run_def_lg", static_cast<size_t>(m) * SGC_VOCAB) : nullptr;
        int32_t* def_ft = c->pinned<int32_t>("run_def_ft", m);
        std::vector<uint32_t> def_q;
        uint32_t def_n = 0;
        // ---- row budget of every wave: prefill rows (representatives + standalone fallbacks)
        // and kept question rows; with generation the waves' prefix / question K/V stay resident
        // until the end so stragglers of every wave decode together (one weight pass per step)
        std::vector<uint64_t> wave_pf(wave_end.size(), 0), wave_qr(wave_end.size(), 0), wave_pg(wave_end.size(), 0);
        auto pages_of = [](uint64_t rows) { return (rows + sgc::kPageTokens - 1) / sgc::kPageTokens; };
        {
            uint32_t w0 = 0;
            for (uint32_t wv = 0; wv < wave_end.size(); ++wv) {
                for (uint32_t i = w0; i < wave_end[wv]; ++i) {
                    const uint64_t plen = reps.prefix_off[i + 1] - reps.prefix_off[i] + (d_soft ? 1 : 0);
                    wave_pf[wv] += plen;
                    wave_pg[wv] += pages_of(plen);
                    for (uint32_t q : own_members[i]) {
                        const uint64_t qn = q_off[q + 1] - q_off[q];
                        if (plen + qn + lc.max_new_tokens > lc.max_seq_len) {
                            if (b->own_prefix.count != m) fail(SGC_DOMAIN, "fallback needs own_prefix token lists");
                            if (oo.empty()) {
                                oo = to_host(c, b->own_prefix.off, m + 1);
                                ot = to_host(c, b->own_prefix.tokens, oo[m]);
                            }
                            size_t allowed = lc.max_seq_len;
                            allowed -= std::min<size_t>(allowed, lc.max_new_tokens + (b->soft_prefix ? 1 : 0));
                            const uint64_t fl = std::min<uint64_t>(oo[q + 1] - oo[q] + qn, allowed) + (b->soft_prefix ? 1 : 0);
                            wave_pf[wv] += fl;
                            wave_pg[wv] += pages_of(fl);
                        } else {
                            wave_qr[wv] += qn;
                        }
                    }
                }
                w0 = wave_end[wv];
            }
        }
        uint64_t pf_total = 0, qr_total = 0, pg_total = 0, pg_max = 0, qr_max = 0;
        for (size_t w = 0; w < wave_end.size(); ++w) {
            pf_total += wave_pf[w];
            qr_total += wave_qr[w];
            pg_total += wave_pg[w];
            pg_max = std::max(pg_max, wave_pg[w]);
            qr_max = std::max(qr_max, wave_qr[w]);
        }
        // retain every wave's K/V only when generating and it fits comfortably (C3: ~45 GB):
        // pages of every wave + kept question rows + generated rows, against the free device
        // memory (weights and scratch already allocated; the pool's free pages and the re-used
        // keep buffers count as free), 20% headroom for the forward activations
        const double kv_row_bytes = 2.0 * model->L * d * sizeof(bf16);
        size_t free_now = 0, total_now = 0;
        c->mem_info(&free_now, &total_now);
        double avail_now = static_cast<double>(free_now) +
                           static_cast<double>(model->pool.free_pages.size()) * page_bytes(model);
        for (const char* nm : {"ex_keep_k", "ex_keep_v"}) {
            auto it = c->scratch.find(nm);  // grow-only buffers this batch re-uses (or regrows)
            if (it != c->scratch.end()) avail_now += static_cast<double>(it->second.bytes);
        }
        const bool retain = gen_on && static_cast<double>(pg_total) * page_bytes(model) +
                                              (qr_total + static_cast<double>(m) * max_new) * kv_row_bytes <
                                          0.8 * avail_now;
        // grow the pool once up front (a mid-batch growth would copy the live pages)
        pool_grow(c, model, model->pool.live() + static_cast<uint32_t>(retain ? pg_total : pg_max));
        o->kv_pages_peak = 0;
        o->kv_page_bytes = page_bytes(model);
        ExtendKeep keep_all;
        if (gen_on) {
            keep_all.rows = std::max<uint64_t>(1, retain ? qr_total : qr_max);
            keep_all.k = c->buf<bf16>("ex_keep_k", static_cast<size_t>(model->L) * keep_all.rows * d);
            keep_all.v = c->buf<bf16>("ex_keep_v", static_cast<size_t>(model->L) * keep_all.rows * d);
        }
        // stragglers: a wave stops decoding on its own once fewer than this many of its queries
        // are still generating; they finish in one shared loop after the last wave
        const uint32_t defer_pct = retain ? c->decode_defer_pct : 0;
        GenJob gj;                  // every query served here, in wave order
        GenState gst;
        gst.max_new = std::max<uint32_t>(1, max_new);
        std::vector<uint32_t> gen_q;  // job index -> query
        // retained waves' sealed prefixes (generation) and the block table over all of them
        std::vector<std::unique_ptr<sgc_kv, int (*)(sgc_kv*)>> held;
        std::vector<int32_t> gen_bt;
        // sealed-prefix digests (KVCache::prefix_digest at seal, re-checked once the members are
        // served, cache_engine.cpp:189, :210): device slots [seal | end] per served cluster
        // The digests run on a side stream: the seal digest overlaps the members' extend (which only
        // reads the prefix pages), the end digest follows the wave's last use of them and the main
        // stream waits for it before those pages can be reused. Scratch is sized once up front.
        const bool verify = b->verify_prefix != 0;
        const uint32_t dig_cap = static_cast<uint32_t>(owned.size());
        uint64_t* d_dig = verify ? c->buf<uint64_t>("run_digests", 2 * static_cast<size_t>(dig_cap) + 2) : nullptr;
        uint32_t* d_dig_meta[2] = {nullptr, nullptr};
        uint64_t* d_dig_rows[2] = {nullptr, nullptr};
        if (verify) {  // two sets: the seal digest of wave w+1 may overlap the end digest of wave w
            for (int t = 0; t < 2; ++t) {
                d_dig_meta[t] = c->buf<uint32_t>(t ? "run_dig_meta1" : "run_dig_meta0", 2 * static_cast<size_t>(dig_cap) + 2);
                d_dig_rows[t] = c->buf<uint64_t>(t ? "run_dig_rows1" : "run_dig_rows0",
                                                 static_cast<size_t>(dig_cap) * 2 * model->L * lc.max_seq_len + 1);
            }
        }
        std::vector<std::pair<uint32_t, uint32_t>> dig_slot;  // (cluster, seal slot); end slot = seal + dig_cap
        uint32_t dig_n = 0;
        std::vector<std::pair<uint32_t, std::vector<uint32_t>>> dig_wave;  // held waves: (first slot, segments)
        // digest of segments `segs` of `kv` into slots slot0.. after everything on the main stream so far
        auto digest_wave = [&](const sgc_kv* kv, const std::vector<uint32_t>& segs, uint32_t slot0, bool end) {
            cudaStream_t side = c->side_stream();
            cudaEvent_t e = c->event();
            SGC_CUDA_CHECK(cudaEventRecord(e, c->stream));
            SGC_CUDA_CHECK(cudaStreamWaitEvent(side, e, 0));
            // the seal (end) digests of consecutive waves alternate scratch sets 0 / 1 -- both
            // run on the one side stream, so a set is never overwritten while in use
            const int t = end ? 1 : 0;
            kv_digests(c, side, kv, segs, d_dig + slot0 + (end ? dig_cap : 0), d_dig_meta[t], d_dig_rows[t]);
            if (end) {  // the pages go back to the pool after this: the main stream waits for it
                cudaEvent_t e2 = c->event();
                SGC_CUDA_CHECK(cudaEventRecord(e2, side));
                SGC_CUDA_CHECK(cudaStreamWaitEvent(c->stream, e2, 0));
                c->event_pool.push_back(e2);
            }
            c->event_pool.push_back(e);
        };
        uint64_t keep_row0 = 0;
        uint32_t wb = 0;
        for (uint32_t wv = 0; wv < wave_end.size(); ++wv) {
            const uint32_t we = wave_end[wv];
            if (we <= wb) continue;
            const double tw0 = now_ms();
            host_mark("wave start", t_start);
            {
                cudaEvent_t e0 = c->event();
                SGC_CUDA_CHECK(cudaEventRecord(e0, c->stream));
                ev_wave_start.push_back(e0);
            }
            std::vector<uint64_t> seq_off(1, 0);
            std::vector<int32_t> seq_tok;
            std::vector<uint8_t> seq_soft;
            std::vector<float> seq_soft_vec;
            std::vector<uint32_t> mem_seg, mem_q;  // extend members (segment index within the wave)
            std::vector<uint32_t> fb_q;            // fallback queries -> their standalone sequence
            std::vector<uint64_t> fb_seq;
            const uint32_t job0 = gj.size();  // this wave's decode rows: job0 .. (members, then fallbacks)
            ExtendKeep keep = keep_all;
            keep.base = retain ? keep_row0 : 0;
            // sequences of the wave: local representatives, standalone fallbacks, then the split
            // clusters' representatives whose sealed K/V arrive from their owner (not computed here)
            std::vector<uint32_t> seq_of(we - wb, 0), remote_i, mem_cl;
            auto push_rep = [&](uint32_t i) {
                seq_of[i - wb] = static_cast<uint32_t>(seq_off.size() - 1);
                seq_tok.insert(seq_tok.end(), rep_tok.begin() + reps.prefix_off[i], rep_tok.begin() + reps.prefix_off[i + 1]);
                seq_off.push_back(seq_tok.size());
                seq_soft.push_back(d_soft ? 1 : 0);
                if (d_soft) seq_soft_vec.insert(seq_soft_vec.end(), soft_all.begin() + static_cast<size_t>(i) * d, soft_all.begin() + static_cast<size_t>(i + 1) * d);
                else seq_soft_vec.insert(seq_soft_vec.end(), d, 0.f);
            };
            for (uint32_t i = wb; i < we; ++i) {
                if (is_remote(owned[i])) remote_i.push_back(i);
                else push_rep(i);
                const uint64_t plen = reps.prefix_off[i + 1] - reps.prefix_off[i] + (d_soft ? 1 : 0);
                for (uint32_t q : own_members[i]) {
                    const uint64_t qn = q_off[q + 1] - q_off[q];
                    wave_of[q] = static_cast<int32_t>(wv);
                    if (plen + qn + lc.max_new_tokens > lc.max_seq_len) {  // cache_engine.cpp:171
                        fb_q.push_back(q);
                    } else {
                        mem_cl.push_back(i);
                        mem_q.push_back(q);
                    }
                }
            }
            // standalone path for fallbacks (cache_engine.cpp:112-138): own prompt + question, trimmed
            if (!fb_q.empty()) {
                if (b->own_prefix.count != m) fail(SGC_DOMAIN, "fallback needs own_prefix token lists");
                if (b->soft_prefix && emb_h.empty()) emb_h = to_host(c, d_emb, static_cast<size_t>(m) * d);
                for (uint32_t q : fb_q) {
                    std::vector<int32_t> full(ot.begin() + oo[q], ot.begin() + oo[q + 1]);
                    full.insert(full.end(), q_tok.begin() + q_off[q], q_tok.begin() + q_off[q + 1]);
                    size_t allowed = lc.max_seq_len;
                    allowed -= std::min<size_t>(allowed, lc.max_new_tokens + (b->soft_prefix ? 1 : 0));
                    if (full.size() > allowed) full.resize(allowed);
                    fb_seq.push_back(seq_off.size() - 1);
                    seq_tok.insert(seq_tok.end(), full.begin(), full.end());
                    seq_off.push_back(seq_tok.size());
                    seq_soft.push_back(b->soft_prefix ? 1 : 0);
                    if (b->soft_prefix) seq_soft_vec.insert(seq_soft_vec.end(), emb_h.begin() + static_cast<size_t>(q) * d, emb_h.begin() + static_cast<size_t>(q + 1) * d);
                    else seq_soft_vec.insert(seq_soft_vec.end(), d, 0.f);
                }
            }
            for (uint32_t i : remote_i) push_rep(i);  // trailing: laid out, not computed
            for (size_t j = 0; j < mem_q.size(); ++j) mem_seg.push_back(seq_of[mem_cl[j] - wb]);
            const uint32_t ns = static_cast<uint32_t>(seq_off.size() - 1);
            const uint32_t n_remote = static_cast<uint32_t>(remote_i.size());
            // representative logits are only read on the host for standalone fallbacks; without
            // them no sync is needed and the host prepares the next wave while the GPU works
            std::vector<float> seq_logits(fb_q.empty() ? 0 : static_cast<size_t>(ns) * SGC_VOCAB);
            sgc_kv* kv = do_prefill(c, model, ns, seq_off.data(), seq_tok.data(), seq_soft_vec.data(),
                                    seq_soft.data(), fb_q.empty() ? nullptr : seq_logits.data(),
                                    /*sync=*/!fb_q.empty(), n_remote);
            std::unique_ptr<sgc_kv, int (*)(sgc_kv*)> kv_guard(kv, sgc_kv_release);
            for (uint32_t s = 0; s < ns - n_remote; ++s) prefill_rows += kv->len[s];
            o->kv_pages_peak = std::max<uint64_t>(o->kv_pages_peak, model->pool.live());
            // decode jobs index prefix pages through one block table: every retained wave's pages
            // back to back (generation), or this wave's own
            const int32_t bt_base = retain ? static_cast<int32_t>(gen_bt.size()) : 0;
            if (retain) gen_bt.insert(gen_bt.end(), kv->pages.begin(), kv->pages.end());
            for (uint32_t i = wb; i < we; ++i)
                if (o->prefilled && !is_remote(owned[i])) o->prefilled[owned[i]] = 1;
            if (wv == 0 && n_split > 0) {
                // the split clusters' sealed K/V, owner -> other serving ranks, all layers; both
                // sides walk clusters in ascending index order, so every pair posts its messages
                // in the same order (one grouped exchange per rank)
                std::vector<std::pair<uint32_t, uint32_t>> mine;  // (cluster, wave-local index)
                for (uint32_t i = wb; i < we; ++i)
                    if (is_split(owned[i])) mine.push_back({owned[i], i});
                std::sort(mine.begin(), mine.end());
                // pages differ between ranks: the owner packs a segment's rows of every layer
                // ([L][len][d] for K, then V) into a staging buffer, the receiver unpacks into its pages
                std::vector<sgc::P2P> sends, recvs;
                size_t stage_elems = 0;
                for (auto [ci, i] : mine) stage_elems += 2ull * model->L * kv->len[seq_of[i - wb]] * d;
                bf16* stage = c->buf<bf16>("xfer_stage", std::max<size_t>(1, stage_elems));
                std::vector<std::pair<uint32_t, size_t>> unpack;  // (sequence, staging offset)
                size_t so = 0;
                for (auto [ci, i] : mine) {
                    const uint32_t s = seq_of[i - wb];
                    const size_t n = static_cast<size_t>(model->L) * kv->len[s] * d, bytes = n * sizeof(bf16);
                    bf16 *ks = stage + so, *vs = stage + so + n;
                    if (owner[ci] == me) {
                        sgc::kv_pages_pack(c, ks, model->pool.k, kv->layer_elems(), kv->d_bt + kv->bt_off[s],
                                           static_cast<int>(kv->len[s]), model->L, d, true);
                        sgc::kv_pages_pack(c, vs, model->pool.v, kv->layer_elems(), kv->d_bt + kv->bt_off[s],
                                           static_cast<int>(kv->len[s]), model->L, d, true);
                        for (uint32_t p : peers[ci]) {
                            sends.push_back({ks, bytes, static_cast<int>(p)});
                            sends.push_back({vs, bytes, static_cast<int>(p)});
                            o->prefix_bytes_sent += 2 * bytes;
                        }
                    } else {
                        recvs.push_back({ks, bytes, static_cast<int>(owner[ci])});
                        recvs.push_back({vs, bytes, static_cast<int>(owner[ci])});
                        o->prefix_bytes_received += 2 * bytes;
                        unpack.push_back({s, so});
                    }
                    so += 2 * n;
                }
                comm->exchange(c, sends, recvs);
                for (auto [s, off] : unpack) {
                    const size_t n = static_cast<size_t>(model->L) * kv->len[s] * d;
                    sgc::kv_pages_pack(c, stage + off, model->pool.k, kv->layer_elems(), kv->d_bt + kv->bt_off[s],
                                       static_cast<int>(kv->len[s]), model->L, d, false);
                    sgc::kv_pages_pack(c, stage + off + n, model->pool.v, kv->layer_elems(), kv->d_bt + kv->bt_off[s],
                                       static_cast<int>(kv->len[s]), model->L, d, false);
                }
            }
            {
                cudaEvent_t es = c->event();
                SGC_CUDA_CHECK(cudaEventRecord(es, c->stream));
                ev_seal.push_back(es);
            }
            uint32_t dig0 = 0;
            std::vector<uint32_t> dig_segs;  // the wave's representatives (fallbacks are private)
            if (verify) {  // sealed: digest every representative of the wave (after the exchange)
                dig0 = dig_n;
                for (uint32_t i = wb; i < we; ++i) {
                    dig_slot.push_back({owned[i], dig0 + static_cast<uint32_t>(dig_segs.size())});
                    dig_segs.push_back(seq_of[i - wb]);
                }
                digest_wave(kv, dig_segs, dig0, false);
                dig_n += static_cast<uint32_t>(dig_segs.size());
            }
            const double tw1 = now_ms();
            pf_ms += tw1 - tw0;
            // ---- (5) per-query reuse: every member of the wave's clusters in one cascade pass
            if (!mem_q.empty()) {
                std::vector<uint64_t> mq_off(1, 0), ma_off(1, 0);
                std::vector<int32_t> mq_tok, ma_tok;
                for (uint32_t q : mem_q) {
                    mq_tok.insert(mq_tok.end(), q_tok.begin() + q_off[q], q_tok.begin() + q_off[q + 1]);
                    mq_off.push_back(mq_tok.size());
                    if (ans) ma_tok.insert(ma_tok.end(), a_tok.begin() + a_off[q], a_tok.begin() + a_off[q + 1]);
                    ma_off.push_back(ma_tok.size());
                    extend_rows += q_off[q + 1] - q_off[q];
                }
                const uint32_t nm = static_cast<uint32_t>(mem_q.size());
                if (!gen_on) {
                    // first tokens only: results stay on the stream (pinned host copies), read once
                    // after the last wave
                    ExtendDefer dd;
                    dd.logits = o->logits ? def_lg + static_cast<size_t>(def_n) * SGC_VOCAB : nullptr;
                    dd.first = def_ft + def_n;
                    do_extend(c, model, kv, nm, mem_seg.data(), mq_off.data(), mq_tok.data(),
                              ans ? ma_off.data() : nullptr, ans ? ma_tok.data() : nullptr, b->pointer_bonus,
                              nullptr, nullptr, nullptr, &dd);
                    for (uint32_t k = 0; k < nm; ++k) def_q.push_back(mem_q[dd.order[k]]);
                    def_n += nm;
                }
                std::vector<float> lg(gen_on ? static_cast<size_t>(nm) * SGC_VOCAB : 0);
                std::vector<int32_t> ft(gen_on ? nm : 0);
                if (gen_on)
                    do_extend(c, model, kv, nm, mem_seg.data(), mq_off.data(), mq_tok.data(), ans ? ma_off.data() : nullptr,
                              ans ? ma_tok.data() : nullptr, b->pointer_bonus, lg.data(), ft.data(), &keep);
                for (uint32_t j = 0; gen_on && j < nm; ++j) {
                    const uint32_t q = mem_q[j];
                    if (gen_on) {
                        const int32_t S = static_cast<int32_t>(q_off[q + 1] - q_off[q]);
                        gen_q.push_back(q);
                        gj.pfx_bt.push_back(bt_base + static_cast<int32_t>(kv->bt_off[mem_seg[j]]));
                        gj.pfx_len.push_back(static_cast<int32_t>(kv->len[mem_seg[j]]));
                        gj.q_lo.push_back(keep.q_lo[j]);
                        gj.q_n.push_back(S);
                        gj.pos0.push_back(static_cast<int32_t>(kv->len[mem_seg[j]]) + S);
                        gj.first.push_back(ft[j]);
                        gj.gen_row0.push_back(static_cast<int32_t>(q * gst.max_new));
                        gj.hint.push_back(keep.hint[j]);
                        if (ans) gj.a_tok.insert(gj.a_tok.end(), a_tok.begin() + a_off[q], a_tok.begin() + a_off[q + 1]);
                        gj.a_off.push_back(gj.a_tok.size());
                    }
                    if (o->logits)
                        std::memcpy(o->logits + static_cast<size_t>(q) * SGC_VOCAB, lg.data() + static_cast<size_t>(j) * SGC_VOCAB,
                                    SGC_VOCAB * sizeof(float));
                    if (o->first_token) o->first_token[q] = ft[j];
                    if (o->fallback) o->fallback[q] = 0;
                }
            }
            // fallback first tokens: standalone logits, hint over the own prompt prefix
            for (size_t f = 0; f < fb_q.size(); ++f) {
                const uint32_t q = fb_q[f];
                const uint64_t s = fb_seq[f];
                const float* lg = seq_logits.data() + s * SGC_VOCAB;
                // CopyPointerHint::search_limit of the standalone path (cache_engine.cpp:82-85,
                // :124-129): token_count minus the TRIMMED question = the kept prompt prefix (+ soft)
                const uint64_t full_len = seq_off[s + 1] - seq_off[s];
                const uint64_t limit = std::min<uint64_t>(oo[q + 1] - oo[q], full_len) + (b->soft_prefix ? 1 : 0);
                int target = -1;
                if (ans && a_off[q + 1] > a_off[q]) {
                    std::vector<int32_t> ctxv;
                    if (b->soft_prefix) ctxv.push_back(259);
                    ctxv.insert(ctxv.end(), seq_tok.begin() + seq_off[s], seq_tok.begin() + seq_off[s + 1]);
                    const int32_t* a = a_tok.data() + a_off[q];
                    const uint64_t al = a_off[q + 1] - a_off[q];
                    for (uint64_t st = 0; st + al <= limit && target < 0; ++st)
                        if (std::equal(a, a + al, ctxv.begin() + st)) target = a[0];
                }
                int best = 0;
                float bv = lg[0] + (target == 0 ? b->pointer_bonus : 0.0f);
                for (int v = 1; v < SGC_VOCAB; ++v) {
                    float val = lg[v] + (v == target ? b->pointer_bonus : 0.0f);
                    if (val > bv) {
                        bv = val;
                        best = v;
                    }
                }
                if (o->logits) std::memcpy(o->logits + static_cast<size_t>(q) * SGC_VOCAB, lg, SGC_VOCAB * sizeof(float));
                if (o->first_token) o->first_token[q] = best;
                if (o->fallback) o->fallback[q] = 1;
                fb_flag[q] = 1;
                if (gen_on) {  // standalone decode continues from its own sealed prompt
                    gen_q.push_back(q);
                    gj.pfx_bt.push_back(bt_base + static_cast<int32_t>(kv->bt_off[s]));
                    gj.pfx_len.push_back(static_cast<int32_t>(kv->len[s]));
                    gj.q_lo.push_back(0);
                    gj.q_n.push_back(0);
                    gj.pos0.push_back(static_cast<int32_t>(kv->len[s]));
                    gj.first.push_back(best);
                    gj.gen_row0.push_back(static_cast<int32_t>(q * gst.max_new));
                    gj.hint.push_back(target >= 0 ? 1 : 0);
                    if (ans) gj.a_tok.insert(gj.a_tok.end(), a_tok.begin() + a_off[q], a_tok.begin() + a_off[q + 1]);
                    gj.a_off.push_back(gj.a_tok.size());
                }
            }
            cudaEvent_t e = c->event();
            SGC_CUDA_CHECK(cudaEventRecord(e, c->stream));
            ev_wave.push_back(e);
            ex_ms += now_ms() - tw1;
            // ---- (6) batched greedy decode of the wave's queries (RT)
            if (gen_on && gj.size() > job0) {
                const double td0 = now_ms();
                // new members' state (first token already produced)
                const uint64_t max_seq = lc.max_seq_len;
                for (uint32_t j = job0; j < gj.size(); ++j) {
                    gst.tokens.resize(static_cast<size_t>(j + 1) * gst.max_new, -1);
                    gst.tokens[static_cast<size_t>(j) * gst.max_new] = gj.first[j];
                    gst.count.push_back(1);
                    gst.done.push_back(gst.max_new <= 1 || gj.first[j] == SGC_EOS ||
                                       static_cast<uint64_t>(gj.pos0[j]) + 1 > max_seq);
                    gst.last_ev.push_back(-1);
                }
                std::vector<uint32_t> sel;
                for (uint32_t j = job0; j < gj.size(); ++j) sel.push_back(j);
                const uint32_t min_active = static_cast<uint32_t>((static_cast<uint64_t>(sel.size()) * defer_pct + 99) / 100);
                GenBuffers gb = gen_buffers(c, model, retain ? gen_bt : kv->pages, &keep_all, gj,
                                            static_cast<size_t>(m) * gst.max_new);
                decode_steps(c, model, gb, gj, gst, sel, min_active, b->pointer_bonus);
                dec_ms += now_ms() - td0;
            }
            for (uint32_t j = job0; j < gj.size(); ++j) wave_of_job.push_back(static_cast<int32_t>(wv));
            if (retain) {
                keep_row0 += wave_qr[wv];
                held.push_back(std::move(kv_guard));  // its pages stay until the stragglers are done
                dig_wave.push_back({dig0, dig_segs});
            } else if (verify) {
                digest_wave(kv, dig_segs, dig0, true);  // served: re-check before the pages are released
            }
            wb = we;
        }
        // ---- stragglers of every wave, one shared decode loop (retained K/V)
        if (gen_on && retain) {
            std::vector<uint32_t> rest;
            for (uint32_t j = 0; j < gj.size(); ++j)
                if (!gst.done[j]) rest.push_back(j);
            if (!rest.empty()) {
                const double td0 = now_ms();
                GenBuffers gb = gen_buffers(c, model, gen_bt, &keep_all, gj, static_cast<size_t>(m) * gst.max_new);
                decode_steps(c, model, gb, gj, gst, rest, 0, b->pointer_bonus);
                dec_ms += now_ms() - td0;
            }
        }
        if (verify)
            for (size_t w = 0; w < held.size(); ++w) digest_wave(held[w].get(), dig_wave[w].second, dig_wave[w].first, true);
        if (gen_on) {
            decode_rows = gst.rows;
            for (uint32_t j = 0; j < gj.size(); ++j) {
                const uint32_t q = gen_q[j];
                if (o->tokens)
                    std::memcpy(o->tokens + static_cast<size_t>(q) * max_new, gst.tokens.data() + static_cast<size_t>(j) * max_new,
                                max_new * sizeof(int32_t));
                if (o->n_tokens) o->n_tokens[q] = gst.count[j];
            }
        }
        c->sync();
        check_forward_flags(c);
        if (o->prefix_digest)
            for (uint32_t ci = 0; ci < k; ++ci) o->prefix_digest[ci] = 0;
        if (verify && dig_n) {
            // the sealed prefix must be byte-identical after serving its members (cache_engine.cpp:210)
            std::vector<uint64_t> dg(2 * static_cast<size_t>(dig_cap) + 2);
            sgc::copy_out(c, dg.data(), d_dig, dg.size());
            c->sync();
            for (auto [ci, slot] : dig_slot) {
                if (dg[slot] != dg[slot + dig_cap])
                    fail(SGC_LOGIC, "sealed prefix KV bytes changed while serving members (cluster " +
                                        std::to_string(ci) + ")");
                if (o->prefix_digest) o->prefix_digest[ci] = dg[slot];
            }
        }
        for (uint32_t k = 0; k < def_n; ++k) {
            const uint32_t q = def_q[k];
            if (o->logits)
                std::memcpy(o->logits + static_cast<size_t>(q) * SGC_VOCAB, def_lg + static_cast<size_t>(k) * SGC_VOCAB,
                            SGC_VOCAB * sizeof(float));
            if (o->first_token) o->first_token[q] = def_ft[k];
            if (o->fallback) o->fallback[q] = 0;
        }
        std::vector<float> wave_ms;
        for (cudaEvent_t e : ev_wave) {
            float ms = 0;
            SGC_CUDA_CHECK(cudaEventElapsedTime(&ms, ev_start, e));
            wave_ms.push_back(ms);
            c->event_pool.push_back(e);
        }
        if (o->rt_ms) {
            for (uint32_t q = 0; q < m; ++q) o->rt_ms[q] = -1.0f;
            for (uint32_t j = 0; j < gj.size(); ++j) {
                const uint32_t q = gen_q[j];
                cudaEvent_t e = gst.last_ev[j] >= 0 ? gst.events[gst.last_ev[j]] : ev_wave[wave_of_job[j]];
                float ms = 0.f;
                SGC_CUDA_CHECK(cudaEventElapsedTime(&ms, ev_start, e));
                o->rt_ms[q] = static_cast<float>(t_rep - t_start) + ms;
            }
        }
        for (cudaEvent_t e : gst.events) c->event_pool.push_back(e);
        c->event_pool.push_back(ev_start);
        // TTFT (submission -> first token): batch start to the end of the query's wave; the
        // encode/cluster/represent stages before ev_start are added from the host clock
        const double pre_ms = t_rep - t_start;
        if (o->ttft_ms)
            for (uint32_t q = 0; q < m; ++q)
                o->ttft_ms[q] = wave_of[q] >= 0 ? static_cast<float>(pre_ms + wave_ms[wave_of[q]]) : -1.0f;
        {
            // ledger / report timings from the per-wave events
            std::vector<float> seal_w(ev_seal.size()), start_w(ev_wave_start.size());
            for (size_t w = 0; w < ev_seal.size(); ++w) {
                SGC_CUDA_CHECK(cudaEventElapsedTime(&seal_w[w], ev_start, ev_seal[w]));
                SGC_CUDA_CHECK(cudaEventElapsedTime(&start_w[w], ev_start, ev_wave_start[w]));
            }
            if (o->seal_ms) {
                for (uint32_t ci = 0; ci < k; ++ci) o->seal_ms[ci] = -1.0f;
                uint32_t w0 = 0;
                for (size_t w = 0; w < wave_end.size() && w < seal_w.size(); ++w) {
                    for (uint32_t i = w0; i < wave_end[w]; ++i) o->seal_ms[owned[i]] = static_cast<float>(pre_ms + seal_w[w]);
                    w0 = wave_end[w];
                }
            }
            if (o->ttft_dequeue_ms)
                for (uint32_t q = 0; q < m; ++q)
                    o->ttft_dequeue_ms[q] = wave_of[q] >= 0 ? wave_ms[wave_of[q]] - start_w[wave_of[q]] : -1.0f;
            if (o->pftt_ms)
                for (uint32_t q = 0; q < m; ++q) {
                    const int wq = wave_of[q];
                    if (wq < 0) {
                        o->pftt_ms[q] = -1.0f;
                        continue;
                    }
                    // members: from their wave's extend (= the seal event); fallbacks: from the
                    // wave's prefill start (their standalone prefill)
                    const bool fbq = fb_flag[q] != 0;
                    o->pftt_ms[q] = wave_ms[wq] - (fbq ? start_w[wq] : seal_w[wq]);
                }
            // device-side stage times (the host runs ahead of the GPU without per-wave syncs):
            // prefill = wave start -> seal, extend = seal -> the wave's first tokens
            dev_pf_ms = dev_ex_ms = 0.0;
            for (size_t w = 0; w < seal_w.size() && w < wave_ms.size(); ++w) {
                dev_pf_ms += seal_w[w] - start_w[w];
                dev_ex_ms += wave_ms[w] - seal_w[w];
            }
            for (cudaEvent_t e : ev_seal) c->event_pool.push_back(e);
            for (cudaEvent_t e : ev_wave_start) c->event_pool.push_back(e);
        }
        o->waves = static_cast<uint32_t>(ev_wave.size());
        const double t_pf = t_rep + pf_ms;
        const double t_ext = now_ms();
        host_mark("waves done", t_start);
        (void)t_pf;
        (void)t_ext;
        if (o->embeddings) sgc::copy_out(c, o->embeddings, d_emb, static_cast<size_t>(m) * d);
        if (o->labels) sgc::copy_out(c, o->labels, d_lab, m);
        if (o->merge_left) sgc::copy_out(c, o->merge_left, d_left, m - k);
        if (o->merge_right) sgc::copy_out(c, o->merge_right, d_right, m - k);
        if (o->merge_dist) sgc::copy_out(c, o->merge_dist, d_dist, m - k);
        c->sync();
        if (use_comm) {
            // gather every query's outputs to rank 0: one fixed-size record per
            // served query, in ascending query order per rank (rank 0 knows every rank's list).
            // Every rank passes the same set of optional outputs.
            const size_t gen_w = (gen_on && o->tokens) ? max_new : 0, lg_w = o->logits ? SGC_VOCAB : 0;
            const size_t W = 7 + gen_w + lg_w;  // 4-byte words per record
            auto pack = [&](uint32_t q, uint32_t* r) {
                int32_t ft = o->first_token ? o->first_token[q] : -1;
                std::memcpy(&r[0], &ft, 4);
                r[1] = o->fallback ? o->fallback[q] : 0;
                float f3[3] = {o->ttft_ms ? o->ttft_ms[q] : -1.f, o->pftt_ms ? o->pftt_ms[q] : -1.f,
                               o->rt_ms ? o->rt_ms[q] : -1.f};
                std::memcpy(&r[2], f3, 12);
                r[5] = o->n_tokens ? o->n_tokens[q] : 0;
                const float td = o->ttft_dequeue_ms ? o->ttft_dequeue_ms[q] : -1.f;
                std::memcpy(&r[6], &td, 4);
                if (gen_w) std::memcpy(&r[7], o->tokens + static_cast<size_t>(q) * max_new, gen_w * 4);
                if (lg_w) std::memcpy(&r[7 + gen_w], o->logits + static_cast<size_t>(q) * SGC_VOCAB, lg_w * 4);
            };
            auto unpack = [&](uint32_t q, const uint32_t* r) {
                if (o->first_token) std::memcpy(&o->first_token[q], &r[0], 4);
                if (o->fallback) o->fallback[q] = static_cast<uint8_t>(r[1]);
                float f3[3];
                std::memcpy(f3, &r[2], 12);
                if (o->ttft_ms) o->ttft_ms[q] = f3[0];
                if (o->pftt_ms) o->pftt_ms[q] = f3[1];
                if (o->rt_ms) o->rt_ms[q] = f3[2];
                if (o->n_tokens) o->n_tokens[q] = r[5];
                if (o->ttft_dequeue_ms) std::memcpy(&o->ttft_dequeue_ms[q], &r[6], 4);
                if (gen_w) std::memcpy(o->tokens + static_cast<size_t>(q) * max_new, &r[7], gen_w * 4);
                if (lg_w) std::memcpy(o->logits + static_cast<size_t>(q) * SGC_VOCAB, &r[7 + gen_w], lg_w * 4);
            };
            std::vector<std::vector<uint32_t>> by_rank(world);
            for (uint32_t q = 0; q < m; ++q) by_rank[qrank[q]].push_back(q);
            std::vector<sgc::P2P> sends, recvs;
            std::vector<uint32_t> hbuf;
            uint32_t* dbuf = nullptr;
            if (me != 0 && !by_rank[me].empty()) {
                hbuf.resize(by_rank[me].size() * W);
                for (size_t j = 0; j < by_rank[me].size(); ++j) pack(by_rank[me][j], &hbuf[j * W]);
                dbuf = c->buf<uint32_t>("gather_out", hbuf.size());
                sgc::copy_in(c, dbuf, hbuf.data(), hbuf.size());
                sends.push_back({dbuf, hbuf.size() * 4, 0});
            } else if (me == 0) {
                size_t tot = 0;
                for (int r = 1; r < world; ++r) tot += by_rank[r].size() * W;
                dbuf = c->buf<uint32_t>("gather_out", std::max<size_t>(tot, 1));
                size_t off = 0;
                for (int r = 1; r < world; ++r) {
                    if (!by_rank[r].empty()) recvs.push_back({dbuf + off, by_rank[r].size() * W * 4, r});
                    off += by_rank[r].size() * W;
                }
                hbuf.resize(tot);
            }
            comm->exchange(c, sends, recvs);
            if (me == 0 && !hbuf.empty()) {
                sgc::copy_out(c, hbuf.data(), dbuf, hbuf.size());
                c->sync();
                size_t off = 0;
                for (int r = 1; r < world; ++r)
                    for (uint32_t q : by_rank[r]) {
                        unpack(q, &hbuf[off]);
                        off += W;
                    }
            }
            c->sync();
        }
        o->stage_ms[0] = t_enc - t_start;
        o->stage_ms[1] = t_cl - t_enc;
        o->stage_ms[2] = t_rep - t_cl;
        o->stage_ms[3] = dev_pf_ms;
        o->stage_ms[4] = dev_ex_ms;
        (void)pf_ms;
        (void)ex_ms;
        o->stage_ms[5] = now_ms() - t_start;
        host_mark("end", t_start);
        o->prefill_rows = prefill_rows;
        o->extend_rows = extend_rows;
        o->decode_rows = decode_rows;
        o->stage_ms[6] = dec_ms;
    });
}

#ifdef SGC_ATTN_PROF
}  // extern "C"
namespace sgc {
void attn_prof_read(unsigned long long* out);
void attn_prof_reset();
}
extern "C" {
// debug builds only (make prof): per-CTA phase cycle counters of the tcgen05 attention kernel
int sgc_debug_attn_prof(unsigned long long* out, int reset) {
    if (reset) sgc::attn_prof_reset();
    else sgc::attn_prof_read(out);
    return 0;
}
#endif

int sgc_balance_members(const double* prefill_cost, uint32_t clusters, const uint32_t* labels,
                        const double* member_cost, uint32_t m, int world_size, uint32_t* query_owner,
                        uint32_t* cluster_owner) {
    return guarded([&] {
        if (world_size < 1) fail(SGC_DOMAIN, "world_size must be >= 1");
        std::vector<std::vector<uint32_t>> members(clusters);
        for (uint32_t q = 0; q < m; ++q) {
            if (labels[q] >= clusters) fail(SGC_DOMAIN, "label out of range");
            members[labels[q]].push_back(q);
        }
        std::vector<uint32_t> co;
        std::vector<uint32_t> qo = balance_members(std::vector<double>(prefill_cost, prefill_cost + clusters), members,
                                                   std::vector<double>(member_cost, member_cost + m), world_size, co);
        std::copy(qo.begin(), qo.end(), query_owner);
        if (cluster_owner) std::copy(co.begin(), co.end(), cluster_owner);
    });
}

int sgc_lpt_assign(const double* cost, uint32_t clusters, int world_size, uint32_t* owner) {
    return guarded([&] {
        if (world_size < 1) fail(SGC_DOMAIN, "world_size must be >= 1");
        std::vector<uint32_t> o = lpt_assign(std::vector<double>(cost, cost + clusters), world_size);
        std::copy(o.begin(), o.end(), owner);
    });
}

int sgc_gemm_bf16(sgc_ctx* ctx, const void* a, const void* b, void* d, uint32_t M, uint32_t N, uint32_t K, int epi) {
    return guarded([&] {
        sgc::GemmEpi e;
        e.splitk_ok = (epi & 256) != 0;  // decode-step GEMM: stream-K / split-K allowed
        epi &= 255;
        e.mode = epi;
        e.out = d;
        e.ldo = static_cast<int>(N);
        if (epi == sgc::EPI_QKV) fail(SGC_DOMAIN, "QKV epilogue is internal");
        sgc::gemm_bf16(current(&ctx->c), a, b, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), e);
        ctx->c.sync();
    });
}

int sgc_attention_bf16(sgc_ctx* ctx, const void* q, const void* k_pfx, const void* v_pfx,
                       uint32_t pfx_rows, const void* k_loc, const void* v_loc, const int32_t* seg_lo,
                       const int32_t* work, uint32_t n_work, uint32_t rows, uint32_t d, uint32_t heads,
                       void* out) {
    return guarded([&] {
        if (heads == 0 || d % heads != 0) fail(SGC_DOMAIN, "attention: d must be a multiple of heads");
        const int hd = static_cast<int>(d / heads);
        const int tile = attn_tile(hd);
        Ctx* c = current(&ctx->c);
        std::vector<sgc::AttnWork> w(n_work);
        for (uint32_t i = 0; i < n_work; ++i) {
            w[i] = {work[4 * i], work[4 * i + 1], work[4 * i + 2], work[4 * i + 3], -1};  // contiguous rows
            if (w[i].nrows < 1 || w[i].nrows > tile || w[i].row0 < 0 ||
                static_cast<uint32_t>(w[i].row0 + w[i].nrows) > rows ||
                static_cast<uint32_t>(w[i].pfx_off + w[i].pfx_len) > pfx_rows)
                fail(SGC_DOMAIN, "attention: work unit out of range");
        }
        sgc::AttnWork* d_work = c->buf<sgc::AttnWork>("dbg_attn_work", n_work);
        sgc::copy_in_staged(c, d_work, w.data(), n_work);
        sgc::AttnParams ap;
        ap.q = static_cast<const bf16*>(q);
        ap.out = static_cast<bf16*>(out);
        ap.k_pfx = static_cast<const bf16*>(k_pfx);
        ap.v_pfx = static_cast<const bf16*>(v_pfx);
        ap.k_loc = static_cast<const bf16*>(k_loc);
        ap.v_loc = static_cast<const bf16*>(v_loc);
        ap.loc_kv0 = 0;
        ap.seg_lo = seg_lo;
        ap.work = d_work;
        ap.d = static_cast<int>(d);
        ap.scale = 1.0f / std::sqrt(static_cast<float>(hd));
        if (sgc::attention_tc_supported(hd))
            sgc::cascade_attention_tc(c, ap, static_cast<int>(n_work), static_cast<int>(heads), hd,
                                      static_cast<int>(rows), static_cast<int>(std::max(1u, pfx_rows)),
                                      static_cast<int>(rows));
        else
            sgc::cascade_attention(c, ap, static_cast<int>(n_work), static_cast<int>(heads), hd);
        c->sync();
    });
}

int sgc_set_option(sgc_ctx* ctx, const char* name, int64_t value) {
    return guarded([&] {
        if (std::string(name) == "gemm_pairs") sgc::gemm_set_pairs(value != 0);
        else if (std::string(name) == "gemm_raster") sgc::gemm_set_raster(static_cast<int>(value));
        else if (std::string(name) == "gemm_streamk") sgc::gemm_set_streamk(static_cast<int>(value));
        else if (std::string(name) == "agglomerate_global") sgc::agglomerate_set_global(value != 0);
        else if (std::string(name) == "attn_split") sgc::attention_set_split(value != 0);
        else if (std::string(name) == "attn_kernel") sgc::attention_set_kernel(static_cast<int>(value));
        else if (std::string(name) == "attn_kernel_partial") sgc::attention_set_kernel_partial(static_cast<int>(value));
        else if (std::string(name) == "gnn_tile") ctx->c.gnn_tile = static_cast<int>(value);
        else if (std::string(name) == "gnn_dedup") ctx->c.gnn_dedup = value != 0 ? 1 : 0;
        else if (std::string(name) == "decode_defer_pct") ctx->c.decode_defer_pct = static_cast<uint32_t>(std::max<int64_t>(0, value));
        else fail(SGC_DOMAIN, std::string("unknown option ") + name);
    });
}

int sgc_gnn_stats(const sgc_ctx* ctx, uint64_t* state_rows, uint64_t* node_instances) {
    if (state_rows) *state_rows = ctx->c.gnn_state_rows;
    if (node_instances) *node_instances = ctx->c.gnn_node_instances;
    return SGC_OK;
}

int sgc_probe_fp64_tflops(sgc_ctx* ctx, double* tflops) {
    return guarded([&] {
        sgc::Ctx* c = current(&ctx->c);
        *tflops = std::max(sgc::fp64_probe_tflops(c), sgc::dmma_probe_tflops(c));
    });
}

int sgc_set_timing(sgc_ctx* ctx, int enable) {
    return guarded([&] {
        ctx->c.sync();
        ctx->c.resolve_timings();  // recycle the pending pairs; the totals restart
        ctx->c.timing = enable != 0;
        ctx->c.timings.clear();
    });
}

int sgc_get_timing(sgc_ctx* ctx, const char* kernel, double* total_ms, uint64_t* launches) {
    return guarded([&] {
        ctx->c.sync();
        ctx->c.resolve_timings();
        auto it = ctx->c.timings.find(kernel);
        *total_ms = it == ctx->c.timings.end() ? 0.0 : it->second.ms;
        *launches = it == ctx->c.timings.end() ? 0 : it->second.launches;
    });
}

}  // extern "C"

namespace sgc {
void trace_launch(Ctx* c, const char* file, int line) {
    std::fprintf(stderr, "[sgc trace] launch #%llu %s:%d ...", static_cast<unsigned long long>(c->launches),
                 file, line);
    std::fflush(stderr);
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e = cudaStreamSynchronize(c->stream);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, " %s %.3f ms\n", cudaGetErrorString(e), ms);
    std::fflush(stderr);
}
}  // namespace sgc
