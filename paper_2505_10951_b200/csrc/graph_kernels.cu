// graph_kernels.cu -- text features (TextEncoder::embed), representative union
// (merge_subgraphs) and prompt construction (build_prompt + tokenize) on the device.
#include <cstring>

#include "common.cuh"
#include "graph_kernels.cuh"

namespace sgc {
namespace {

// encoders.cpp:57-93 -- one CTA per graph element. acc[k] sums the element's token columns
// in token order (double, exact as the reference); the norm is a sequential sum over k
// by one thread, so the float result is bit-identical to the reference.
__global__ void text_feature_kernel(float* out, const uint32_t* bucket, const int8_t* sign,
                                    const uint64_t* tok_off, int n_elem, const float* proj_t,
                                    int dim) {
    extern __shared__ double acc[];
    __shared__ double norm_s;
    const int e = blockIdx.x;
    if (e >= n_elem) return;
    const uint64_t t0 = tok_off[e], t1 = tok_off[e + 1];
    for (int k = threadIdx.x; k < dim; k += blockDim.x) {
        double a = 0.0;
        for (uint64_t t = t0; t < t1; ++t) {
            double s = sign[t] > 0 ? 1.0 : -1.0;
            a = __dadd_rn(a, __dmul_rn(s, static_cast<double>(proj_t[static_cast<size_t>(bucket[t]) * dim + k])));
        }
        acc[k] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double n = 0.0;
        for (int k = 0; k < dim; ++k) n = __dadd_rn(n, __dmul_rn(acc[k], acc[k]));
        norm_s = __dsqrt_rn(n);
    }
    __syncthreads();
    const double nrm = norm_s;
    float* o = out + static_cast<size_t>(e) * dim;
    for (int k = threadIdx.x; k < dim; k += blockDim.x)
        o[k] = (t1 > t0 && nrm > 0.0) ? static_cast<float>(__ddiv_rn(acc[k], nrm)) : 0.0f;
}

// node ids -> dense node indices (ids ascending in the graph), -1 when absent
__global__ void node_index_kernel(int32_t* out, const uint32_t* ids, uint64_t n,
                                  const uint32_t* sorted_ids, int n_nodes) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t id = ids[i];
        int lo = 0, hi = n_nodes;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (sorted_ids[mid] < id) lo = mid + 1;
            else hi = mid;
        }
        out[i] = (lo < n_nodes && sorted_ids[lo] == id) ? lo : -1;
    }
}

__device__ __forceinline__ int block_excl_scan(int v, int* tmp) {
    // blockDim.x <= 1024, warp-shuffle scan
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffff, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) tmp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < (int)(blockDim.x / 32) ? tmp[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffff, w, o);
            if (lane >= o) w += y;
        }
        tmp[lane] = w;  // inclusive per-warp totals
    }
    __syncthreads();
    int base = warp > 0 ? tmp[warp - 1] : 0;
    int total = tmp[blockDim.x / 32 - 1];
    __syncthreads();
    tmp[32] = total;
    return base + x - v;
}

// merge_subgraphs (graph_store.cpp:223-235) + the prefix side of build_prompt
// (cache_engine.cpp:43-62): one CTA per cluster. Bitmap union with atomicOr, ascending
// compaction by block scan (== std::set order), then the closed-form truncation cut.
__global__ void __launch_bounds__(1024)
    union_prompt_kernel(const int32_t* sub_nodes, const uint64_t* sub_node_off,
                        const uint32_t* sub_edges, const uint64_t* sub_edge_off,
                        const uint32_t* members, const uint64_t* member_off,  // per cluster
                        uint32_t* node_bm, uint32_t* edge_bm, int node_words, int edge_words,
                        const uint32_t* node_row_len, const uint32_t* edge_row_len,
                        int n_nodes, int n_edges, uint32_t budget_bytes, uint32_t base_bytes,
                        uint32_t* sel_nodes, uint32_t* sel_edges,    // [c x n_nodes], [c x n_edges]
                        uint32_t* node_pre, uint32_t* edge_pre,      // exclusive row byte offsets
                        uint32_t* stats /* [c x 6]: n_sel, e_sel, kn, ke, node_bytes, edge_bytes */,
                        int* status) {
    __shared__ int tmp[33];
    const int k = blockIdx.x;
    uint32_t* nbm = node_bm + static_cast<size_t>(k) * node_words;
    uint32_t* ebm = edge_bm + static_cast<size_t>(k) * edge_words;
    for (int i = threadIdx.x; i < node_words; i += blockDim.x) nbm[i] = 0;
    for (int i = threadIdx.x; i < edge_words; i += blockDim.x) ebm[i] = 0;
    __syncthreads();
    for (uint64_t mi = member_off[k]; mi < member_off[k + 1]; ++mi) {
        const uint32_t q = members[mi];
        for (uint64_t i = sub_node_off[q] + threadIdx.x; i < sub_node_off[q + 1]; i += blockDim.x) {
            int idx = sub_nodes[i];
            if (idx < 0) {
                atomicExch(status, SGC_INTEGRITY);
                continue;
            }
            atomicOr(&nbm[idx >> 5], 1u << (idx & 31));
        }
        for (uint64_t i = sub_edge_off[q] + threadIdx.x; i < sub_edge_off[q + 1]; i += blockDim.x) {
            uint32_t idx = sub_edges[i];
            if (idx >= static_cast<uint32_t>(n_edges)) {
                atomicExch(status, SGC_INTEGRITY);
                continue;
            }
            atomicOr(&ebm[idx >> 5], 1u << (idx & 31));
        }
    }
    __syncthreads();
    // compaction in ascending order, words processed in chunks of blockDim.x
    uint32_t* sn = sel_nodes + static_cast<size_t>(k) * n_nodes;
    uint32_t* se = sel_edges + static_cast<size_t>(k) * n_edges;
    int n_sel = 0;
    for (int w0 = 0; w0 < node_words; w0 += blockDim.x) {
        int w = w0 + threadIdx.x;
        uint32_t bits = w < node_words ? nbm[w] : 0u;
        int off = n_sel + block_excl_scan(__popc(bits), tmp);
        int tot = tmp[32];
        while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            sn[off++] = w * 32 + b;
        }
        n_sel += tot;
        __syncthreads();
    }
    int e_sel = 0;
    for (int w0 = 0; w0 < edge_words; w0 += blockDim.x) {
        int w = w0 + threadIdx.x;
        uint32_t bits = w < edge_words ? ebm[w] : 0u;
        int off = e_sel + block_excl_scan(__popc(bits), tmp);
        int tot = tmp[32];
        while (bits) {
            int b = __ffs(bits) - 1;
            bits &= bits - 1;
            se[off++] = w * 32 + b;
        }
        e_sel += tot;
        __syncthreads();
    }
    __syncthreads();
    // row byte prefix sums (row bytes + '\n'), exclusive
    uint32_t* np = node_pre + static_cast<size_t>(k) * (n_nodes + 1);
    uint32_t* ep = edge_pre + static_cast<size_t>(k) * (n_edges + 1);
    int run = 0;
    for (int i0 = 0; i0 < n_sel; i0 += blockDim.x) {
        int i = i0 + threadIdx.x;
        int v = i < n_sel ? static_cast<int>(node_row_len[sn[i]]) + 1 : 0;
        int off = run + block_excl_scan(v, tmp);
        if (i < n_sel) np[i] = off;
        run += tmp[32];
        __syncthreads();
    }
    const uint32_t node_bytes = run;
    if (threadIdx.x == 0) np[n_sel] = node_bytes;
    run = 0;
    for (int i0 = 0; i0 < e_sel; i0 += blockDim.x) {
        int i = i0 + threadIdx.x;
        int v = i < e_sel ? static_cast<int>(edge_row_len[se[i]]) + 1 : 0;
        int off = run + block_excl_scan(v, tmp);
        if (i < e_sel) ep[i] = off;
        run += tmp[32];
        __syncthreads();
    }
    const uint32_t edge_bytes = run;
    if (threadIdx.x == 0) ep[e_sel] = edge_bytes;
    __syncthreads();
    // truncation (cache_engine.cpp:55-57): keep_edges = #{e >= 1 : total(all nodes, e) <= budget},
    // then keep_nodes = #{n >= 1 : total(n, keep_edges) <= budget}; both predicates are monotone.
    __shared__ int cnt_e, cnt_n;
    if (threadIdx.x == 0) {
        cnt_e = 0;
        cnt_n = 0;
    }
    __syncthreads();
    for (int e = 1 + threadIdx.x; e <= e_sel; e += blockDim.x)
        if (base_bytes + node_bytes + ep[e] <= budget_bytes) atomicAdd(&cnt_e, 1);
    __syncthreads();
    const int ke = cnt_e;
    const uint32_t kept_edge_bytes = ep[ke];
    for (int n = 1 + threadIdx.x; n <= n_sel; n += blockDim.x)
        if (base_bytes + np[n] + kept_edge_bytes <= budget_bytes) atomicAdd(&cnt_n, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int kn = cnt_n;
        uint32_t total = base_bytes + np[kn] + kept_edge_bytes;
        if (total > budget_bytes) atomicExch(status, SGC_CAPACITY);
        uint32_t* st = stats + static_cast<size_t>(k) * 6;
        st[0] = n_sel;
        st[1] = e_sel;
        st[2] = kn;
        st[3] = ke;
        st[4] = np[kn];
        st[5] = kept_edge_bytes;
    }
}

// prompt headers travel as a by-value kernel parameter (no per-device constant state: a
// context on another device launches with the same bytes)
struct PromptHeaders {
    char head[128];  // header + node csv header + '\n'
    char edge[32];   // edge csv header + '\n'
};

// tokenize (tokenizer.cpp:5-11) of the truncated prompt: BOS + bytes, as int32 tokens.
__global__ void prompt_gather_kernel(int32_t* tokens, const uint64_t* tok_off,
                                     const uint32_t* stats, const uint32_t* sel_nodes,
                                     const uint32_t* sel_edges, const uint32_t* node_pre,
                                     const uint32_t* edge_pre, const char* node_text,
                                     const uint64_t* node_text_off, const char* edge_text,
                                     const uint64_t* edge_text_off, int n_nodes, int n_edges,
                                     int head_len, int ehead_len, const PromptHeaders hdr) {
    const int k = blockIdx.y;
    const uint32_t* st = stats + static_cast<size_t>(k) * 6;
    const uint32_t kn = st[2], ke = st[3], nb = st[4], eb = st[5];
    const uint64_t P = tok_off[k + 1] - tok_off[k];
    int32_t* out = tokens + tok_off[k];
    const uint32_t* sn = sel_nodes + static_cast<size_t>(k) * n_nodes;
    const uint32_t* se = sel_edges + static_cast<size_t>(k) * n_edges;
    const uint32_t* np = node_pre + static_cast<size_t>(k) * (n_nodes + 1);
    const uint32_t* ep = edge_pre + static_cast<size_t>(k) * (n_edges + 1);
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < P;
         j += (uint64_t)gridDim.x * blockDim.x) {
        if (j == 0) {
            out[0] = 256;  // BOS
            continue;
        }
        uint32_t q = static_cast<uint32_t>(j - 1);
        unsigned char ch;
        if (q < static_cast<uint32_t>(head_len)) {
            ch = hdr.head[q];
        } else if ((q -= head_len) < nb) {
            int lo = 0, hi = kn - 1;  // last row with np[row] <= q
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (np[mid] <= q) lo = mid;
                else hi = mid - 1;
            }
            uint32_t o = q - np[lo];
            uint32_t node = sn[lo];
            uint64_t len = node_text_off[node + 1] - node_text_off[node];
            ch = o < len ? node_text[node_text_off[node] + o] : '\n';
        } else if ((q -= nb) < static_cast<uint32_t>(ehead_len)) {
            ch = hdr.edge[q];
        } else {
            q -= ehead_len;
            int lo = 0, hi = ke - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (ep[mid] <= q) lo = mid;
                else hi = mid - 1;
            }
            uint32_t o = q - ep[lo];
            uint32_t edge = se[lo];
            uint64_t len = edge_text_off[edge + 1] - edge_text_off[edge];
            ch = o < len ? edge_text[edge_text_off[edge] + o] : '\n';
        }
        out[j] = ch;
    }
}

}  // namespace

void text_features(Ctx* c, float* out, const uint32_t* bucket, const int8_t* sign,
                   const uint64_t* tok_off, int n_elem, const float* proj_t, int dim) {
    if (n_elem <= 0) return;
    size_t smem = static_cast<size_t>(dim) * sizeof(double);
    if (smem > 48 * 1024)
        SGC_CUDA_CHECK(cudaFuncSetAttribute(text_feature_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    Ctx::Timed timer(c, "text_features");
    text_feature_kernel<<<n_elem, 256, smem, c->stream>>>(out, bucket, sign, tok_off, n_elem, proj_t, dim);
    SGC_LAUNCH_CHECK(c);
}

void node_index(Ctx* c, int32_t* out, const uint32_t* ids, uint64_t n, const uint32_t* sorted_ids,
                int n_nodes) {
    if (!n) return;
    unsigned g = ceil_div(n, 256);
    node_index_kernel<<<g < 4096 ? g : 4096, 256, 0, c->stream>>>(out, ids, n, sorted_ids, n_nodes);
    SGC_LAUNCH_CHECK(c);
}

void union_prompt(Ctx* c, const UnionArgs& a) {
    Ctx::Timed timer(c, "union_prompt");
    union_prompt_kernel<<<a.clusters, 1024, 0, c->stream>>>(
        a.sub_nodes, a.sub_node_off, a.sub_edges, a.sub_edge_off, a.members, a.member_off,
        a.node_bm, a.edge_bm, a.node_words, a.edge_words, a.node_row_len, a.edge_row_len,
        a.n_nodes, a.n_edges, a.budget_bytes, a.base_bytes, a.sel_nodes, a.sel_edges, a.node_pre,
        a.edge_pre, a.stats, a.status);
    SGC_LAUNCH_CHECK(c);
}

void prompt_gather(Ctx* c, const GatherArgs& a) {
    PromptHeaders hdr{};
    if (a.head_len > static_cast<int>(sizeof(hdr.head)) || a.ehead_len > static_cast<int>(sizeof(hdr.edge)))
        fail(SGC_LOGIC, "prompt header too long");
    std::memcpy(hdr.head, a.head, a.head_len);
    std::memcpy(hdr.edge, a.ehead, a.ehead_len);
    Ctx::Timed timer(c, "prompt_gather");
    dim3 grid(ceil_div(a.max_tokens, 256), a.clusters);
    prompt_gather_kernel<<<grid, 256, 0, c->stream>>>(
        a.tokens, a.tok_off, a.stats, a.sel_nodes, a.sel_edges, a.node_pre, a.edge_pre, a.node_text,
        a.node_text_off, a.edge_text, a.edge_text_off, a.n_nodes, a.n_edges, a.head_len, a.ehead_len, hdr);
    SGC_LAUNCH_CHECK(c);
}

// ---- retrieval scoring ----------------------------------------------------------------------
namespace {
constexpr int RT = 16;   // pairs per CTA side
constexpr int RK = 64;   // feature chunk staged in shared memory

// one thread per (i, j) pair of a 16 x 16 tile; the feature axis is walked in order (chunks of
// 64 staged in smem), so each sum is the reference's sequential double accumulation
__global__ void __launch_bounds__(256) retrieval_dot_kernel(double* dot, const float* A, int na, const float* B,
                                                            int nb, int d) {
    __shared__ float As[RT][RK + 1], Bs[RT][RK + 1];
    const int i0 = blockIdx.y * RT, j0 = blockIdx.x * RT;
    const int ti = threadIdx.x / RT, tj = threadIdx.x % RT;
    double acc = 0.0;
    for (int k0 = 0; k0 < d; k0 += RK) {
        const int kc = min(RK, d - k0);
        for (int t = threadIdx.x; t < RT * RK; t += blockDim.x) {
            const int r = t / RK, k = t % RK;
            As[r][k] = (i0 + r < na && k < kc) ? A[static_cast<size_t>(i0 + r) * d + k0 + k] : 0.f;
            Bs[r][k] = (j0 + r < nb && k < kc) ? B[static_cast<size_t>(j0 + r) * d + k0 + k] : 0.f;
        }
        __syncthreads();
        for (int k = 0; k < kc; ++k)
            acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(As[ti][k]), static_cast<double>(Bs[tj][k])));
        __syncthreads();
    }
    if (i0 + ti < na && j0 + tj < nb) dot[static_cast<size_t>(i0 + ti) * nb + j0 + tj] = acc;
}

__global__ void sq_norm_kernel(double* out, const float* A, int n, int d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    const float* a = A + static_cast<size_t>(i) * d;
    for (int k = 0; k < d; ++k) s = __dadd_rn(s, __dmul_rn(static_cast<double>(a[k]), static_cast<double>(a[k])));
    out[i] = s;
}

// retrieval.cpp:175-189: pooled = mean of the ego net's node then edge attribute embeddings
// (double accumulation in member order, one division, cast to float)
__global__ void ego_pool_kernel(float* pooled, const float* feat, const uint32_t* mem_off,
                                const uint32_t* mem_idx, int d) {
    const int e = blockIdx.x;
    const uint32_t m0 = mem_off[e], m1 = mem_off[e + 1];
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double s = 0.0;
        for (uint32_t t = m0; t < m1; ++t) s = __dadd_rn(s, static_cast<double>(feat[static_cast<size_t>(mem_idx[t]) * d + k]));
        pooled[static_cast<size_t>(e) * d + k] = static_cast<float>(__ddiv_rn(s, static_cast<double>(m1 - m0)));
    }
}

__global__ void pair_dot_kernel(double* dot, double* sq, const float* q, const int32_t* qi, const float* p,
                                int n, int d) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const float* a = q + static_cast<size_t>(qi[e]) * d;
    const float* b = p + static_cast<size_t>(e) * d;
    double s = 0.0, nb2 = 0.0;
    for (int k = 0; k < d; ++k) {
        s = __dadd_rn(s, __dmul_rn(static_cast<double>(a[k]), static_cast<double>(b[k])));
        nb2 = __dadd_rn(nb2, __dmul_rn(static_cast<double>(b[k]), static_cast<double>(b[k])));
    }
    dot[e] = s;
    sq[e] = nb2;
}
}  // namespace

void retrieval_dots(Ctx* c, double* dot, double* sq_a, double* sq_b, const float* A, int na, const float* B,
                    int nb, int d) {
    if (na <= 0 || nb <= 0) return;
    Ctx::Timed timer(c, "retrieval");
    retrieval_dot_kernel<<<dim3(ceil_div(nb, RT), ceil_div(na, RT)), 256, 0, c->stream>>>(dot, A, na, B, nb, d);
    SGC_LAUNCH_CHECK(c);
    sq_norm_kernel<<<ceil_div(na, 128), 128, 0, c->stream>>>(sq_a, A, na, d);
    SGC_LAUNCH_CHECK(c);
    sq_norm_kernel<<<ceil_div(nb, 128), 128, 0, c->stream>>>(sq_b, B, nb, d);
    SGC_LAUNCH_CHECK(c);
}

void ego_pool_dots(Ctx* c, float* pooled, double* pair_dot, double* pair_sq, const float* feat,
                   const uint32_t* mem_off, const uint32_t* mem_idx, const float* q, const int32_t* qi,
                   int n_ego, int d) {
    if (n_ego <= 0) return;
    Ctx::Timed timer(c, "retrieval");
    ego_pool_kernel<<<n_ego, 128, 0, c->stream>>>(pooled, feat, mem_off, mem_idx, d);
    SGC_LAUNCH_CHECK(c);
    pair_dot_kernel<<<ceil_div(n_ego, 128), 128, 0, c->stream>>>(pair_dot, pair_sq, q, qi, pooled, n_ego, d);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace sgc
