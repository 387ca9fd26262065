// lm_kernels.cu -- ToyLm support kernels: seeded weight generation, embedding gather,
// RMSNorm (no gain), fp32 head + RMSNorm for the logit rows, copy-pointer search and the
// biased greedy argmax of the first token.
#include "common.cuh"
#include "lm_kernels.cuh"
#include "rng.cuh"

namespace sgc {
namespace {

__global__ void gen_uniform_f32(float* out, uint64_t n, uint64_t state0, float lo, float hi) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = uniform_at(state0, i, lo, hi);
}

__global__ void gen_uniform_bf16(__nv_bfloat16* out, uint64_t n, uint64_t state0, float lo,
                                 float hi) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = __float2bfloat16_rn(uniform_at(state0, i, lo, hi));
}

// text projection [dim x 4096] (encoders.cpp:50-55) stored transposed [4096 x dim]
__global__ void gen_projection_t(float* out_t, uint32_t dim, uint64_t state0) {
    uint64_t n = (uint64_t)dim * 4096;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = i / 4096, b = i % 4096;
        out_t[b * dim + k] = uniform_at(state0, i, -1.0f, 1.0f);
    }
}

// embed_tokens (lm_core.cpp:163-173) + soft slot (:308-320): x[r] = tok_emb[id] or soft[s]
// (+ the first layer's fused RMSNorm inputs: bf16(x) and the row's sum of squares)
__global__ void embed_kernel(float* x, const int32_t* tokens, const float* tok_emb,
                             const float* soft, const int32_t* soft_idx, int d, int rows,
                             int* bad, __nv_bfloat16* xb, float* ss_out) {
    int r = blockIdx.x;
    if (r >= rows) return;
    int id = tokens[r];
    const float* src;
    if (id == 259 && soft_idx && soft_idx[r] >= 0) {
        src = soft + static_cast<size_t>(soft_idx[r]) * d;
    } else {
        if (id < 0 || id >= SGC_VOCAB) {
            if (threadIdx.x == 0) atomicExch(bad, 1);
            src = tok_emb;  // keep the block convergent; the batch fails after the forward
        } else {
            src = tok_emb + static_cast<size_t>(id) * d;
        }
    }
    float ss = 0.f;
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
        const float4 v = reinterpret_cast<const float4*>(src)[i];
        reinterpret_cast<float4*>(x + static_cast<size_t>(r) * d)[i] = v;
        if (xb) {
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
            __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&a);
            pk.y = *reinterpret_cast<uint32_t*>(&b);
            reinterpret_cast<uint2*>(xb + static_cast<size_t>(r) * d)[i] = pk;
        }
    }
    if (!xb) return;
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
        ss_out[r] = t;
    }
}

// rmsnorm (lm_core.cpp:26-31): out = bf16(x / sqrt(mean(x^2) + 1e-5)), one CTA per row
__global__ void rmsnorm_bf16_kernel(__nv_bfloat16* out, const float* x, int d, int rows) {
    int r = blockIdx.x;
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(r) * d);
    float ss = 0.f;
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
        float4 v = xr[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    __shared__ float red[32];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffff, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const float inv = 1.0f / sqrtf(red[0] / static_cast<float>(d) + 1e-5f);
    uint2* o2 = reinterpret_cast<uint2*>(out + static_cast<size_t>(r) * d);
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
        float4 v = xr[i];
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv, v.y * inv);
        __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv, v.w * inv);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&a);
        w.y = *reinterpret_cast<uint32_t*>(&b);
        o2[i] = w;
    }
}

// final rmsnorm + fp32 head (lm_core.cpp:288-295) for selected rows. CTA = 16 rows x all
// vocab; the head is stored transposed [d x 260] so a thread per vocab id reads coalesced.
constexpr int kHeadRows = 16;
constexpr int kHeadChunk = 512;  // K slice per CTA: the split is a function of d only, so the
                                 // summation order (and the logits, bit for bit) never depends
                                 // on how many rows a call carries

// 1 / sqrt(mean(x^2) + 1e-5) of the logit rows (the final RMSNorm, lm_core.cpp:285-296)
__global__ void head_norm_kernel(float* inv, const float* x, const int32_t* rows, int n, int d) {
    const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (r >= n) return;
    const float* xr = x + static_cast<size_t>(rows[r]) * d;
    float ss = 0.f;
    for (int i = lane; i < d; i += 32) ss += xr[i] * xr[i];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
    if (lane == 0) inv[r] = 1.0f / sqrtf(ss / static_cast<float>(d) + 1e-5f);
}

// partial[ks][r][v] = sum over k in slice ks of head[v][k] * x[row r][k] * inv[r]
__global__ void __launch_bounds__(288) head_kernel(float* partial, const float* x, const float* inv,
                                                   const int32_t* rows, int n, const float* head_t,
                                                   int d) {
    __shared__ float xs[kHeadRows][kHeadChunk];
    const int r0 = blockIdx.x * kHeadRows, k0 = blockIdx.y * kHeadChunk;
    const int kc = min(kHeadChunk, d - k0);
    for (int i = threadIdx.x; i < kHeadRows * kc; i += blockDim.x) {
        const int rr = i / kc, k = i % kc;
        xs[rr][k] = r0 + rr < n ? x[static_cast<size_t>(rows[r0 + rr]) * d + k0 + k] * inv[r0 + rr] : 0.f;
    }
    __syncthreads();
    const int v = threadIdx.x;  // vocab id (260 of 288 threads active)
    if (v >= SGC_VOCAB) return;
    float acc[kHeadRows];
#pragma unroll
    for (int i = 0; i < kHeadRows; ++i) acc[i] = 0.f;
    for (int k = 0; k < kc; ++k) {
        const float w = head_t[static_cast<size_t>(k0 + k) * SGC_VOCAB + v];
#pragma unroll
        for (int i = 0; i < kHeadRows; ++i) acc[i] = fmaf(xs[i][k], w, acc[i]);
    }
    float* out = partial + static_cast<size_t>(blockIdx.y) * n * SGC_VOCAB;
    for (int i = 0; i < kHeadRows; ++i)
        if (r0 + i < n) out[static_cast<size_t>(r0 + i) * SGC_VOCAB + v] = acc[i];
}

// fixed-order reduction of the K slices
__global__ void head_reduce_kernel(float* logits, const float* partial, int n, int splits) {
    const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    const size_t total = static_cast<size_t>(n) * SGC_VOCAB;
    if (i >= total) return;
    float s = partial[i];
    for (int k = 1; k < splits; ++k) s += partial[k * total + i];
    logits[i] = s;
}

// copy pointer (lm_core.cpp:360-374) + first greedy step (:379-385): one CTA per member.
// context = the member's sealed prefix tokens; search_limit = prefix length.
// greedy_argmax (lm_core.cpp:39-50) over one row of logits with bonus on `target`, ties toward
// the lowest id; whole block cooperates, result valid in thread 0
__device__ int block_biased_argmax(const float* lg, int target, float bonus) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = threadIdx.x; v < SGC_VOCAB; v += blockDim.x) {
        float val = lg[v] + (v == target ? bonus : 0.0f);
        if (val > best || (val == best && v < bi)) {
            best = val;
            bi = v;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        float ob = __shfl_xor_sync(0xffffffff, best, o);
        int oi = __shfl_xor_sync(0xffffffff, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    __shared__ float sb[32];
    __shared__ int si[32];
    if (threadIdx.x % 32 == 0) {
        sb[threadIdx.x / 32] = best;
        si[threadIdx.x / 32] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < blockDim.x / 32; ++w)
            if (sb[w] > best || (sb[w] == best && si[w] < bi)) {
                best = sb[w];
                bi = si[w];
            }
    }
    return bi;
}

// first decode step (lm_core.cpp:356-386): the copy pointer fires when the answer occurs in the
// sealed prefix (search_limit = prefix length); hint_out (optional) records it for later steps
__global__ void first_token_kernel(int32_t* first, int8_t* hint_out, const float* logits, int n,
                                   const int32_t* ctx_tokens, const uint64_t* ctx_off,
                                   const uint32_t* member_ctx, const int32_t* ans,
                                   const uint64_t* ans_off, float bonus) {
    const int j = blockIdx.x;
    if (j >= n) return;
    __shared__ int found;
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    int alen = 0;
    const int32_t* a = nullptr;
    if (ans_off) {
        alen = static_cast<int>(ans_off[j + 1] - ans_off[j]);
        a = ans + ans_off[j];
    }
    if (alen > 0) {
        const uint32_t cidx = member_ctx[j];
        const int32_t* c = ctx_tokens + ctx_off[cidx];
        const int clen = static_cast<int>(ctx_off[cidx + 1] - ctx_off[cidx]);
        for (int s = threadIdx.x; s + alen <= clen; s += blockDim.x) {
            int i = 0;
            while (i < alen && c[s + i] == a[i]) ++i;
            if (i == alen) found = 1;
        }
    }
    __syncthreads();
    const int target = found ? a[0] : -1;
    const int bi = block_biased_argmax(logits + static_cast<size_t>(j) * SGC_VOCAB, target, bonus);
    if (threadIdx.x == 0) {
        first[j] = bi;
        if (hint_out) hint_out[j] = static_cast<int8_t>(found);
    }
}

// decode step t >= 1 (lm_core.cpp:376-381): bias target answer[t] while t < |answer|, then EOS
__global__ void step_token_kernel(int32_t* tok, const float* logits, int n, const int8_t* hint,
                                  const int32_t* ans, const uint64_t* ans_off, const int32_t* member,
                                  const int32_t* step, float bonus) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const int j = member[r], t = step[r];
    int target = -1;
    if (hint && hint[j]) {
        const int alen = static_cast<int>(ans_off[j + 1] - ans_off[j]);
        target = t < alen ? ans[ans_off[j] + t] : SGC_EOS;
    }
    const int bi = block_biased_argmax(logits + static_cast<size_t>(r) * SGC_VOCAB, target, bonus);
    if (threadIdx.x == 0) tok[r] = bi;
}

__global__ void transpose_head(float* out_t, const float* head, int d) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < SGC_VOCAB * d; i += gridDim.x * blockDim.x) {
        int v = i / d, k = i % d;
        out_t[static_cast<size_t>(k) * SGC_VOCAB + v] = head[i];
    }
}

}  // namespace

static unsigned grid_for(uint64_t n, int threads, int sms) {
    uint64_t b = (n + threads - 1) / threads;
    uint64_t cap = static_cast<uint64_t>(sms) * 32;
    return static_cast<unsigned>(b < cap ? (b ? b : 1) : cap);
}

void gen_uniform(Ctx* c, float* out, uint64_t n, uint64_t state0, float lo, float hi) {
    gen_uniform_f32<<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(out, n, state0, lo, hi);
    SGC_LAUNCH_CHECK(c);
}
void gen_uniform(Ctx* c, __nv_bfloat16* out, uint64_t n, uint64_t state0, float lo, float hi) {
    gen_uniform_bf16<<<grid_for(n, 256, c->num_sms), 256, 0, c->stream>>>(out, n, state0, lo, hi);
    SGC_LAUNCH_CHECK(c);
}
void gen_text_projection_t(Ctx* c, float* out_t, uint32_t dim, uint64_t state0) {
    gen_projection_t<<<grid_for((uint64_t)dim * 4096, 256, c->num_sms), 256, 0, c->stream>>>(out_t, dim, state0);
    SGC_LAUNCH_CHECK(c);
}
void embed(Ctx* c, float* x, const int32_t* tokens, const float* tok_emb, const float* soft,
           const int32_t* soft_idx, int d, int rows, int* bad, __nv_bfloat16* xb, float* ss) {
    if (rows <= 0) return;
    Ctx::Timed timer(c, "embed");
    embed_kernel<<<rows, 128, 0, c->stream>>>(x, tokens, tok_emb, soft, soft_idx, d, rows, bad, xb, ss);
    SGC_LAUNCH_CHECK(c);
}
void rmsnorm_bf16(Ctx* c, __nv_bfloat16* out, const float* x, int d, int rows) {
    if (rows <= 0) return;
    Ctx::Timed timer(c, "rmsnorm");
    int threads = d >= 512 ? 128 : 32;
    rmsnorm_bf16_kernel<<<rows, threads, 0, c->stream>>>(out, x, d, rows);
    SGC_LAUNCH_CHECK(c);
}
void head_logits(Ctx* c, float* logits, const float* x, const int32_t* rows, int n,
                 const float* head_t, int d) {
    if (n <= 0) return;
    Ctx::Timed timer(c, "head");
    const int splits = static_cast<int>(ceil_div(d, kHeadChunk));
    float* inv = c->buf<float>("head_inv", n);
    float* partial = splits > 1 ? c->buf<float>("head_partial", static_cast<size_t>(splits) * n * SGC_VOCAB) : logits;
    head_norm_kernel<<<ceil_div(n, 8), 256, 0, c->stream>>>(inv, x, rows, n, d);
    SGC_LAUNCH_CHECK(c);
    head_kernel<<<dim3(ceil_div(n, kHeadRows), splits), 288, 0, c->stream>>>(partial, x, inv, rows, n, head_t, d);
    SGC_LAUNCH_CHECK(c);
    if (splits > 1) {
        head_reduce_kernel<<<ceil_div(static_cast<uint64_t>(n) * SGC_VOCAB, 256), 256, 0, c->stream>>>(logits, partial, n, splits);
        SGC_LAUNCH_CHECK(c);
    }
}
void first_tokens(Ctx* c, int32_t* first, const float* logits, int n, const int32_t* ctx_tokens,
                  const uint64_t* ctx_off, const uint32_t* member_ctx, const int32_t* ans,
                  const uint64_t* ans_off, float bonus, int8_t* hint_out) {
    if (n <= 0) return;
    Ctx::Timed timer(c, "first_token");
    first_token_kernel<<<n, 128, 0, c->stream>>>(first, hint_out, logits, n, ctx_tokens, ctx_off,
                                                 member_ctx, ans, ans_off, bonus);
    SGC_LAUNCH_CHECK(c);
}
void step_tokens(Ctx* c, int32_t* tok, const float* logits, int n, const int8_t* hint, const int32_t* ans,
                 const uint64_t* ans_off, const int32_t* member, const int32_t* step, float bonus) {
    if (n <= 0) return;
    Ctx::Timed timer(c, "first_token");
    step_token_kernel<<<n, 128, 0, c->stream>>>(tok, logits, n, hint, ans, ans_off, member, step, bonus);
    SGC_LAUNCH_CHECK(c);
}
namespace {
// RMSNorm scale of every row from its chunk sums of squares, summed in index order (the scale
// never depends on which tile or warp produced a chunk): 1 / sqrt(sum / d + 1e-5), lm_core.cpp:26-31
// one warp per row: lane l sums parts l, l + 32, ... in order, then a fixed xor tree -- the
// reduction order depends only on n_parts, never on how rows are batched (bit-identical waves)
__global__ void rms_scale_kernel(float* scale, const float* parts, int rows, int n_parts, int d) {
    const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (r >= rows) return;
    const float* pr = parts + static_cast<size_t>(r) * n_parts;
    float ss = 0.f;
    if (n_parts == 128) {  // d = 4096: one float4 per lane, coalesced
        const float4 v = reinterpret_cast<const float4*>(pr)[lane];
        ss = (v.x + v.y) + (v.z + v.w);
    } else {
        for (int i = lane; i < n_parts; i += 32) ss += pr[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) scale[r] = 1.0f / sqrtf(ss / static_cast<float>(d) + 1e-5f);
}
__global__ void gather_rows_kernel(uint4* dst, const uint4* src, const int32_t* rows, size_t row_vecs) {
    const uint4* s = src + static_cast<size_t>(rows[blockIdx.x]) * row_vecs;
    uint4* o = dst + static_cast<size_t>(blockIdx.x) * row_vecs;
    for (size_t k = threadIdx.x; k < row_vecs; k += blockDim.x) o[k] = s[k];
}
__global__ void iota_kernel(int32_t* p, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}
}  // namespace
void rms_scale(Ctx* c, float* scale, const float* parts, int rows, int n_parts, int d) {
    if (rows <= 0) return;
    Ctx::Timed timer(c, "rmsnorm");
    rms_scale_kernel<<<ceil_div(rows, 8), 256, 0, c->stream>>>(scale, parts, rows, n_parts, d);
    SGC_LAUNCH_CHECK(c);
}
void gather_rows(Ctx* c, void* dst, const void* src, const int32_t* rows, int n, size_t row_bytes) {
    if (n <= 0) return;
    if (row_bytes % 16) fail(SGC_DOMAIN, "gather_rows: row bytes must be a multiple of 16");
    gather_rows_kernel<<<n, 256, 0, c->stream>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), rows,
                                                 row_bytes / 16);
    SGC_LAUNCH_CHECK(c);
}
int32_t* Ctx::iota(int n) {
    int32_t* p = buf<int32_t>("iota", n);
    const int cap = static_cast<int>(scratch["iota"].bytes / sizeof(int32_t));
    if (n > iota_n || iota_ptr != p) {
        iota_kernel<<<grid_for(static_cast<uint64_t>(cap), 256, num_sms), 256, 0, stream>>>(p, cap);
        SGC_LAUNCH_CHECK(this);
        iota_n = cap;
        iota_ptr = p;
    }
    return p;
}
namespace {
__global__ void kv_pages_pack_kernel(uint4* packed, uint4* pool, size_t layer_vecs, const int32_t* bt, int len,
                                     int row_vecs, bool pack) {
    const int j = blockIdx.x, l = blockIdx.y;  // row j of layer l
    const size_t prow = static_cast<size_t>(bt[j / 128]) * 128 + j % 128;
    uint4* pp = pool + l * layer_vecs + prow * row_vecs;
    uint4* qq = packed + (static_cast<size_t>(l) * len + j) * row_vecs;
    for (int k = threadIdx.x; k < row_vecs; k += blockDim.x) {
        if (pack) qq[k] = pp[k];
        else pp[k] = qq[k];
    }
}

constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ULL, kFnvPrime = 0x100000001b3ULL;
// level 1: one warp per (segment, layer, K|V, row): lane l hashes the row's 16-byte vectors
// l, l + 32, ... (FNV-1a over 64-bit words, coalesced loads), then the 32 lane digests are folded
// in lane order -- the row digest
__global__ void kv_row_digest_kernel(uint64_t* rowh, const __nv_bfloat16* kp, const __nv_bfloat16* vp,
                                     size_t layer_stride, const int32_t* bt, const uint32_t* bt_off,
                                     const uint32_t* len, int max_len, int layers, int d) {
    const int s = blockIdx.z, lw = blockIdx.y;  // lw = 2 l + which
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    if (j >= static_cast<int>(len[s])) return;  // warp-uniform
    const int l = lw >> 1;
    const __nv_bfloat16* base = ((lw & 1) ? vp : kp) + l * layer_stride;
    const size_t prow = static_cast<size_t>(bt[bt_off[s] + j / 128]) * 128 + j % 128;
    const uint4* r = reinterpret_cast<const uint4*>(base + prow * d);
    uint64_t h = kFnvBasis;
    for (int v = lane; v < d / 8; v += 32) {
        const uint4 u = __ldg(r + v);
        h = (h ^ (static_cast<uint64_t>(u.y) << 32 | u.x)) * kFnvPrime;
        h = (h ^ (static_cast<uint64_t>(u.w) << 32 | u.z)) * kFnvPrime;
    }
    uint64_t row = kFnvBasis;
    for (int t = 0; t < 32; ++t) row = (row ^ __shfl_sync(0xffffffffu, h, t)) * kFnvPrime;
    if (lane == 0) rowh[(static_cast<size_t>(s) * layers * 2 + lw) * max_len + j] = row;
}
// level 2: fold row digests per (segment, layer, K|V) in row order; level 3: fold those in order
__global__ void kv_fold_kernel(uint64_t* out, const uint64_t* rowh, const uint32_t* len, int max_len, int layers) {
    const int s = blockIdx.x;
    __shared__ uint64_t part[256];
    const int n = static_cast<int>(len[s]);
    for (int lw = threadIdx.x; lw < 2 * layers; lw += blockDim.x) {
        const uint64_t* r = rowh + (static_cast<size_t>(s) * layers * 2 + lw) * max_len;
        uint64_t h = kFnvBasis;
        for (int j = 0; j < n; ++j) h = (h ^ r[j]) * kFnvPrime;
        part[lw] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t h = kFnvBasis;
        for (int lw = 0; lw < 2 * layers; ++lw) h = (h ^ part[lw]) * kFnvPrime;
        out[s] = h;
    }
}
}  // namespace

void kv_pages_pack(Ctx* c, __nv_bfloat16* packed, __nv_bfloat16* pool, size_t layer_stride, const int32_t* bt,
                   int len, int layers, int d, bool pack) {
    if (len <= 0 || layers <= 0) return;
    if (d % 8) fail(SGC_DOMAIN, "kv_pages_pack: d must be a multiple of 8");
    const dim3 grid(len, layers);
    kv_pages_pack_kernel<<<grid, 128, 0, c->stream>>>(reinterpret_cast<uint4*>(packed), reinterpret_cast<uint4*>(pool),
                                                      layer_stride / 8, bt, len, d / 8, pack);
    SGC_LAUNCH_CHECK(c);
}

void kv_digest(Ctx* c, cudaStream_t stream, uint64_t* out, uint64_t* rowh, const __nv_bfloat16* k_pool,
               const __nv_bfloat16* v_pool, size_t layer_stride, const int32_t* bt, const uint32_t* bt_off,
               const uint32_t* len, int n, int max_len, int layers, int d) {
    if (n <= 0) return;
    if (2 * layers > 256) fail(SGC_DOMAIN, "kv_digest: at most 128 layers");
    if (max_len > 0) {
        const dim3 grid(ceil_div(max_len, 8), 2 * layers, n);
        kv_row_digest_kernel<<<grid, 256, 0, stream>>>(rowh, k_pool, v_pool, layer_stride, bt, bt_off, len,
                                                       max_len, layers, d);
        SGC_LAUNCH_CHECK(c);
    }
    kv_fold_kernel<<<n, 64, 0, stream>>>(out, rowh, len, max_len, layers);
    SGC_LAUNCH_CHECK(c);
}

void head_transpose(Ctx* c, float* out_t, const float* head, int d) {
    transpose_head<<<grid_for((uint64_t)SGC_VOCAB * d, 256, c->num_sms), 256, 0, c->stream>>>(out_t, head, d);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace sgc
