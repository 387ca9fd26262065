// lm_kernels.cuh -- host interface of lm_kernels.cu
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sgc {
struct Ctx;
void gen_uniform(Ctx* c, float* out, uint64_t n, uint64_t state0, float lo, float hi);
void gen_uniform(Ctx* c, __nv_bfloat16* out, uint64_t n, uint64_t state0, float lo, float hi);
void gen_text_projection_t(Ctx* c, float* out_t, uint32_t dim, uint64_t state0);
void embed(Ctx* c, float* x, const int32_t* tokens, const float* tok_emb, const float* soft,
           const int32_t* soft_idx, int d, int rows, int* bad, __nv_bfloat16* xb = nullptr,
           float* ss = nullptr);
void rmsnorm_bf16(Ctx* c, __nv_bfloat16* out, const float* x, int d, int rows);
// per-row RMSNorm scale from per-chunk sums of squares (n_parts per row), fixed summation order
void rms_scale(Ctx* c, float* scale, const float* parts, int rows, int n_parts, int d);
// dst[i] = src[rows[i]] for i < n, rows of row_bytes (a multiple of 16)
void gather_rows(Ctx* c, void* dst, const void* src, const int32_t* rows, int n, size_t row_bytes);
void head_logits(Ctx* c, float* logits, const float* x, const int32_t* rows, int n,
                 const float* head_t, int d);
void first_tokens(Ctx* c, int32_t* first, const float* logits, int n, const int32_t* ctx_tokens,
                  const uint64_t* ctx_off, const uint32_t* member_ctx, const int32_t* ans,
                  const uint64_t* ans_off, float bonus, int8_t* hint_out = nullptr);
void step_tokens(Ctx* c, int32_t* tok, const float* logits, int n, const int8_t* hint, const int32_t* ans,
                 const uint64_t* ans_off, const int32_t* member, const int32_t* step, float bonus);
void head_transpose(Ctx* c, float* out_t, const float* head, int d);

// ---- paged KV (128-token pages, pool [L][pages * 128][d] per K and V) ------------------------
// rows [0, len) of a segment (block table bt[0..]) of every layer <-> packed [L][len][d]:
// pack = pool -> packed (point-to-point send of a sealed prefix), else packed -> pool
void kv_pages_pack(Ctx* c, __nv_bfloat16* packed, __nv_bfloat16* pool, size_t layer_stride, const int32_t* bt,
                   int len, int layers, int d, bool pack);
// KVCache::prefix_digest analogue over bf16 pages (tree FNV-1a over 64-bit words: row digests,
// per-(layer, K|V) folds in row order, then those folds in layer order, K before V); a row's
// digest folds 32 lane digests, lane l covering the row's 16-byte vectors l, l + 32, ... for n segments at once: out[s] (device)
// rowh: scratch [n][2 layers][max_len] uint64; launched on `stream` (the path overlaps it)
void kv_digest(Ctx* c, cudaStream_t stream, uint64_t* out, uint64_t* rowh, const __nv_bfloat16* k_pool,
               const __nv_bfloat16* v_pool, size_t layer_stride, const int32_t* bt, const uint32_t* bt_off,
               const uint32_t* len, int n, int max_len, int layers, int d);
}  // namespace sgc
