// attention.cuh -- host interface of the cascade attention kernel (attention.cu).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace sgc {

struct Ctx;

// KV pages: 128 tokens (= the tcgen05 kernel's key block). A key sequence is read through a
// block table: key j of a sequence whose pages start at table offset `off` lives at pool row
// bt[off + j / 128] * 128 + j % 128 (bt == nullptr: contiguous rows, key j at row off + j).
constexpr int kPageTokens = 128;
__host__ __device__ inline int kv_row_of(const int32_t* bt, int off, int j) {
    return bt ? bt[off + j / kPageTokens] * kPageTokens + j % kPageTokens : off + j;
}

// A tile of consecutive query rows that share one sealed prefix.
struct AttnWork {
    int row0, nrows;
    int pfx_off;  // prefix: block-table offset of the sealed prefix's pages (bt) or its first row
    int pfx_len;  // prefix keys (0 for representative prefill)
    int loc_bt;   // own keys: -1 = contiguous batch rows of k_loc / v_loc; >= 0 = block-table
                  // offset of the sequence's pages in k_loc / v_loc (paged prefill)
};

struct AttnParams {
    const __nv_bfloat16* q;      // [rows x d], RoPE applied
    __nv_bfloat16* out;          // [rows x d]
    const __nv_bfloat16* k_pfx;  // KV pool (this layer) holding the sealed prefixes
    const __nv_bfloat16* v_pfx;
    const __nv_bfloat16* k_loc;  // KV rows written by this batch: row r at loc_kv0 + r
    const __nv_bfloat16* v_loc;
    int loc_kv0;
    const int32_t* seg_lo;  // [rows] first row of the row's own sequence (causal window start)
    const AttnWork* work;
    const int32_t* bt = nullptr;  // block table of the pages the work items reference (device)
    int d;
    float scale;  // 1/sqrt(head_dim) (lm_core.cpp:188)
    // partial mode (tcgen05 kernel only): prefix keys only, fp32 normalized O + log2-sum-exp
    float* part_o = nullptr;    // [rows x d]
    float* part_lse = nullptr;  // [rows x heads], in units of log2 of the scaled scores
};

void cascade_attention(Ctx* c, const AttnParams& p, int n_work, int heads, int hd);
// tcgen05 version (attention_sm100.cu): units of <= 256 rows (two 128-row tiles); head_dim 64
// or 128. Returns
// false when the shape is not supported by it.
bool cascade_attention_tc(Ctx* c, const AttnParams& p, int n_work, int heads, int hd, int q_rows,
                          int pfx_rows, int loc_rows);
inline bool attention_tc_supported(int hd) { return hd == 64 || hd == 128; }
// split every S row over two softmax warpgroups, or one thread per row (default)
void attention_set_split(bool on);
// 0: two 128-row tiles per item (attn_tc_kernel, default); 1: one tile, S triple-buffered, two
// softmax warpgroups on alternate key blocks (attn_s3_kernel)
void attention_set_kernel(int k);
// the same for partial mode (decode): default 1
void attention_set_kernel_partial(int k);

// Decode step (attention.cu): merge the prefix partial (part_o, part_lse from the tcgen05 kernel
// in partial mode, or none when part_o == nullptr) with each row's own keys: question rows
// [q_lo[r], q_lo[r] + q_n[r]) of (k_q, v_q) and generated rows [g_lo[r], g_lo[r] + g_n[r]) of
// (k_g, v_g); one softmax over all of them (lm_core.cpp:246-274), bf16 out.
struct DecodeAttnParams {
    const __nv_bfloat16* q;
    const __nv_bfloat16 *k_p, *v_p, *k_q, *v_q, *k_g, *v_g;
    // prefix keys [0, p_n) of (k_p, v_p) through the block table p_bt at offset p_lo (p_bt ==
    // nullptr: rows p_lo ..): read here only when part_o == nullptr
    const int32_t *p_lo, *p_n, *q_lo, *q_n, *g_lo, *g_n;
    const int32_t* p_bt = nullptr;
    const float* part_o;
    const float* part_lse;
    __nv_bfloat16* out;
    int rows, d, heads;
    float scale;
};
void decode_attention_local(Ctx* c, const DecodeAttnParams& p);

}  // namespace sgc
