// attention.cuh -- host interface of the cascade attention kernel (attention.cu).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace sgc {

struct Ctx;

// A tile of <= 64 consecutive query rows that share one sealed prefix.
struct AttnWork {
    int row0, nrows;
    int pfx_kv0;  // first KV-pool row of the shared prefix
    int pfx_len;  // prefix keys (0 for representative prefill)
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
    int d;
    float scale;  // 1/sqrt(head_dim) (lm_core.cpp:188)
};

void cascade_attention(Ctx* c, const AttnParams& p, int n_work, int heads, int hd);
// tcgen05 version (attention_sm100.cu): units of <= 256 rows (two 128-row tiles); head_dim 64
// or 128. Returns
// false when the shape is not supported by it.
bool cascade_attention_tc(Ctx* c, const AttnParams& p, int n_work, int heads, int hd, int q_rows,
                          int pfx_rows, int loc_rows);
inline bool attention_tc_supported(int hd) { return hd == 64 || hd == 128; }

}  // namespace sgc
