// gemm.cuh -- host interface of the tcgen05 GEMM (gemm_sm100.cu).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace sgc {

struct Ctx;

enum { EPI_F32 = 0, EPI_BF16 = 1, EPI_RESID = 2, EPI_TANH = 3, EPI_QKV = 4 };

struct GemmEpi {
    int mode = EPI_F32;
    void* out = nullptr;  // F32/BF16/TANH: output; RESID: fp32 residual updated in place
    int ldo = 0;
    // EPI_QKV (N = 3d): q -> q_out[row], k -> k_cache[kv_row[row]], v -> v_cache[kv_row[row]]
    __nv_bfloat16* q_out = nullptr;
    __nv_bfloat16* k_cache = nullptr;
    __nv_bfloat16* v_cache = nullptr;
    const int32_t* kv_row = nullptr;
    const int32_t* pos = nullptr;
    const float* rope_cos = nullptr;  // [max_seq x hd/2]
    const float* rope_sin = nullptr;
    int d = 0;
    int hd = 0;
    // fused RMSNorm (lm_core.cpp:26-31, no gain): A holds bf16(x) UNnormalized and the epilogue
    // multiplies each accumulator row by row_scale[row] = 1 / sqrt(mean(x^2) + 1e-5) (QKV, TANH,
    // F32, BF16), finalized from the producer's per-chunk sums in index order (rms_scale)
    const float* row_scale = nullptr;
    // decode steps: the epilogue finalizes the row scale itself from the producer's per-chunk
    // sums of squares (ss_parts[row * ss_n ..], rms_scale's exact summation tree) instead of a
    // separate rms_scale launch; ss_d = model dim
    const float* ss_parts = nullptr;
    int ss_n = 0;
    int ss_d = 0;
    // EPI_RESID producer side: also store bf16(x_new) to out_xb (ld = ldo) and, per 32-column
    // chunk c of the row, its sum of squares of x_new to out_ss[row * (N / 32) + c]
    __nv_bfloat16* out_xb = nullptr;
    float* out_ss = nullptr;
    // decode steps only: allow the split-K residual path for few rows (changes the fp32
    // summation order, so prefill / extend rows never take it: their results stay
    // independent of how rows are grouped into calls)
    bool splitk_ok = false;
    // stream-K (set by the dispatcher): fp32 partial slots of the pairs, their ready flags and
    // this launch's sequence number
    float* sk_ws = nullptr;
    uint32_t* sk_flags = nullptr;
    uint32_t sk_seq = 0;
};

void gemm_bf16(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep);
// use the CTA-pair (cta_group::2) kernel for 256-wide tiles when M >= 256 (default on)
void gemm_set_pairs(bool on);
// CTA-pair GEMM raster: 0 M-groups (default), 1 chosen by estimated DRAM bytes, 2 N-groups
void gemm_set_raster(int mode);
// decode-step GEMMs (splitk_ok) on a stream-K CTA-pair kernel: 1 = on (default), 0 = split-K
// residual planes / 1-wave tiles
void gemm_set_streamk(int mode);

}  // namespace sgc
