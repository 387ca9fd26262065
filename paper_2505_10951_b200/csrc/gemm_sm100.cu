// gemm_sm100.cu -- persistent, warp-specialized tcgen05/TMEM/TMA GEMM for sm_100a with the
// ToyLm's fused epilogues.
//
// D[M x N] = A[M x K] * B[N x K]^T; A = activations (bf16, row-major), B = a ToyLm weight
// (bf16, row-major [out x in], lm_core.hpp:161-168), fp32 accumulation in TMEM.
//
//   warp 0      TMA producer: A 128x64 and B BNx64 tiles (128B swizzle) into a smem ring
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16) x4 per stage
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld -> fused epilogue -> global stores
//
// Epilogues (the ops the reference runs after each matvec, lm_core.cpp:220-283):
//   EPI_F32 / EPI_BF16   plain store
//   EPI_RESID            x += D                         (residual add, lm_core.cpp:277,283)
//   EPI_TANH             h = bf16(tanh(D))              (FFN activation, :281)
//   EPI_QKV              RoPE(q), RoPE(k) -> K cache, v -> V cache, q -> Q buffer (:227-244)
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "gemm.cuh"
#include "sched.cuh"
#include "sm100_ptx.cuh"
#include "tma.cuh"

namespace sgc {

namespace {

// decode-sized GEMMs (129-256 rows) on CTA pairs (1) or 1-CTA 128-row tiles (0)
#ifndef SGC_DECODE_PAIRS
#define SGC_DECODE_PAIRS 1
#endif
// decode residual split-K at <= 128 rows on CTA pairs (1) or 1-CTA 64-column tiles (0)
#ifndef SGC_RESID_SPLIT_PAIRS_SMALL
#define SGC_RESID_SPLIT_PAIRS_SMALL 0
#endif
// A/B switch: residual epilogue with 32-byte loads/stores (1) or 8-byte column pairs (0)
#ifndef SGC_RESID_V8
#define SGC_RESID_V8 1
#endif
constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
// warps: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator, 3 idle, 4-11 epilogue (two warpgroups,
// each owning half of the tile's 32-column chunks; a warp may only read TMEM lanes 32*(warp%4))
constexpr int kThreads = 384;
constexpr int kEpiThreads = 256;
// per epilogue warp: a 32 x 33 fp32 staging tile (row-major, padded: conflict-free both ways)
constexpr int kStageSmem = 8 * 32 * 33 * 4;
// barrier area: stage / accumulator barriers in the first 256 B, the tile ring in the next 256 B
constexpr int kBarBytes = 512;
constexpr int kRing = 8;  // claimed tiles in flight between the fetcher and the epilogue
using TileRing = UnitRing<kRing>;
static_assert(sizeof(TileRing) <= 256, "tile ring must fit its barrier-area half");

// chunk range of epilogue warpgroup `eg` (0/1): halves of the tile, or everything in group 0 when
// a QKV head (RoPE pairs chunk ch with ch + HD/64) would straddle the halves
template <int BN, int EPI, int HD>
__device__ __forceinline__ void epi_chunks(int eg, int& lo, int& hi) {
    constexpr int NCH = BN / 32;
    constexpr bool split = NCH % 2 == 0 && !(EPI == EPI_QKV && BN < 2 * HD);
    if (split) {
        lo = eg * (NCH / 2);
        hi = lo + NCH / 2;
    } else {
        lo = 0;
        hi = eg == 0 ? NCH : 0;
    }
}

template <int BN>
struct Cfg {
    static constexpr int kStages = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + kBarBytes + kStageSmem;
};

#ifndef SGC_TANH_APPROX
#define SGC_TANH_APPROX 1
#endif
__device__ __forceinline__ float tanh_fast(float x) {
#if SGC_TANH_APPROX
    // MUFU.TANH: max relative error ~2^-11, 8x below the bf16 rounding of the stored activation
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
#endif
    // tanh via exp2: accurate to ~1e-7 relative, saturates cleanly (reference clamps at 9,
    // kernels_scalar.cpp:74-81)
    x = fminf(fmaxf(x, -9.0f), 9.0f);
    float e = exp2f(x * 2.8853900817779268f);  // exp(2x)
    return __fdividef(e - 1.0f, e + 1.0f);
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

// store 32 fp32 values as bf16 (64 contiguous bytes)
__device__ __forceinline__ void store_bf16x32_stream(__nv_bfloat16* dst, const float* v, uint64_t pol) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // 2 x 32 B (STG.256)
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) w[e] = pack_bf16(v[16 * q + 2 * e], v[16 * q + 2 * e + 1]);
        ptx::st_global_v8_hint(dst + 16 * q, w, pol);
    }
}
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) w[e] = pack_bf16(v[16 * q + 2 * e], v[16 * q + 2 * e + 1]);
        ptx::st_global_v8(dst + 16 * q, w);
    }
}

// RoPE on a pair of 32-column chunks (lo = cols i, hi = cols i+half), reference op order
// (lm_core.cpp:231-238) without FMA contraction.
#ifndef SGC_ROPE_PACKED
#define SGC_ROPE_PACKED 1
#endif
// packed fp32x2 helpers (FMUL2 / FFMA2 on sm_100a)
__device__ __forceinline__ uint64_t f2pack_g(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack_g(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t fmul2_g(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t ffma2_g(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fneg2_g(uint64_t a) {
    return a ^ 0x8000000080000000ull;
}
__device__ __forceinline__ void rope_pair(float* lo, float* hi, const float* cosp,
                                          const float* sinp) {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        float c = cosp[j], s = sinp[j];
        float a = lo[j], b = hi[j];
        lo[j] = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
        hi[j] = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
    }
}

// stream-K (decode GEMMs): earlier K segments of this tile, written by other CTA pairs as fp32
// slots laid out [column / 4][128 rows of the CTA][4] (a warp moves 512 contiguous bytes per
// 16-byte access, thread = row); the tile's last segment adds them, in pair order, before its
// fused epilogue
struct PartIn {
    const float* base = nullptr;  // slot of the first contributing pair, this CTA's half
    int n = 0;                    // contributing pairs
    int stride = 0;               // floats between consecutive pairs' slots
    bool valid = true;            // this thread's row exists (rows past M were never stored)
};
constexpr int kSkSlot = 128 * 256;  // floats per CTA per slot (128 rows x BN 256)
__device__ __forceinline__ const float4* sk_at(const float* slot, int ch, int j4, int rr) {
    return reinterpret_cast<const float4*>(slot) + (ch * 8 + j4) * 128 + rr;
}
__device__ __forceinline__ void add_parts(const PartIn& pin, uint32_t* r, int ch) {
    if (pin.n == 0 || !pin.valid) return;
    const int rr = ((threadIdx.x >> 5) & 3) * 32 + (threadIdx.x & 31);
    for (int q = 0; q < pin.n; q += 2) {  // two contributors' loads in flight, added in order
        const bool two = q + 1 < pin.n;
        float4 v0[8], v1[8];
        const float* s0 = pin.base + static_cast<size_t>(q) * pin.stride;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) v0[j4] = __ldcg(sk_at(s0, ch, j4, rr));
        if (two) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) v1[j4] = __ldcg(sk_at(s0 + pin.stride, ch, j4, rr));
        }
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
            float* f = reinterpret_cast<float*>(r + 4 * j4);
            f[0] += v0[j4].x;
            f[1] += v0[j4].y;
            f[2] += v0[j4].z;
            f[3] += v0[j4].w;
        }
        if (two) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
                float* f = reinterpret_cast<float*>(r + 4 * j4);
                f[0] += v1[j4].x;
                f[1] += v1[j4].y;
                f[2] += v1[j4].z;
                f[3] += v1[j4].w;
            }
        }
    }
}

// 1 / sqrt(mean(x^2) + 1e-5) of one row from its d/32 chunk sums, in rms_scale_kernel's exact
// order (lm_kernels.cu: lane l's sum of parts l, l+32, .. -- 4 contiguous parts per lane when
// n = 128 -- then the xor butterfly lane 0 ends with), so the scale is bit-identical to the
// separate launch it replaces
__device__ __forceinline__ float rms_inv_row(const float* pr, int n, int d) {
    float s[32];
    if (n == 128) {
#pragma unroll
        for (int l = 0; l < 32; ++l) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(pr) + l);
            s[l] = (v.x + v.y) + (v.z + v.w);
        }
    } else {
#pragma unroll
        for (int l = 0; l < 32; ++l) s[l] = 0.f;
        for (int i = 0; i < n; ++i) s[i % 32] += __ldg(pr + i);
    }
    // butterfly: after the step with offset o, lane l holds (its value) + (lane l^o's value)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int l = 0; l < o; ++l) s[l] = s[l] + s[l + o];
    }
    return 1.0f / sqrtf(s[0] / static_cast<float>(d) + 1e-5f);
}

// Epilogue of one 128 x BN accumulator tile held in TMEM (lanes = rows): `tbase` addresses
// this warp's 32 lanes at the tile's first column, `row` is this thread's output row.
template <int BN, int EPI, int HD>
__device__ __forceinline__ void epilogue_tile(uint32_t tbase, int row, bool valid, int n0,
                                              const GemmEpi& ep, int ch_lo, int ch_hi, float* stage,
                                              int ep_rows, const PartIn& pin = PartIn{}) {
    // fused RMSNorm of the A rows: one scale per accumulator row
    float inv = 1.0f;
    if (ep.row_scale && valid) inv = ep.row_scale[row];
    else if (ep.ss_parts && valid) inv = rms_inv_row(ep.ss_parts + static_cast<size_t>(row) * ep.ss_n, ep.ss_n, ep.ss_d);
    if constexpr (EPI == EPI_QKV) {
        // one tile never straddles the q/k/v sections (d % BN == 0)
        const int d = ep.d;
        const int section = n0 / d;
        const int c0 = n0 - section * d;
        constexpr int HALF = HD / 2;
        int pos = 0, kvr = 0;
        if (valid) {
            pos = ep.pos[row];
            kvr = ep.kv_row[row];
        }
        if (section == 2) {
#pragma unroll 1
            for (int ch = ch_lo; ch < ch_hi; ++ch) {
                uint32_t r[32];
                ptx::tmem_ld32(tbase + ch * 32, r);
                ptx::tmem_ld_wait();
                add_parts(pin, r, ch);
                if (valid) {
                    float* v = reinterpret_cast<float*>(r);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= inv;
                    store_bf16x32(ep.v_cache + static_cast<size_t>(kvr) * d + c0 + ch * 32, v);
                }
            }
        } else {
            __nv_bfloat16* dst = section == 0
                                     ? ep.q_out + static_cast<size_t>(row) * d
                                     : ep.k_cache + static_cast<size_t>(kvr) * d;
            const float* cosp = ep.rope_cos + static_cast<size_t>(pos) * HALF;
            const float* sinp = ep.rope_sin + static_cast<size_t>(pos) * HALF;
            if constexpr (HALF >= 32) {
                // pairs span two chunks: (ch, ch + HALF/32) within each head
#pragma unroll 1
                for (int ch = ch_lo; ch < ch_hi; ++ch) {
                    const int in_head = (ch * 32) % HD;
                    if (in_head >= HALF) continue;
                    const int ch2 = ch + HALF / 32;
                    // RoPE table rows (128 B aligned) in flight while the accumulator loads
                    float cs[32], sn[32];
                    if (valid) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {  // LDG.256
                            ptx::ld_nc_f8(cosp + in_head + 8 * j, cs + 8 * j);
                            ptx::ld_nc_f8(sinp + in_head + 8 * j, sn + 8 * j);
                        }
                    }
                    uint32_t lo[32], hi[32];
                    ptx::tmem_ld32(tbase + ch * 32, lo);
                    ptx::tmem_ld32(tbase + ch2 * 32, hi);
                    ptx::tmem_ld_wait();
                    add_parts(pin, lo, ch);
                    add_parts(pin, hi, ch2);
                    if (valid) {
#if SGC_ROPE_PACKED
                        // RMSNorm scale + RoPE on packed fp32 pairs (FMUL2 / FFMA2): the epilogue's
                        // issue slots, not the tensor pipe, were the QKV GEMM's margin
                        const uint64_t inv2 = f2pack_g(inv, inv);
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            const uint64_t c2 = f2pack_g(cs[j], cs[j + 1]);
                            const uint64_t a2 = fmul2_g(f2pack_g(__uint_as_float(lo[j]), __uint_as_float(lo[j + 1])), inv2);
                            const uint64_t b2 = fmul2_g(f2pack_g(__uint_as_float(hi[j]), __uint_as_float(hi[j + 1])), inv2);
                            const uint64_t sp = f2pack_g(sn[j], sn[j + 1]);
                            // lo' = a c - b s ; hi' = b c + a s
                            const uint64_t l2 = ffma2_g(a2, c2, fmul2_g(b2, fneg2_g(sp)));
                            const uint64_t h2 = ffma2_g(b2, c2, fmul2_g(a2, sp));
                            float x0, x1, y0, y1;
                            f2unpack_g(l2, x0, x1);
                            f2unpack_g(h2, y0, y1);
                            reinterpret_cast<float*>(lo)[j] = x0;
                            reinterpret_cast<float*>(lo)[j + 1] = x1;
                            reinterpret_cast<float*>(hi)[j] = y0;
                            reinterpret_cast<float*>(hi)[j + 1] = y1;
                        }
#else
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            reinterpret_cast<float*>(lo)[j] *= inv;
                            reinterpret_cast<float*>(hi)[j] *= inv;
                        }
                        rope_pair(reinterpret_cast<float*>(lo), reinterpret_cast<float*>(hi),
                                  cs, sn);
#endif
                        store_bf16x32(dst + c0 + ch * 32, reinterpret_cast<float*>(lo));
                        store_bf16x32(dst + c0 + ch2 * 32, reinterpret_cast<float*>(hi));
                    }
                }
            } else {
                // whole heads inside one 32-column chunk
#pragma unroll 1
                for (int ch = ch_lo; ch < ch_hi; ++ch) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tbase + ch * 32, r);
                    ptx::tmem_ld_wait();
                    add_parts(pin, r, ch);
                    if (valid) {
                        float* v = reinterpret_cast<float*>(r);
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] *= inv;
                        float o[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int i = j % HD;
                            if (i < HALF) {
                                float c = __ldg(cosp + i), s = __ldg(sinp + i);
                                float a = v[j], b = v[j + HALF];
                                o[j] = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, s));
                                o[j + HALF] = __fadd_rn(__fmul_rn(b, c), __fmul_rn(a, s));
                            }
                        }
                        store_bf16x32(dst + c0 + ch * 32, o);
                    }
                }
            }
        }
    } else {
        // Coalesced epilogue: each warp owns a 32-row x 32-column chunk per step; the accumulator
        // (thread = row) goes through a padded shared-memory tile and leaves along rows: lane l
        // handles rows 2i + l/16 and the column pair 2(l%16), so every warp instruction moves two
        // full 128 B (fp32) / 64 B (bf16) row segments instead of touching 32 lines -- the L1TEX
        // path stays free for the TMA operand loads.
        if constexpr (EPI == EPI_TANH || EPI == EPI_BF16) {
            // bf16 outputs: each thread stores its own row's 64 B per chunk (measured faster for
            // the FFN activation than the transposed path: 97.7% vs 92% tensor-active); streamed
            // with evict_first so they do not push the group's operand tiles out of L2
            const uint64_t stream_pol = ptx::policy_evict_first();
#pragma unroll 1
            for (int ch = ch_lo; ch < ch_hi; ++ch) {
                uint32_t r[32];
                ptx::tmem_ld32(tbase + ch * 32, r);
                ptx::tmem_ld_wait();
                add_parts(pin, r, ch);
                if (!valid) continue;
                float* v = reinterpret_cast<float*>(r);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    v[j] *= inv;
                    if constexpr (EPI == EPI_TANH) v[j] = tanh_fast(v[j]);
                }
                store_bf16x32_stream(static_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(row) * ep.ldo + n0 + ch * 32, v,
                                     stream_pol);
            }
            (void)stage;
            (void)ep_rows;
            return;
        }
#if SGC_RESID_V8
        if constexpr (EPI == EPI_RESID) {
            // transposed residual epilogue with 32-byte accesses: lane = (row 8i + lane/4,
            // columns 8*(lane%4)..+7) of the warp's 32 x 32 chunk; stage reads conflict-free
            // (bank = row + column mod 32 covers all 32 banks)
            const uint64_t resid_pol = ptx::policy_evict_first();
            const int lane = threadIdx.x & 31;
            const int row0 = row - lane;
            const int rsub = lane >> 2, cq = (lane & 3) * 8;
#pragma unroll 1
            for (int ch = ch_lo; ch < ch_hi; ++ch) {
                const int col = n0 + ch * 32 + cq;
                float xo[4][8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int gr = row0 + 8 * i + rsub;
                    if (gr < ep_rows)
                        ptx::ld_global_f8_hint(static_cast<const float*>(ep.out) + static_cast<size_t>(gr) * ep.ldo + col,
                                               xo[i], resid_pol);
                    else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) xo[i][e] = 0.f;
                    }
                }
                uint32_t r[32];
                ptx::tmem_ld32(tbase + ch * 32, r);
                ptx::tmem_ld_wait();
                add_parts(pin, r, ch);
                // 16-byte staging with an XOR swizzle of the 4-float groups (row r's group k at
                // k ^ (r & 7)): STS.128 / LDS.128, conflict-free on both sides, no padding
                float4* st4 = reinterpret_cast<float4*>(stage);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    st4[lane * 8 + (k ^ (lane & 7))] = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]),
                                                                   __uint_as_float(r[4 * k + 2]), __uint_as_float(r[4 * k + 3]));
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int lr = 8 * i + rsub, gr = row0 + lr;
                    float val[8];
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const float4 a = st4[lr * 8 + ((cq / 4 + h2) ^ (lr & 7))];
                        val[4 * h2 + 0] = a.x;
                        val[4 * h2 + 1] = a.y;
                        val[4 * h2 + 2] = a.z;
                        val[4 * h2 + 3] = a.w;
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) val[e] += xo[i][e];
                    if (ep.out_ss) {  // keep x_new for the row sums below
                        st4[lr * 8 + ((cq / 4) ^ (lr & 7))] = make_float4(val[0], val[1], val[2], val[3]);
                        st4[lr * 8 + ((cq / 4 + 1) ^ (lr & 7))] = make_float4(val[4], val[5], val[6], val[7]);
                    }
                    if (gr < ep_rows) {
                        const size_t off = static_cast<size_t>(gr) * ep.ldo + col;
                        ptx::st_global_v8_hint(static_cast<float*>(ep.out) + off, *reinterpret_cast<uint32_t(*)[8]>(val),
                                               resid_pol);
                        if (ep.out_xb) {
                            uint4 w;
                            w.x = pack_bf16(val[0], val[1]);
                            w.y = pack_bf16(val[2], val[3]);
                            w.z = pack_bf16(val[4], val[5]);
                            w.w = pack_bf16(val[6], val[7]);
                            *reinterpret_cast<uint4*>(ep.out_xb + off) = w;
                        }
                    }
                }
                __syncwarp();
                if (ep.out_ss) {  // this row's sum of squares over the chunk, columns in order
                    float cs = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float4 a = st4[lane * 8 + (k ^ (lane & 7))];
                        cs = fmaf(a.x, a.x, cs);
                        cs = fmaf(a.y, a.y, cs);
                        cs = fmaf(a.z, a.z, cs);
                        cs = fmaf(a.w, a.w, cs);
                    }
                    if (valid) ep.out_ss[static_cast<size_t>(row) * (ep.ldo / 32) + (n0 / 32 + ch)] = cs;
                }
                __syncwarp();
            }
            return;
        }
#endif
        float ss = 0.f;  // EPI_RESID with out_ss: this row's partial sum of squares of x_new
        // the fp32 residual stream is read and written once per launch: evict_first keeps it from
        // pushing the raster group's operand tiles out of L2
        const uint64_t resid_pol = ptx::policy_evict_first();
        const int lane = threadIdx.x & 31;
        const int row0 = row - lane;    // the warp's first row
        const int half = lane >> 4;     // row parity handled by this lane
        const int c2 = 2 * (lane & 15);  // column pair within the chunk
#pragma unroll 1
        for (int ch = ch_lo; ch < ch_hi; ++ch) {
            const int col = n0 + ch * 32 + c2;
            // residual inputs (16 row pairs) in flight with the TMEM load
            float2 xo[16];
            if constexpr (EPI == EPI_RESID) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int gr = row0 + 2 * i + half;
                    xo[i] = gr < ep_rows ? ptx::ld_global_f2_hint(static_cast<const float*>(ep.out) +
                                                                      static_cast<size_t>(gr) * ep.ldo + col,
                                                                  resid_pol)
                                         : make_float2(0.f, 0.f);
                }
            }
            uint32_t r[32];
            ptx::tmem_ld32(tbase + ch * 32, r);
            ptx::tmem_ld_wait();
            add_parts(pin, r, ch);
            float* v = reinterpret_cast<float*>(r);
            if constexpr (EPI != EPI_RESID) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] *= inv;
            }
            if constexpr (EPI == EPI_TANH) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = tanh_fast(v[j]);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) stage[lane * 33 + j] = v[j];
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int lr = 2 * i + half, gr = row0 + lr;
                float2 val = make_float2(stage[lr * 33 + c2], stage[lr * 33 + c2 + 1]);
                const size_t off = static_cast<size_t>(gr) * ep.ldo + col;
                if constexpr (EPI == EPI_RESID) {
                    val.x += xo[i].x;
                    val.y += xo[i].y;
                    stage[lr * 33 + c2] = val.x;
                    stage[lr * 33 + c2 + 1] = val.y;
                }
                if (gr < ep_rows) {
                    if constexpr (EPI == EPI_RESID) {
                        ptx::st_global_f2_hint(static_cast<float*>(ep.out) + off, val, resid_pol);
                        if (ep.out_xb) *reinterpret_cast<__nv_bfloat162*>(ep.out_xb + off) = __floats2bfloat162_rn(val.x, val.y);
                    } else if constexpr (EPI == EPI_F32) {
                        *reinterpret_cast<float2*>(static_cast<float*>(ep.out) + off) = val;
                    } else {
                        *reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(ep.out) + off) =
                            __floats2bfloat162_rn(val.x, val.y);
                    }
                }
            }
            __syncwarp();
            if constexpr (EPI == EPI_RESID) {
                if (ep.out_ss) {  // this row's sum of squares over the chunk -> its own slot
                    float cs = 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float xv = stage[lane * 33 + j];
                        cs = fmaf(xv, xv, cs);
                    }
                    if (valid) ep.out_ss[static_cast<size_t>(row) * (ep.ldo / 32) + (n0 / 32 + ch)] = cs;
                }
                __syncwarp();
            }
        }
        (void)ss;
    }
}

template <int BN, int EPI, int HD>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                int M, int N, int K, GemmEpi ep, int ksplit, uint32_t* sched_ctr) {
    using C = Cfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smemA = smem;
    uint8_t* smemB = smem + C::kStages * C::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + C::kStages;
    uint64_t* tfull = bars + 2 * C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    TileRing* ring = reinterpret_cast<TileRing*>(reinterpret_cast<uint8_t*>(bars) + 256);

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int m_tiles = (M + BM - 1) / BM;
    const int n_tiles = N / BN;
    // split-K (few-row decode GEMMs): work item = (output tile, K slice); slice s accumulates
    // k-blocks [s * num_kb, (s + 1) * num_kb) and the fp32 epilogue writes plane s of `out`
    const int num_tiles = m_tiles * n_tiles * ksplit;
    const int num_kb = K / BK / ksplit;
    // grouped raster: GROUP m-tiles sweep all n-tiles before moving on, so both the
    // activation rows and the weight tiles of the concurrently running CTAs stay in L2
    const int GROUP = max(4, min(64, (48 << 20) / (BM * K * 2)));

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < C::kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], kEpiThreads);
        }
        sched::init(ring, 1 + kEpiThreads / 32);  // consumers: the MMA thread + 8 epilogue warps
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto tile_coords = [&](int t, int& m0, int& n0) {
        t /= ksplit;
        int per_group = GROUP * n_tiles;
        int g = t / per_group;
        int first_m = g * GROUP;
        int gsize = min(GROUP, m_tiles - first_m);
        int r = t % per_group;
        m0 = (first_m + r % gsize) * BM;
        n0 = (r / gsize) * BN;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // operands are re-read across the raster group's tiles: keep them in L2 ahead of the
            // streamed epilogue outputs
            const uint64_t keep = ptx::policy_evict_last();
            uint32_t next = sched::claim(sched_ctr, num_tiles, gridDim.x, 0);
            for (uint32_t k = 0;; ++k) {
                const uint32_t tu = next;
                sched::publish(ring, k, tu);
                if (tu >= static_cast<uint32_t>(num_tiles)) break;
                next = sched::claim(sched_ctr, num_tiles, gridDim.x, k + 1);
                const int t = static_cast<int>(tu);
                int m0, n0;
                tile_coords(t, m0, n0);
                const int kb0 = (t % ksplit) * num_kb;
                for (int kb = kb0; kb < kb0 + num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_expect_tx(&full[stage], C::kStageBytes);
                    ptx::tma_load_2d_hint(smemA + stage * C::kABytes, &tmA, &full[stage], kb * BK, m0, keep);
                    ptx::tma_load_2d_hint(smemB + stage * C::kBBytes, &tmB, &full[stage], kb * BK, n0, keep);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            for (uint32_t local = 0;; ++local) {
                const uint32_t tu = sched::wait(ring, local);
                sched::release(ring, local);
                if (tu >= static_cast<uint32_t>(num_tiles)) break;
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smemA + stage * C::kABytes);
                    const uint32_t b_addr = ptx::smem_u32(smemB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad = ptx::umma_desc_sw128(a_addr + k * 32);
                        uint64_t bd = ptx::umma_desc_sw128(b_addr + k * 32);
                        ptx::mma_bf16(tmem_d, ad, bd, idesc, (kb | k) != 0);
                    }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        const int ew = warp & 3;  // TMEM lanes 32*ew .. 32*ew+31
        int ch_lo, ch_hi;
        epi_chunks<BN, EPI, HD>((warp - 4) / 4, ch_lo, ch_hi);
        float* stage = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes) + (warp - 4) * 32 * 33;
        for (uint32_t local = 0;; ++local) {
            const uint32_t tu = sched::wait(ring, local);
            __syncwarp();
            if (lane == 0) sched::release(ring, local);
            if (tu >= static_cast<uint32_t>(num_tiles)) break;
            const int t = static_cast<int>(tu);
            int m0, n0;
            tile_coords(t, m0, n0);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int row = m0 + ew * 32 + lane;
            const bool valid = row < M;
            const uint32_t tbase = tmem_base + ((ew * 32) << 16) + acc * BN;
            GemmEpi eps = ep;
            if (ksplit > 1)  // fp32 partial plane of this K slice
                eps.out = static_cast<float*>(ep.out) + static_cast<size_t>(t % ksplit) * M * ep.ldo;
            epilogue_tile<BN, EPI, HD>(tbase, row, valid, n0, eps, ch_lo, ch_hi, stage, M);
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
        }
    }

    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// ---- CTA-pair variant (tcgen05.mma.cta_group::2) -------------------------------------------
// A cluster of 2 CTAs computes a 256 x 256 tile: each CTA TMA-loads its 128 rows of A and its
// 128 rows of B (half of N) into its own smem, the leader issues M=256 x N=256 MMAs that read
// both CTAs' operands, and each CTA's TMEM receives its own 128 x 256 accumulator rows. Per CTA
// this halves the B traffic of the 1-CTA 128 x 256 tile (32 KB instead of 48 KB per k-block).
constexpr int kStages2 = 6;
struct Cfg2 {
    static constexpr int kABytes = BM * BK * 2;  // this CTA's 128 rows of A
    static constexpr int kBBytes = BM * BK * 2;  // this CTA's 128 rows of B
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kSmem = kStages2 * kStageBytes + 1024 + kBarBytes + kStageSmem;
};

template <int EPI, int HD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 int M, int N, int K, GemmEpi ep, int ksplit, uint32_t* sched_ctr, int ngroup) {
    constexpr int BN = 256;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smemA = smem;
    uint8_t* smemB = smem + kStages2 * Cfg2::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages2 * Cfg2::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages2;
    uint64_t* tfull = bars + 2 * kStages2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    // the leader's producer claims pair-tiles and publishes them to both CTAs' rings
    TileRing* ring = reinterpret_cast<TileRing*>(reinterpret_cast<uint8_t*>(bars) + 256);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int npairs = gridDim.x >> 1;
    const int m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const int n_tiles = N / BN;
    // split-K (decode residual GEMMs): work item = (pair-tile, K slice); the fp32 epilogue writes
    // plane `slice` of `out`, a fixed-order reduction adds the planes
    const int num_tiles = m_tiles * n_tiles * ksplit;
    const int num_kb = K / BK / ksplit;
    // pair-tiles of 256 rows per raster group: the group's A rows (GROUP x 256 x K bf16) stay
    // L2-resident (~32 MB) while the group sweeps every n-tile; larger K -> smaller group
// residual GEMMs' raster group (scripts/gpu_lib_gemm_ab.sh, final kernels, gemm_resid ms/step):
// 24 MB 293-296, 32 MB 294-295, 48 MB 296, 64 MB 297-299
#ifndef SGC_RESID_GROUP_MB
#define SGC_RESID_GROUP_MB 32
#endif
// raster-group budget (A rows of a group kept L2-resident while it sweeps the n-tiles):
// measured at C3, 24-32 MB beats 48 (~0.7% GEMM time) and 96 (-4%); re-swept on the final
// kernels: 16 MB 201 / 227 ms (QKV / W1 per step), 24 and 40 MB within noise of 32 (198-199 / 225)
#ifndef SGC_GROUP_MB
#define SGC_GROUP_MB 32
#endif
    constexpr int kGroupBytes = (EPI == EPI_RESID ? SGC_RESID_GROUP_MB : SGC_GROUP_MB) << 20;
    const int GROUP = max(2, min(32, kGroupBytes / (2 * BM * K * 2)));

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < kStages2; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 2 * kEpiThreads);  // both CTAs' epilogue threads release
        }
        // leader slot consumers: its MMA thread + 8 epilogue warps, the peer's producer + 8
        // epilogue warps (the peer's own empty barriers are unused)
        sched::init(ring, 2 + 2 * (kEpiThreads / 32));
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_2sm<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // peer barriers initialized before any remote arrive / TMA signal
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    auto tile_coords = [&](int t, int& m0, int& n0) {
        t /= ksplit;
        if (ngroup > 0) {
            // N-group raster (host-chosen when it moves fewer DRAM bytes): `ngroup` n-tiles of
            // the weights stay L2-resident while the group sweeps every m-tile, so the weights
            // are read once and the activations once per group
            int per_group = ngroup * m_tiles;
            int g = t / per_group;
            int first_n = g * ngroup;
            int gsize = min(ngroup, n_tiles - first_n);
            int r = t % per_group;
            n0 = (first_n + r % gsize) * BN;
            m0 = (r / gsize) * 2 * BM;
            return;
        }
        int per_group = GROUP * n_tiles;
        int g = t / per_group;
        int first_m = g * GROUP;
        int gsize = min(GROUP, m_tiles - first_m);
        int r = t % per_group;
        m0 = (first_m + r % gsize) * 2 * BM;
        n0 = (r / gsize) * BN;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t keep = ptx::policy_evict_last();  // operands re-read across the group
            uint32_t next = leader ? sched::claim(sched_ctr, num_tiles, npairs, 0) : 0;
            for (uint32_t k = 0;; ++k) {
                uint32_t tu;
                if (leader) {
                    tu = next;
                    sched::publish_pair(ring, k, tu);
                    if (tu < static_cast<uint32_t>(num_tiles)) next = sched::claim(sched_ctr, num_tiles, npairs, k + 1);
                } else {
                    tu = sched::wait_remote(ring, k);
                    sched::release_to(ring, k, 0);
                }
                if (tu >= static_cast<uint32_t>(num_tiles)) break;
                const int t = static_cast<int>(tu);
                int m0, n0;
                tile_coords(t, m0, n0);
                const int kb0 = (t % ksplit) * num_kb;
                for (int kb = kb0; kb < kb0 + num_kb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) ptx::mbar_expect_tx(&full[stage], 2 * Cfg2::kStageBytes);
                    ptx::tma_load_2d_2sm_hint(smemA + stage * Cfg2::kABytes, &tmA, &full[stage], kb * BK,
                                              m0 + rank * BM, keep);
                    ptx::tma_load_2d_2sm_hint(smemB + stage * Cfg2::kBBytes, &tmB, &full[stage], kb * BK,
                                              n0 + rank * BM, keep);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            for (uint32_t local = 0;; ++local) {
                const uint32_t tu = sched::wait(ring, local);
                sched::release(ring, local);
                if (tu >= static_cast<uint32_t>(num_tiles)) break;
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smemA + stage * Cfg2::kABytes);
                    const uint32_t b_addr = ptx::smem_u32(smemB + stage * Cfg2::kBBytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        ptx::mma_bf16_2sm(tmem_d, ptx::umma_desc_sw128(a_addr + k * 32),
                                          ptx::umma_desc_sw128(b_addr + k * 32), idesc, (kb | k) != 0);
                    ptx::mma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_2sm(&tfull[acc], 0x3);
            }
        }
    } else if (warp >= 4) {
        const int ew = warp & 3;
        int ch_lo, ch_hi;
        epi_chunks<BN, EPI, HD>((warp - 4) / 4, ch_lo, ch_hi);
        float* stage = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes) + (warp - 4) * 32 * 33;
        for (uint32_t local = 0;; ++local) {
            uint32_t tu;
            if (leader) {
                tu = sched::wait(ring, local);
                __syncwarp();
                if (lane == 0) sched::release(ring, local);
            } else {
                tu = sched::wait_remote(ring, local);
                __syncwarp();
                if (lane == 0) sched::release_to(ring, local, 0);
            }
            if (tu >= static_cast<uint32_t>(num_tiles)) break;
            const int t = static_cast<int>(tu);
            int m0, n0;
            tile_coords(t, m0, n0);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int row = m0 + static_cast<int>(rank) * BM + ew * 32 + lane;
            const uint32_t tbase = tmem_base + ((ew * 32) << 16) + acc * BN;
            GemmEpi eps = ep;
            if (ksplit > 1)  // fp32 partial plane of this K slice
                eps.out = static_cast<float*>(ep.out) + static_cast<size_t>(t % ksplit) * M * ep.ldo;
            epilogue_tile<BN, EPI, HD>(tbase, row, row < M, n0, eps, ch_lo, ch_hi, stage, M);
            ptx::tc_fence_before();
            ptx::mbar_arrive_cluster(&tempty[acc], 0);
        }
    }

    __syncthreads();
    ptx::cluster_sync();  // neither CTA frees TMEM while the pair may still use it
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<512>(tmem_base);
    }
}

// ---- stream-K CTA-pair variant (decode steps) ----------------------------------------------
// A decode step has few rows (M <= 512), so the pair-tiles (48 for the QKV weights) cannot fill
// the 74 SM pairs and every weight byte is streamed by only 2/3 of the SMs. Here the
// (tile, k-block) space is cut into one equal contiguous range per pair: a pair's range is a run
// of segments (tile, k-block range). The tile's LAST segment owns the fused epilogue; every
// earlier segment of that tile (at most one per pair: the one that ends its range) stores its
// fp32 accumulator to the pair's workspace slot and raises a flag (this launch's sequence
// number). Each pair processes that partial segment FIRST, so no flag depends on another wait:
// all pairs are resident (grid <= SM pairs) and the owners' waits always resolve. The owner adds
// the partials in pair order (deterministic for a given shape) before the usual epilogue.
struct SkRange {
    int lo, hi;  // [lo, hi) over the tiles x k-blocks space
};
__device__ __forceinline__ SkRange sk_range(int p, int P, int W) {
    return {static_cast<int>(static_cast<int64_t>(p) * W / P), static_cast<int>(static_cast<int64_t>(p + 1) * W / P)};
}
struct SkSeg {
    int t, kb0, kb1;  // tile, k-blocks [kb0, kb1) within the tile
    int kind;         // 0 whole tile, 1 partial (ends before the tile does), 2 owner (adds partials)
    int q0;           // owner: first contributing pair (contributors q0 .. p-1)
};
__device__ __forceinline__ int sk_nseg(const SkRange& r, int KB) { return (r.hi - 1) / KB - r.lo / KB + 1; }
// i-th segment in PROCESSING order: the range's trailing partial (if any) first
__device__ __forceinline__ SkSeg sk_seg(int p, int P, int W, int KB, const SkRange& r, int i) {
    const int n = sk_nseg(r, KB);
    const bool tail_partial = r.hi % KB != 0;
    const int nat = tail_partial ? (i == 0 ? n - 1 : i - 1) : i;
    const int t = r.lo / KB + nat;
    const int a = max(r.lo, t * KB), b = min(r.hi, (t + 1) * KB);
    SkSeg s;
    s.t = t;
    s.kb0 = a - t * KB;
    s.kb1 = b - t * KB;
    s.q0 = p;
    if (b < (t + 1) * KB) s.kind = 1;
    else if (a > t * KB) {
        s.kind = 2;
        int q = p - 1;  // ranges are non-empty (P <= W): walk back to the pair holding k-block t*KB
        while (q > 0 && sk_range(q, P, W).lo > t * KB) --q;
        s.q0 = q;
    } else s.kind = 0;
    return s;
}

#ifdef SGC_SK_PROF  // A/B builds only: per-CTA phase cycles of the stream-K kernel (scripts/sk_prof.py)
}  // namespace
__device__ unsigned long long g_sk_prof[148 * 32];
namespace {
#define SK_T0(v) const long long v = clock64()
#define SK_ACC(slot, t0) atomicAdd(&g_sk_prof[(blockIdx.x % 148) * 32 + (slot)], (unsigned long long)(clock64() - (t0)))
#else
#define SK_T0(v)
#define SK_ACC(slot, t0)
#endif
template <int EPI, int HD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2_sk_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M, int N, int K, GemmEpi ep) {
    constexpr int BN = 256;
    SK_T0(t_start);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* smemA = smem;
    uint8_t* smemB = smem + kStages2 * Cfg2::kABytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages2 * Cfg2::kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages2;
    uint64_t* tfull = bars + 2 * kStages2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint64_t* pub = tempty + 3;  // this CTA's epilogue threads stored the pair's partial

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int P = gridDim.x >> 1, p = blockIdx.x >> 1;
    const int m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const int n_tiles = N / BN;
    const int KB = K / BK;
    const int W = m_tiles * n_tiles * KB;
    const SkRange rg = sk_range(p, P, W);
    const int nseg = sk_nseg(rg, KB);
    // tile t -> (m0, n0): m-tiles of one weight tile adjacent (its second read hits L2)
    auto tile_coords = [&](int t, int& m0, int& n0) {
        m0 = (t % m_tiles) * 2 * BM;
        n0 = (t / m_tiles) * BN;
    };

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < kStages2; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 2 * kEpiThreads);
        }
        ptx::mbar_init(pub, kEpiThreads);  // one phase: a pair stores at most one partial per launch
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_2sm<512>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 128) SK_ACC(0, t_start);
    SK_T0(t_main);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint64_t keep = ptx::policy_evict_last();  // A is re-read by every pair
            const uint64_t stream = ptx::policy_evict_first();  // each weight byte is read once
            for (int i = 0; i < nseg; ++i) {
                const SkSeg sg = sk_seg(p, P, W, KB, rg, i);
                int m0, n0;
                tile_coords(sg.t, m0, n0);
                for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
                    SK_T0(t_w);
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    SK_ACC(8, t_w);
#ifdef SGC_SK_NOLOAD  // A/B builds only: the MMA side alone
                    if (leader) ptx::mbar_arrive(&full[stage]);
                    (void)keep;
                    (void)stream;
#else
                    if (leader) ptx::mbar_expect_tx(&full[stage], 2 * Cfg2::kStageBytes);
                    ptx::tma_load_2d_2sm_hint(smemA + stage * Cfg2::kABytes, &tmA, &full[stage], kb * BK,
                                              m0 + rank * BM, keep);
                    ptx::tma_load_2d_2sm_hint(smemB + stage * Cfg2::kBBytes, &tmB, &full[stage], kb * BK,
                                              n0 + rank * BM, m_tiles > 1 ? keep : stream);
#endif
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0; i < nseg; ++i) {
                const SkSeg sg = sk_seg(p, P, W, KB, rg, i);
                const int acc = i & 1;
                const uint32_t acc_phase = (i >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = sg.kb0; kb < sg.kb1; ++kb) {
                    SK_T0(t_w);
                    ptx::mbar_wait(&full[stage], phase);
                    SK_ACC(6, t_w);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(smemA + stage * Cfg2::kABytes);
                    const uint32_t b_addr = ptx::smem_u32(smemB + stage * Cfg2::kBBytes);
#ifndef SGC_SK_NOMMA  // A/B builds only: the operand stream alone
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        ptx::mma_bf16_2sm(tmem_d, ptx::umma_desc_sw128(a_addr + k * 32),
                                          ptx::umma_desc_sw128(b_addr + k * 32), idesc, (kb != sg.kb0) | (k != 0));
#else
                    (void)a_addr;
                    (void)b_addr;
                    (void)idesc;
#endif
                    ptx::mma_commit_2sm(&empty[stage], 0x3);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_2sm(&tfull[acc], 0x3);
            }
            SK_ACC(7, t_main);
        }
    } else if (warp >= 4) {
        const int ew = warp & 3, eg = (warp - 4) / 4;
        int ch_lo, ch_hi;
        epi_chunks<BN, EPI, HD>(eg, ch_lo, ch_hi);
        float* stage = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes) + (warp - 4) * 32 * 33;
        const int rr = ew * 32 + lane;  // this thread's row within the CTA's 128
        for (int i = 0; i < nseg; ++i) {
            const SkSeg sg = sk_seg(p, P, W, KB, rg, i);
            int m0, n0;
            tile_coords(sg.t, m0, n0);
            const int acc = i & 1;
            const uint32_t acc_phase = (i >> 1) & 1;
            SK_T0(t_w);
            ptx::mbar_wait(&tfull[acc], acc_phase);
            if (threadIdx.x == 128) SK_ACC(1, t_w);
            SK_T0(t_e);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + ((ew * 32) << 16) + acc * BN;
            if (sg.kind == 1) {
                // partial: raw fp32 accumulator -> this pair's slot (both warpgroups, 4 chunks each);
                // rows past M are neither stored nor read back
                float* slot = ep.sk_ws + static_cast<size_t>(2 * p + rank) * kSkSlot;
                const bool row_ok = m0 + static_cast<int>(rank) * BM + rr < M;
#pragma unroll 1
                for (int ch = eg * 4; ch < eg * 4 + 4; ++ch) {
                    uint32_t r[32];
                    ptx::tmem_ld32(tbase + ch * 32, r);
                    ptx::tmem_ld_wait();
                    if (!row_ok) continue;
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4)
                        __stcg(const_cast<float4*>(sk_at(slot, ch, j4, rr)),
                               make_float4(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]),
                                           __uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])));
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive_cluster(&tempty[acc], 0);
                // every epilogue thread of this CTA stored -> publish (release, GPU scope)
                __threadfence();
                ptx::mbar_arrive(pub);
                if (warp == 4 && lane == 0) {
                    ptx::mbar_wait(pub, 0);
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ep.sk_flags + 2 * p + rank), "r"(ep.sk_seq)
                                 : "memory");
                }
                if (threadIdx.x == 128) SK_ACC(4, t_e);
                continue;
            }
            PartIn pin;
            if (sg.kind == 2) {
                for (int q = sg.q0; q < p; ++q) {
                    const uint32_t* f = ep.sk_flags + 2 * q + rank;
                    uint32_t v;
                    do {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    } while (v != ep.sk_seq);
                }
                pin.base = ep.sk_ws + static_cast<size_t>(2 * sg.q0 + rank) * kSkSlot;
                pin.n = p - sg.q0;
                pin.stride = 2 * kSkSlot;
                pin.valid = m0 + static_cast<int>(rank) * BM + rr < M;
                if (threadIdx.x == 128) SK_ACC(2, t_e);
            }
            SK_T0(t_ep);
            const int row = m0 + static_cast<int>(rank) * BM + rr;
            epilogue_tile<BN, EPI, HD>(tbase, row, row < M, n0, ep, ch_lo, ch_hi, stage, M, pin);
            ptx::tc_fence_before();
            ptx::mbar_arrive_cluster(&tempty[acc], 0);
            if (threadIdx.x == 128) SK_ACC(sg.kind == 2 ? 3 : 9, t_ep);
        }
        if (threadIdx.x == 128) SK_ACC(5, t_main);
    }

    __syncthreads();
    ptx::cluster_sync();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<512>(tmem_base);
    }
}

// ---- host side ----------------------------------------------------------------------------

// CUDA-event timing category per fused epilogue (bench.py sums "gemm*" for the roofline)
constexpr const char* gemm_timer_name(int epi) {
    return epi == EPI_QKV ? "gemm_qkv" : epi == EPI_RESID ? "gemm_resid" : epi == EPI_TANH ? "gemm_tanh" : "gemm";
}

template <int BN, int EPI, int HD>
void launch(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep, int ksplit = 1) {
    using Cf = Cfg<BN>;
    static bool attr_set = false;  // per-instantiation (per process; single device type)
    auto kfn = gemm_kernel<BN, EPI, HD>;
    if (!attr_set) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem));
        attr_set = true;
    }
    CUtensorMap ta = make_map_2d(A, M, K, BM, BK);
    CUtensorMap tb = make_map_2d(B, N, K, BN, BK);
    int tiles = ((M + BM - 1) / BM) * (N / BN) * ksplit;
    int grid = tiles < c->num_sms ? tiles : c->num_sms;
    Ctx::Timed timer(c, gemm_timer_name(ksplit > 1 ? EPI_RESID : EPI));
    kfn<<<grid, kThreads, Cf::kSmem, c->stream>>>(ta, tb, M, N, K, ep, ksplit, c->sched_counter());
    SGC_LAUNCH_CHECK(c);
}

// 0: M-group raster (default), 1: by estimated operand DRAM bytes, 2: N-groups (sgc_set_option
// "gemm_raster"). Measured at C3 (scripts/gpu_raster_ab.sh): N-groups cut the residual GEMMs' DRAM
// reads 4.88 -> 3.76 GB per launch but raise QKV / W1 reads 1.54 -> 3.45 GB (the activation rows of
// the slab's m-tiles do not survive in L2 next to a 64 MB weight slab) and every family ran 1-2%
// slower, so the M-group raster stays the default.
int g_gemm_raster = 0;

template <int EPI, int HD>
void launch2(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep, int ksplit = 1) {
    static bool attr_set = false;
    auto kfn = gemm2_kernel<EPI, HD>;
    if (!attr_set) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::kSmem));
        attr_set = true;
    }
    CUtensorMap ta = make_map_2d(A, M, K, BM, BK);
    CUtensorMap tb = make_map_2d(B, N, K, BM, BK);
    const int m_tiles = (M + 2 * BM - 1) / (2 * BM), n_tiles = N / 256;
    int tiles = m_tiles * n_tiles * ksplit;
    int grid = 2 * tiles < c->num_sms ? 2 * tiles : (c->num_sms & ~1);
    // raster orientation by estimated DRAM bytes for the operands: M-groups (the group's
    // activation rows resident, weights re-read once per group) or N-groups (a weight slab of
    // ~kNGroupBytes resident, activations re-read once per slab)
    int ngroup = 0;
    if (g_gemm_raster != 0 && m_tiles > 1) {
        constexpr double kNGroupBytes = 64.0 * (1 << 20);
        const int mgroup = std::max(2, std::min(32, ((EPI == EPI_RESID ? 48 : 32) << 20) / (2 * BM * K * 2)));
        const double a = 2.0 * M * K, b = 2.0 * N * K;
        const int m_groups = (m_tiles + mgroup - 1) / mgroup;
        const int ng = std::max(1, static_cast<int>(kNGroupBytes / (256.0 * K * 2)));
        const int n_groups = (n_tiles + ng - 1) / ng;
        const double traffic_m = a + b * m_groups, traffic_n = a * n_groups + b;
        if (g_gemm_raster == 2 || traffic_n < 0.9 * traffic_m) ngroup = ng;
    }
    Ctx::Timed timer(c, gemm_timer_name(ksplit > 1 ? EPI_RESID : EPI));
    kfn<<<grid, kThreads, Cfg2::kSmem, c->stream>>>(ta, tb, M, N, K, ep, ksplit, c->sched_counter(), ngroup);
    SGC_LAUNCH_CHECK(c);
}

bool g_gemm_pairs = true;  // CTA-pair kernel for large tiles (sgc_set_gemm_pairs toggles)
int g_gemm_streamk = 1;    // decode GEMMs on the stream-K pair kernel (sgc_set_option "gemm_streamk"; 2 = every decode shape)

// decode-step GEMM on the stream-K pair kernel: one equal (tile, k-block) range per SM pair
template <int EPI, int HD>
void launch2_sk(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep) {
    static bool attr_set = false;
    auto kfn = gemm2_sk_kernel<EPI, HD>;
    if (!attr_set) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2::kSmem));
        attr_set = true;
    }
    CUtensorMap ta = make_map_2d(A, M, K, BM, BK);
    CUtensorMap tb = make_map_2d(B, N, K, BM, BK);
    // one pair per co-resident cluster slot: a pair launched only after others retire would
    // serialize its owners' waits behind a second wave (the GPCs' SM counts are not all even,
    // so fewer than num_sms / 2 pairs fit at once)
    static int max_pairs = 0;
    if (!max_pairs) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = 2;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.gridDim = dim3(c->num_sms & ~1);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = Cfg2::kSmem;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int n = 0;
        SGC_CUDA_CHECK(cudaOccupancyMaxActiveClusters(&n, kfn, &cfg));
        max_pairs = std::max(1, std::min(n, c->num_sms / 2));
        if (std::getenv("SGC_TRACE_SK")) std::fprintf(stderr, "stream-K: %d co-resident CTA pairs\n", n);
    }
    const int m_tiles = (M + 2 * BM - 1) / (2 * BM);
    const int W = m_tiles * (N / 256) * (K / BK);
    const int P = std::min(max_pairs, W);
    if (!c->sk_flags) {
        c->sk_flags = c->buf<uint32_t>("gemm_sk_flags", 512);
        SGC_CUDA_CHECK(cudaMemsetAsync(c->sk_flags, 0, 512 * sizeof(uint32_t), c->stream));
    }
    if (2 * P > 512) fail(SGC_DOMAIN, "gemm: stream-K grid exceeds its flag array");
    GemmEpi e = ep;
    e.sk_ws = c->buf<float>("gemm_sk_ws", static_cast<size_t>(2 * P) * kSkSlot);
    e.sk_flags = c->sk_flags;
    e.sk_seq = ++c->sk_seq;
    if (e.sk_seq == 0) e.sk_seq = ++c->sk_seq;  // 0 is the flags' initial value
    if (std::getenv("SGC_TRACE_SK"))
        std::fprintf(stderr, "stream-K launch: M %d N %d K %d W %d P %d seq %u ws %p flags %p\n", M, N, K, W, P, e.sk_seq,
                     (void*)e.sk_ws, (void*)e.sk_flags);
    Ctx::Timed timer(c, gemm_timer_name(EPI));
    kfn<<<2 * P, kThreads, Cfg2::kSmem, c->stream>>>(ta, tb, M, N, K, e);
    SGC_LAUNCH_CHECK(c);
}

// split-K residual for decode-sized GEMMs: x += sum_s partial[s] in a fixed order, then bf16(x)
// and the row's sum of squares for the next GEMM's fused RMSNorm (one CTA per row)
__global__ void __launch_bounds__(256) resid_reduce_kernel(float* x, __nv_bfloat16* xb, float* ss_out,
                                                           const float* partial, int M, int N, int splits) {
    const int r = blockIdx.x;
    float ss = 0.f;
    const size_t plane = static_cast<size_t>(M) * N;
    // the row's sum of squares leaves as N/32 chunk slots (part 0 = the whole row, the rest 0)
    if (ss_out)
        for (int p = threadIdx.x + 1; p < N / 32; p += blockDim.x) ss_out[static_cast<size_t>(r) * (N / 32) + p] = 0.f;
    for (int c = threadIdx.x * 4; c < N; c += blockDim.x * 4) {
        const size_t off = static_cast<size_t>(r) * N + c;
        float4 v = *reinterpret_cast<const float4*>(x + off);
        for (int s2 = 0; s2 < splits; ++s2) {
            const float4 p = *reinterpret_cast<const float4*>(partial + s2 * plane + off);
            v.x += p.x;
            v.y += p.y;
            v.z += p.z;
            v.w += p.w;
        }
        *reinterpret_cast<float4*>(x + off) = v;
        if (xb) {
            __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&a);
            pk.y = *reinterpret_cast<uint32_t*>(&b);
            *reinterpret_cast<uint2*>(xb + off) = pk;
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
    }
    if (!ss_out) return;
    __shared__ float red[8];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += red[w];
        ss_out[static_cast<size_t>(r) * (N / 32)] = t;
    }
}

template <int EPI, int HD>
void dispatch_bn(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep) {
    // widest tile that divides N (and d, for the QKV section split)
    int lim = EPI == EPI_QKV ? ep.d : N;
    const int m_tiles = (M + BM - 1) / BM;
    // decode steps: stream-K over all SM pairs where it measured faster in the C3 generation run
    // (scripts/decode_probe.py): the FFN activation GEMM at <= 128 and 257-1024 rows, the residual
    // GEMMs at 257-1024 rows (W2 at 513-1024 rows: 130 -> 68-85 us; <= 256 rows keep their split-K planes, whose fixed-order reduction
    // beats a 4-5-way stream-K fixup); never the QKV GEMM, whose RoPE / K-V scatter epilogue then
    // runs on the owners' critical path over a 256-column tile (57 vs 40 us per launch)
    const bool sk_rows = EPI != EPI_QKV && (M > 2 * BM || (M <= BM && EPI != EPI_RESID));
    if (g_gemm_streamk && ep.splitk_ok && g_gemm_pairs && (sk_rows || g_gemm_streamk == 2) && M <= 8 * BM && N % 256 == 0 && lim % 256 == 0 &&
        N >= 2048 && K >= 1024 && HD <= 128) {
        launch2_sk<EPI, HD>(c, A, B, M, N, K, ep);
        return;
    }
    if constexpr (EPI == EPI_RESID) {
        // decode-sized residual GEMMs (N = d): too few output tiles to stream the weight matrix at
        // full bandwidth -> 4-way split-K into fp32 planes + a fixed-order reduction
        constexpr int kSplit = 4;
        if (ep.splitk_ok && M <= 2 * BM && m_tiles * (N / 64) < c->num_sms && N % 64 == 0 && (K / BK) % kSplit == 0) {
            float* partial = c->buf<float>("gemm_splitk", static_cast<size_t>(kSplit) * M * N);
            GemmEpi pe;
            pe.mode = EPI_F32;
            pe.out = partial;
            pe.ldo = N;
            // 129-256 rows: one CTA pair per 256-column tile reads each weight tile once and
            // every activation row once per 256 columns (the 1-CTA 64-column tiles re-read all
            // rows 4x as often); same K slices, so the same partial sums
            // <= 128 rows: pairs for the long-K W2 (40.7 -> 34.4 us at 64 rows), 64-column 1-CTA
            // tiles for Wo (18.5 vs 21 us on pairs; scripts/decode_gemm_sweep.py)
            if (SGC_DECODE_PAIRS && g_gemm_pairs && (M > BM || K >= 2 * N || SGC_RESID_SPLIT_PAIRS_SMALL) && N % 256 == 0)
                launch2<EPI_F32, 0>(c, A, B, M, N, K, pe, kSplit);
            else launch<64, EPI_F32, 0>(c, A, B, M, N, K, pe, kSplit);
            Ctx::Timed timer(c, "gemm_resid");
            resid_reduce_kernel<<<M, 256, 0, c->stream>>>(static_cast<float*>(ep.out), ep.out_xb, ep.out_ss, partial, M,
                                                          N, kSplit);
            SGC_LAUNCH_CHECK(c);
            return;
        }
    }
    // 129-256 rows (decode steps of ~150 members): one CTA pair covers all rows, so every weight
    // tile is read once (two 128-row m-tiles would each stream it) and a wide N fits one wave
    if (SGC_DECODE_PAIRS && g_gemm_pairs && EPI != EPI_RESID && M > BM && M <= 2 * BM && N % 256 == 0 &&
        lim % 256 == 0 && 2 * (N / 256) >= c->num_sms / 2) {
        launch2<EPI, HD>(c, A, B, M, N, K, ep);
        return;
    }
    // few rows (decode steps): the GEMM is weight-bandwidth bound, so spread the weight matrix
    // over as many CTAs as possible -- the narrowest tile that still yields >= one wave
    // (the QKV epilogue needs whole heads inside a tile: BN >= head_dim)
    if (m_tiles * (N / 256) < c->num_sms && N % 64 == 0 && lim % 64 == 0 && HD <= 128) {
        if ((N % 128 == 0 && lim % 128 == 0 && m_tiles * (N / 128) >= c->num_sms) || HD > 64)
            launch<128, EPI, HD>(c, A, B, M, N, K, ep);
        else
            launch<64, EPI, HD>(c, A, B, M, N, K, ep);
    } else if (g_gemm_pairs && M >= 2 * BM && N % 256 == 0 && lim % 256 == 0) launch2<EPI, HD>(c, A, B, M, N, K, ep);
    else if (N % 256 == 0 && lim % 256 == 0) launch<256, EPI, HD>(c, A, B, M, N, K, ep);
    else if (N % 128 == 0 && lim % 128 == 0) launch<128, EPI, HD>(c, A, B, M, N, K, ep);
    else if (N % 64 == 0 && lim % 64 == 0) launch<64, EPI, HD>(c, A, B, M, N, K, ep);
    else fail(SGC_DOMAIN, "gemm: N must be a multiple of 64");
}

}  // namespace

void gemm_set_pairs(bool on) { g_gemm_pairs = on; }
void gemm_set_raster(int mode) { g_gemm_raster = mode; }
void gemm_set_streamk(int mode) { g_gemm_streamk = mode; }

void gemm_bf16(Ctx* c, const void* A, const void* B, int M, int N, int K, const GemmEpi& ep) {
    if (M <= 0) return;
    if (K % BK != 0) fail(SGC_DOMAIN, "gemm: K must be a multiple of 64");
    switch (ep.mode) {
        case EPI_F32: dispatch_bn<EPI_F32, 0>(c, A, B, M, N, K, ep); break;
        case EPI_BF16: dispatch_bn<EPI_BF16, 0>(c, A, B, M, N, K, ep); break;
        case EPI_RESID: dispatch_bn<EPI_RESID, 0>(c, A, B, M, N, K, ep); break;
        case EPI_TANH: dispatch_bn<EPI_TANH, 0>(c, A, B, M, N, K, ep); break;
        case EPI_QKV:
            if (ep.hd == 128) dispatch_bn<EPI_QKV, 128>(c, A, B, M, N, K, ep);
            else if (ep.hd == 64) dispatch_bn<EPI_QKV, 64>(c, A, B, M, N, K, ep);
            else if (ep.hd == 32) dispatch_bn<EPI_QKV, 32>(c, A, B, M, N, K, ep);
            else if (ep.hd == 16) dispatch_bn<EPI_QKV, 16>(c, A, B, M, N, K, ep);
            else fail(SGC_DOMAIN, "gemm: head_dim must be 16, 32, 64 or 128");
            break;
        default: fail(SGC_DOMAIN, "gemm: unknown epilogue");
    }
}

}  // namespace sgc

#ifdef SGC_SK_PROF
extern "C" int sgc_debug_sk_prof(unsigned long long* out, int reset) {
    if (reset) {
        static unsigned long long z[148 * 32] = {};
        cudaMemcpyToSymbol(sgc::g_sk_prof, z, sizeof(z));
    } else {
        cudaMemcpyFromSymbol(out, sgc::g_sk_prof, sizeof(unsigned long long) * 148 * 32);
    }
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
#endif
