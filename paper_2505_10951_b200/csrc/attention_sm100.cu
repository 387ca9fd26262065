// attention_sm100.cu -- tcgen05/TMEM/TMA cascade attention for sm_100a (head_dim 64 / 128).
//
// Same semantics as attention.cu (lm_core.cpp:246-274: one softmax over the sealed prefix keys
// followed by the row's own causal suffix keys), re-laid out for the 5th-gen tensor cores:
//
//   warp 0      TMA loader: Q tile (128 rows) once per item and K blocks (128 keys) of the
//               cluster's prefix (phase A) then of the batch's own rows (phase B), 3-stage ring
//               released as soon as S = Q K^T has consumed a slot
//   warp 3      TMA loader for the V blocks, 2-stage ring released after O += P V
//   warp 1      MMA issuer (one thread): S_b = Q K_b^T into a double-buffered TMEM S, and
//               O += P_{b-1} V_{b-1} into TMEM O (P from smem, V as an MN-major operand)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..11 softmax, two warpgroups: thread (r, half) owns keys [64 half, 64 half + 64) of
//               query row r (TMEM lane r) and O columns [HD/2 half, ...). Reads its S half-row
//               from TMEM, masks, agrees on the row max with its partner through smem, online
//               softmax in base 2 with lazy O rescale (only when the running max grows by > 2^8),
//               writes its P half-row (bf16, 128B-swizzled) for the PV MMA, and at the end
//               normalizes and stores its half of the O row.
//
// The kernel is persistent: CTAs loop over (tile, head) items; a tile is <= 128 query rows of
// one cluster, so the prefix K/V blocks are fetched once per tile for every member row in it.
#include "attention.cuh"
#include "common.cuh"
#include "sm100_ptx.cuh"
#include "tma.cuh"

namespace sgc {
namespace {

constexpr int BQ = 128;   // query rows per item
constexpr int BKV = 128;  // keys per block
constexpr int kThreads = 384;  // 4 control warps + 2 softmax warpgroups

template <int HD>
struct TcCfg {
    static constexpr int kSub = HD / 64;            // 64-element (128 B) swizzle sub-tiles
    static constexpr int kQBytes = BQ * HD * 2;
    static constexpr int kKBytes = BKV * HD * 2;
    static constexpr int kVBytes = BKV * HD * 2;
    static constexpr int kPBytes = BQ * BKV * 2;
    static constexpr int kKStages = 3;  // K slots are freed as soon as S = Q K^T completes
    static constexpr int kVStages = 2;  // V slots are freed after O += P V
    static constexpr int kRedBytes = 2 * 2 * BQ * 4;
    static constexpr int kSmem = kQBytes + kPBytes + kKStages * kKBytes + kVStages * kVBytes +
                                 kRedBytes + 256;
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kO = 256;             // TMEM column of the O accumulator
};

// Compile with -DSGC_ATTN_PROF to accumulate per-phase clock64() cycles into a global
// [148][16] counter array (debug builds only; see scripts/attn_prof.py).
#ifdef SGC_ATTN_PROF
__device__ unsigned long long g_attn_prof[148 * 16];
#define PROF_T0() long long _pt = clock64()
#define PROF_ACC(slot)                                                             \
    do {                                                                           \
        long long _n = clock64();                                                  \
        atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 16 + (slot)], (unsigned long long)(_n - _pt)); \
        _pt = _n;                                                                  \
    } while (0)
#else
#define PROF_T0()
#define PROF_ACC(slot)
#endif

struct TcParams {
    const AttnWork* work;
    int n_work, heads;
    const int32_t* seg_lo;
    __nv_bfloat16* out;
    int d;
    float scale_log2;
};

// MUFU.EX2 without the denormal-range fixups of exp2f (inputs are <= 8; ex2(-inf) = +0)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA/ALU pipes (FA4-style MUFU offload): round-to-nearest split x = i + f,
// f in [-0.5, 0.5], degree-3 fit of 2^f (max rel. error 7.7e-5, far below the bf16 rounding
// of P), exponent added in the integer domain. Inputs are clamped at -125 (result ~1e-38).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -125.0f);
    const float t = x + 12582912.0f;  // 1.5 * 2^23: rounds x to the nearest integer
    const float f = x - (t - 12582912.0f);
    const float p = fmaf(fmaf(fmaf(0.05508868f, f, 0.24260405f), f, 0.69327623f), f, 0.99992895f);
    const int e = __float_as_int(t) - 0x4B400000;
    return __int_as_float(__float_as_int(p) + (e << 23));
}

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void item_blocks(const AttnWork& w, const int32_t* seg_lo, int& nA,
                                            int& nB, int& loc_first) {
    nA = (w.pfx_len + BKV - 1) / BKV;
    loc_first = seg_lo[w.row0];
    const int loc_last = w.row0 + w.nrows - 1;
    nB = (loc_last - loc_first + BKV) / BKV;
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKp,
                   const __grid_constant__ CUtensorMap tmVp, const __grid_constant__ CUtensorMap tmKl,
                   const __grid_constant__ CUtensorMap tmVl, TcParams p) {
    using C = TcCfg<HD>;
    // all shared memory is dynamic (no static arrays), so the base is 1024-byte aligned
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem;
    uint8_t* sP = sQ + C::kQBytes;
    uint8_t* sK = sP + C::kPBytes;                       // [kKStages][BKV x HD]
    uint8_t* sV = sK + C::kKStages * C::kKBytes;         // [kVStages][BKV x HD]
    float (*red_max)[2][BQ] = reinterpret_cast<float (*)[2][BQ]>(sV + C::kVStages * C::kVBytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(red_max) + C::kRedBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;    // [3]
    uint64_t* k_empty = bars + 5;   // [3]
    uint64_t* v_full = bars + 8;    // [2]
    uint64_t* v_empty = bars + 10;  // [2]
    uint64_t* s_full = bars + 12;   // [2]
    uint64_t* s_empty = bars + 14;  // [2]
    uint64_t* p_full = bars + 16;
    uint64_t* p_empty = bars + 17;
    uint64_t* o_full = bars + 18;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_items = p.n_work * p.heads;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmKp);
        ptx::tma_prefetch_desc(&tmVp);
        ptx::tma_prefetch_desc(&tmKl);
        ptx::tma_prefetch_desc(&tmVl);
        ptx::mbar_init(q_full, 1);
        ptx::mbar_init(q_empty, 1);
        for (int i = 0; i < C::kKStages; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&s_empty[i], 256);
        }
        ptx::mbar_init(p_full, 256);
        ptx::mbar_init(p_empty, 1);
        ptx::mbar_init(o_full, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // warp 0: Q + K loader (3-stage ring), warp 3: V loader (2-stage ring)
        if (lane == 0) {
            const bool kload = warp == 0;
            uint32_t g = 0, it = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                const int h = item / p.n_work;
                const AttnWork w = p.work[item % p.n_work];
                int nA, nB, loc_first;
                item_blocks(w, p.seg_lo, nA, nB, loc_first);
                if (kload) {
                    ptx::mbar_wait(q_empty, (it & 1) ^ 1);
                    ptx::mbar_expect_tx(q_full, C::kQBytes);
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s)
                        ptx::tma_load_2d(sQ + s * (BQ * 128), &tmQ, q_full, h * HD + s * 64, w.row0);
                }
                for (int b = 0; b < nA + nB; ++b, ++g) {
                    const bool pfx = b < nA;
                    const int row = pfx ? w.pfx_kv0 + b * BKV : loc_first + (b - nA) * BKV;
                    if (kload) {
                        const int st = g % C::kKStages;
                        ptx::mbar_wait(&k_empty[st], ((g / C::kKStages) & 1) ^ 1);
                        ptx::mbar_expect_tx(&k_full[st], C::kKBytes);
                        uint8_t* dst = sK + st * C::kKBytes;
#pragma unroll
                        for (int s = 0; s < C::kSub; ++s)
                            ptx::tma_load_2d(dst + s * (BKV * 128), pfx ? &tmKp : &tmKl, &k_full[st],
                                             h * HD + s * 64, row);
                    } else {
                        const int st = g & 1;
                        ptx::mbar_wait(&v_empty[st], ((g >> 1) & 1) ^ 1);
                        ptx::mbar_expect_tx(&v_full[st], C::kVBytes);
                        uint8_t* dst = sV + st * C::kVBytes;
#pragma unroll
                        for (int s = 0; s < C::kSub; ++s)
                            ptx::tma_load_2d(dst + s * (BKV * 128), pfx ? &tmVp : &tmVl, &v_full[st],
                                             h * HD + s * 64, row);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
            constexpr uint32_t idO = ptx::idesc_bf16_f32_bmn(BQ, HD);
            const uint32_t q_addr = ptx::smem_u32(sQ), p_addr = ptx::smem_u32(sP);
            uint32_t g = 0, it = 0;
            auto issue_pv = [&](uint32_t gb, bool first) {
                PROF_T0();
                ptx::mbar_wait(&v_full[gb & 1], (gb >> 1) & 1);
                PROF_ACC(0);
                ptx::mbar_wait(p_full, gb & 1);
                PROF_ACC(1);
                ptx::tc_fence_after();
                const uint32_t v_addr = ptx::smem_u32(sV + (gb & 1) * C::kVBytes);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    uint64_t ad = ptx::umma_desc_sw128(p_addr + (kk / 4) * (BQ * 128) + (kk % 4) * 32);
                    uint64_t bd = ptx::umma_desc_sw128_lbo(v_addr + kk * 16 * 128, BKV * 128, 1024);
                    ptx::mma_bf16(tmem_base + C::kO, ad, bd, idO, (!first || kk > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&v_empty[gb & 1]);
                ptx::mma_commit(p_empty);
            };
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                const AttnWork w = p.work[item % p.n_work];
                int nA, nB, loc_first;
                item_blocks(w, p.seg_lo, nA, nB, loc_first);
                const int nb = nA + nB;
                ptx::mbar_wait(q_full, it & 1);
                for (int b = 0; b < nb; ++b, ++g) {
                    const int st = g & 1;
                    const int ks = g % C::kKStages;
                    PROF_T0();
                    ptx::mbar_wait(&k_full[ks], (g / C::kKStages) & 1);
                    PROF_ACC(2);
                    ptx::mbar_wait(&s_empty[st], ((g >> 1) & 1) ^ 1);
                    PROF_ACC(3);
                    ptx::tc_fence_after();
                    const uint32_t k_addr = ptx::smem_u32(sK + ks * C::kKBytes);
#pragma unroll
                    for (int kc = 0; kc < HD / 16; ++kc) {
                        uint64_t ad = ptx::umma_desc_sw128(q_addr + (kc / 4) * (BQ * 128) + (kc % 4) * 32);
                        uint64_t bd = ptx::umma_desc_sw128(k_addr + (kc / 4) * (BKV * 128) + (kc % 4) * 32);
                        ptx::mma_bf16(tmem_base + st * BKV, ad, bd, idS, kc > 0 ? 1u : 0u);
                    }
                    ptx::mma_commit(&s_full[st]);
                    ptx::mma_commit(&k_empty[ks]);
                    if (b == nb - 1) ptx::mma_commit(q_empty);
                    if (b >= 1) issue_pv(g - 1, b - 1 == 0);
                }
                issue_pv(g - 1, nb == 1);
                ptx::mma_commit(o_full);
            }
        }
    } else if (warp >= 4) {
        // two softmax warpgroups split each row's 128 keys (and O's HD columns) in halves;
        // thread pairs (r, half 0/1) agree on the row max through smem once per block
        const int half = (warp - 4) >> 2;
        const int r = (threadIdx.x - 128) & (BQ - 1);  // query row within the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>(((warp - 4) & 3) * 32) << 16;
        constexpr int KH = BKV / 2;  // keys per thread
        constexpr int OH = HD / 2;   // O columns per thread
        uint32_t g = 0, it = 0;
        // P row r inside the swizzled [128 x 128] bf16 tile: this half = one 64-key sub-tile
        uint8_t* prow = sP + half * (BQ * 128) + (r >> 3) * 1024 + (r & 7) * 128;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
            const int h = item / p.n_work;
            const AttnWork w = p.work[item % p.n_work];
            int nA, nB, loc_first;
            item_blocks(w, p.seg_lo, nA, nB, loc_first);
            const int nb = nA + nB;
            const bool valid = r < w.nrows;
            const int row = w.row0 + r;
            const int seg = valid ? p.seg_lo[row] : 0x7fffffff;
            float m = -INFINITY, l = 0.f;
            for (int b = 0; b < nb; ++b, ++g) {
                const int st = g & 1;
#ifdef SGC_ATTN_PROF
                const bool prof_thr = threadIdx.x == 128;
                long long _pt = clock64();
#define SPROF(slot)                                                                            \
    if (prof_thr) {                                                                            \
        long long _n = clock64();                                                              \
        atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 16 + (slot)], (unsigned long long)(_n - _pt)); \
        _pt = _n;                                                                              \
    }
#else
#define SPROF(slot)
#endif
                ptx::mbar_wait(&s_full[st], (g >> 1) & 1);
                SPROF(4);
                ptx::tc_fence_after();
                float s[KH];
#pragma unroll
                for (int c = 0; c < KH / 32; ++c)
                    ptx::tmem_ld32(tmem_base + lane_base + st * BKV + half * KH + c * 32,
                                   *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&s_empty[st]);
                SPROF(5);
                // visible key window [klo, khi] of this row, in block-local key index
                int k0, klo, khi;
                if (b < nA) {
                    k0 = b * BKV;
                    klo = 0;
                    khi = valid ? min(BKV, w.pfx_len - k0) - 1 : -1;
                } else {
                    k0 = loc_first + (b - nA) * BKV;
                    klo = max(0, seg - k0);
                    khi = valid ? min(BKV - 1, row - k0) : -1;
                }
                const int cb = half * KH;
                // fast path (interior prefix blocks): no masking, scale folded into the FFMA
                const bool full = klo <= cb && khi >= cb + KH - 1;
                float mx;
                if (full) {
                    float m4[4] = {s[0], s[1], s[2], s[3]};  // 4 independent chains
#pragma unroll
                    for (int j = 4; j < KH; ++j) m4[j & 3] = fmaxf(m4[j & 3], s[j]);
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])) * p.scale_log2;
                } else {
                    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int j = 0; j < KH; ++j) {
                        s[j] = (cb + j >= klo && cb + j <= khi) ? s[j] * p.scale_log2 : -INFINITY;
                        m4[j & 3] = fmaxf(m4[j & 3], s[j]);
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                }
                SPROF(6);
                red_max[st][half][r] = mx;
                named_bar_sync(1, 256);
                mx = fmaxf(mx, red_max[st][half ^ 1][r]);
                SPROF(7);
                // lazy rescale: keep the running max unless it grows by more than 8 (2^8)
                float alpha = 1.f;
                bool rescale = false;
                if (mx > -INFINITY) {
                    if (m == -INFINITY) {
                        m = mx;  // O and l are still zero
                    } else if (mx > m + 8.f) {
                        alpha = ex2_approx(m - mx);
                        m = mx;
                        rescale = true;
                    }
                }
                float rs = 0.f;
                uint32_t pk[KH / 2];
                if (m == -INFINITY) {
#pragma unroll
                    for (int j = 0; j < KH / 2; ++j) pk[j] = 0u;
                } else if (full) {
                    const float sc = p.scale_log2, nm = -m;
                    float rs2[2] = {0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < KH / 2; ++j) {
                        const float xa = fmaf(s[2 * j], sc, nm), xc = fmaf(s[2 * j + 1], sc, nm);
                        // ~30% of the exponentials on the FMA pipe, the rest on MUFU
                        const bool emu = (j % 3) == 2;
                        float a = emu ? ex2_poly(xa) : ex2_approx(xa);
                        float c = emu ? ex2_poly(xc) : ex2_approx(xc);
                        rs2[j & 1] += a + c;
                        __nv_bfloat162 v = __floats2bfloat162_rn(a, c);
                        pk[j] = *reinterpret_cast<uint32_t*>(&v);
                    }
                    rs = rs2[0] + rs2[1];
                } else {
#pragma unroll
                    for (int j = 0; j < KH / 2; ++j) {
                        float a = ex2_approx(s[2 * j] - m), c = ex2_approx(s[2 * j + 1] - m);
                        rs += a + c;
                        __nv_bfloat162 v = __floats2bfloat162_rn(a, c);
                        pk[j] = *reinterpret_cast<uint32_t*>(&v);
                    }
                }
                l = l * alpha + rs;  // this half's share of the row sum
                SPROF(8);
                // P buffer free and O stable once PV of the previous block completed
                ptx::mbar_wait(p_empty, (g & 1) ^ 1);
                SPROF(9);
                ptx::tc_fence_after();
                if (rescale && b > 0) {
#pragma unroll 1
                    for (int c = 0; c < OH / 32; ++c) {
                        uint32_t o[32];
                        const uint32_t ta = tmem_base + lane_base + C::kO + half * OH + c * 32;
                        ptx::tmem_ld32(ta, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                        ptx::tmem_st32(ta, o);
                    }
                    ptx::tmem_st_wait();
                }
                // P half-row: 8 chunks of 8 keys (16 B) with the 128B XOR swizzle
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    uint4 v = make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
                    *reinterpret_cast<uint4*>(prow + ((cc ^ (r & 7)) << 4)) = v;
                }
                SPROF(10);
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                ptx::mbar_arrive(p_full);
                SPROF(11);

            }
            // epilogue: O / l -> bf16 (each half stores HD/2 columns); the row sums are
            // exchanged through red_max[0] once both halves are past their last max exchange
            named_bar_sync(1, 256);
            red_max[0][half][r] = l;
            named_bar_sync(1, 256);
            const float lt = l + red_max[0][half ^ 1][r];
            ptx::mbar_wait(o_full, it & 1);
            ptx::tc_fence_after();
            const float il = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll 1
            for (int c = 0; c < OH / 32; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32(tmem_base + lane_base + C::kO + half * OH + c * 32, o);
                ptx::tmem_ld_wait();
                if (valid) {
                    uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<size_t>(row) * p.d + h * HD +
                                                          half * OH + c * 32);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t wv[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(o[8 * q + 2 * e]) * il,
                                                                     __uint_as_float(o[8 * q + 2 * e + 1]) * il);
                            wv[e] = *reinterpret_cast<uint32_t*>(&v);
                        }
                        dst[q] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                    }
                }
            }
            ptx::tc_fence_before();
            named_bar_sync(1, 256);  // red_max[0] is reused by the next item
        }
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

template <int HD>
void launch_tc(Ctx* c, const AttnParams& a, int n_work, int heads, int q_rows, int pfx_rows, int loc_rows) {
    using Cf = TcCfg<HD>;
    auto kfn = attn_tc_kernel<HD>;
    static bool attr = false;
    if (!attr) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem));
        attr = true;
    }
    const int d = a.d;
    CUtensorMap tq = make_map_2d(a.q, q_rows, d, BQ, 64);
    CUtensorMap tkp = make_map_2d(a.k_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tvp = make_map_2d(a.v_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tkl = make_map_2d(a.k_loc, loc_rows, d, BKV, 64);
    CUtensorMap tvl = make_map_2d(a.v_loc, loc_rows, d, BKV, 64);
    TcParams p{a.work, n_work, heads, a.seg_lo, a.out, d, a.scale * 1.4426950408889634f};
    const int items = n_work * heads;
    const int grid = items < c->num_sms ? items : c->num_sms;
    Ctx::Timed timer(c, "attention");
    kfn<<<grid, kThreads, Cf::kSmem, c->stream>>>(tq, tkp, tvp, tkl, tvl, p);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace

#ifdef SGC_ATTN_PROF
void attn_prof_read(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_attn_prof, sizeof(unsigned long long) * 148 * 16);
}
void attn_prof_reset() {
    static unsigned long long z[148 * 16] = {};
    cudaMemcpyToSymbol(g_attn_prof, z, sizeof(z));
}
#endif

bool cascade_attention_tc(Ctx* c, const AttnParams& p, int n_work, int heads, int hd, int q_rows,
                          int pfx_rows, int loc_rows) {
    if (n_work <= 0) return true;
    if (p.loc_kv0 != 0) return false;
    switch (hd) {
        case 64: launch_tc<64>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows); return true;
        case 128: launch_tc<128>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows); return true;
        default: return false;
    }
}

}  // namespace sgc
