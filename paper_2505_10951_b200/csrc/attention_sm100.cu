// attention_sm100.cu -- tcgen05/TMEM/TMA cascade attention for sm_100a (head_dim 64 / 128).
//
// Same semantics as attention.cu (lm_core.cpp:246-274: one softmax over the sealed prefix keys
// followed by the row's own causal suffix keys), re-laid out for the 5th-gen tensor cores:
//
//   warp 0      TMA loader: Q tile (128 rows) once per item; K and V blocks (128 keys) of the
//               cluster's prefix (phase A) then of the batch's own rows (phase B), 2-stage ring
//   warp 1      MMA issuer (one thread): S_b = Q K_b^T into a double-buffered TMEM S, and
//               O += P_{b-1} V_{b-1} into TMEM O (P from smem, V as an MN-major operand)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4..7  softmax: thread r owns query row r (TMEM lane r). Reads its S row from TMEM,
//               masks, online softmax in base 2 with lazy O rescale (only when the running max
//               grows by > 2^8), writes its P row (bf16, 128B-swizzled) for the PV MMA, and at
//               the end normalizes its O row and stores it.
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
constexpr int kThreads = 256;

template <int HD>
struct TcCfg {
    static constexpr int kSub = HD / 64;            // 64-element (128 B) swizzle sub-tiles
    static constexpr int kQBytes = BQ * HD * 2;
    static constexpr int kKBytes = BKV * HD * 2;
    static constexpr int kVBytes = BKV * HD * 2;
    static constexpr int kPBytes = BQ * BKV * 2;
    static constexpr int kStageBytes = kKBytes + kVBytes;
    static constexpr int kSmem = 1024 + kQBytes + kPBytes + 2 * kStageBytes + 256;
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kO = 256;             // TMEM column of the O accumulator
};

struct TcParams {
    const AttnWork* work;
    int n_work, heads;
    const int32_t* seg_lo;
    __nv_bfloat16* out;
    int d;
    float scale_log2;
};

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
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem;
    uint8_t* sP = sQ + C::kQBytes;
    uint8_t* sKV = sP + C::kPBytes;  // stage s: K at sKV + s*kStageBytes, V right after K
    uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + 2 * C::kStageBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* kv_full = bars + 2;   // [2]
    uint64_t* kv_empty = bars + 4;  // [2]
    uint64_t* s_full = bars + 6;    // [2]
    uint64_t* s_empty = bars + 8;   // [2]
    uint64_t* p_full = bars + 10;
    uint64_t* p_empty = bars + 11;
    uint64_t* o_full = bars + 12;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

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
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&kv_full[i], 1);
            ptx::mbar_init(&kv_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&s_empty[i], 128);
        }
        ptx::mbar_init(p_full, 128);
        ptx::mbar_init(p_empty, 1);
        ptx::mbar_init(o_full, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t g = 0, it = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                const int h = item / p.n_work;
                const AttnWork w = p.work[item % p.n_work];
                int nA, nB, loc_first;
                item_blocks(w, p.seg_lo, nA, nB, loc_first);
                ptx::mbar_wait(q_empty, (it & 1) ^ 1);
                ptx::mbar_expect_tx(q_full, C::kQBytes);
#pragma unroll
                for (int s = 0; s < C::kSub; ++s)
                    ptx::tma_load_2d(sQ + s * (BQ * 128), &tmQ, q_full, h * HD + s * 64, w.row0);
                for (int b = 0; b < nA + nB; ++b, ++g) {
                    const int st = g & 1;
                    ptx::mbar_wait(&kv_empty[st], ((g >> 1) & 1) ^ 1);
                    ptx::mbar_expect_tx(&kv_full[st], C::kStageBytes);
                    uint8_t* sK = sKV + st * C::kStageBytes;
                    uint8_t* sV = sK + C::kKBytes;
                    const bool pfx = b < nA;
                    const int row = pfx ? w.pfx_kv0 + b * BKV : loc_first + (b - nA) * BKV;
                    const CUtensorMap* mk = pfx ? &tmKp : &tmKl;
                    const CUtensorMap* mv = pfx ? &tmVp : &tmVl;
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s) {
                        ptx::tma_load_2d(sK + s * (BKV * 128), mk, &kv_full[st], h * HD + s * 64, row);
                        ptx::tma_load_2d(sV + s * (BKV * 128), mv, &kv_full[st], h * HD + s * 64, row);
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
                ptx::mbar_wait(p_full, gb & 1);
                ptx::tc_fence_after();
                const uint32_t v_addr = ptx::smem_u32(sKV + (gb & 1) * C::kStageBytes + C::kKBytes);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    uint64_t ad = ptx::umma_desc_sw128(p_addr + (kk / 4) * (BQ * 128) + (kk % 4) * 32);
                    uint64_t bd = ptx::umma_desc_sw128_lbo(v_addr + kk * 16 * 128, BKV * 128, 1024);
                    ptx::mma_bf16(tmem_base + C::kO, ad, bd, idO, (!first || kk > 0) ? 1u : 0u);
                }
                ptx::mma_commit(&kv_empty[gb & 1]);
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
                    ptx::mbar_wait(&kv_full[st], (g >> 1) & 1);
                    ptx::mbar_wait(&s_empty[st], ((g >> 1) & 1) ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t k_addr = ptx::smem_u32(sKV + st * C::kStageBytes);
#pragma unroll
                    for (int kc = 0; kc < HD / 16; ++kc) {
                        uint64_t ad = ptx::umma_desc_sw128(q_addr + (kc / 4) * (BQ * 128) + (kc % 4) * 32);
                        uint64_t bd = ptx::umma_desc_sw128(k_addr + (kc / 4) * (BKV * 128) + (kc % 4) * 32);
                        ptx::mma_bf16(tmem_base + st * BKV, ad, bd, idS, kc > 0 ? 1u : 0u);
                    }
                    ptx::mma_commit(&s_full[st]);
                    if (b == nb - 1) ptx::mma_commit(q_empty);
                    if (b >= 1) issue_pv(g - 1, b - 1 == 0);
                }
                issue_pv(g - 1, nb == 1);
                ptx::mma_commit(o_full);
            }
        }
    } else if (warp >= 4) {
        const int r = threadIdx.x - 128;  // query row within the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp - 4) * 32) << 16;
        uint32_t g = 0, it = 0;
        // P row r inside the swizzled [128 x 128] bf16 tile (two 64-key sub-tiles)
        uint8_t* prow = sP + (r >> 3) * 1024 + (r & 7) * 128;
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
                ptx::mbar_wait(&s_full[st], (g >> 1) & 1);
                ptx::tc_fence_after();
                float s[BKV];
#pragma unroll
                for (int c = 0; c < BKV / 32; ++c)
                    ptx::tmem_ld32(tmem_base + lane_base + st * BKV + c * 32,
                                   *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&s_empty[st]);
                // mask + scale (base-2 logits)
                float mx = -INFINITY;
                if (b < nA) {
                    const int kend = w.pfx_len - b * BKV;
#pragma unroll
                    for (int j = 0; j < BKV; ++j) {
                        s[j] = (valid && j < kend) ? s[j] * p.scale_log2 : -INFINITY;
                        mx = fmaxf(mx, s[j]);
                    }
                } else {
                    const int k0 = loc_first + (b - nA) * BKV;
#pragma unroll
                    for (int j = 0; j < BKV; ++j) {
                        const int key = k0 + j;
                        s[j] = (key >= seg && key <= row) ? s[j] * p.scale_log2 : -INFINITY;
                        mx = fmaxf(mx, s[j]);
                    }
                }
                // lazy rescale: keep the running max unless it grows by more than 8 (2^8)
                float alpha = 1.f;
                bool rescale = false;
                if (mx > -INFINITY) {
                    if (m == -INFINITY) {
                        m = mx;  // O and l are still zero
                    } else if (mx > m + 8.f) {
                        alpha = exp2f(m - mx);
                        m = mx;
                        rescale = true;
                    }
                }
                float rs = 0.f;
                uint32_t pk[BKV / 2];
                if (m == -INFINITY) {
#pragma unroll
                    for (int j = 0; j < BKV / 2; ++j) pk[j] = 0u;
                } else {
#pragma unroll
                    for (int j = 0; j < BKV / 2; ++j) {
                        float a = exp2f(s[2 * j] - m), c = exp2f(s[2 * j + 1] - m);
                        rs += a + c;
                        __nv_bfloat162 v = __floats2bfloat162_rn(a, c);
                        pk[j] = *reinterpret_cast<uint32_t*>(&v);
                    }
                }
                l = l * alpha + rs;
                // P buffer free and O stable once PV of the previous block completed
                ptx::mbar_wait(p_empty, (g & 1) ^ 1);
                ptx::tc_fence_after();
                if (rescale && b > 0) {
#pragma unroll 1
                    for (int c = 0; c < HD / 32; ++c) {
                        uint32_t o[32];
                        const uint32_t ta = tmem_base + lane_base + C::kO + c * 32;
                        ptx::tmem_ld32(ta, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                        ptx::tmem_st32(ta, o);
                    }
                    ptx::tmem_st_wait();
                }
                // P row: 16 chunks of 8 keys (16 B), sub-tile = chunk / 8, 128B XOR swizzle
#pragma unroll
                for (int q = 0; q < BKV / 8; ++q) {
                    const int sub = q >> 3, cc = q & 7;
                    uint4 v = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    *reinterpret_cast<uint4*>(prow + sub * (BQ * 128) + ((cc ^ (r & 7)) << 4)) = v;
                }
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                ptx::mbar_arrive(p_full);
            }
            // epilogue: O / l -> bf16
            ptx::mbar_wait(o_full, it & 1);
            ptx::tc_fence_after();
            const float il = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
            for (int c = 0; c < HD / 32; ++c) {
                uint32_t o[32];
                ptx::tmem_ld32(tmem_base + lane_base + C::kO + c * 32, o);
                ptx::tmem_ld_wait();
                if (valid) {
                    uint4* dst = reinterpret_cast<uint4*>(p.out + static_cast<size_t>(row) * p.d + h * HD + c * 32);
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
