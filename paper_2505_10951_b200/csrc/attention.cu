// attention.cu -- shared-prefix ("cascade") flash attention for the ToyLm (lm_core.cpp:246-274).
//
// One kernel serves both hot-path attention shapes:
//   * representative prefill: each row attends causally to its own sequence (no prefix);
//   * per-query reuse (members): each row attends to its cluster's sealed prefix KV (all
//     P keys, non-causal) and then causally to its own member's suffix keys.
// A CTA owns a tile of up to 64 query rows of ONE cluster and one head; it streams the
// cluster's prefix K/V once for all member rows in the tile (phase A), then the tile's
// local suffix keys with a block-diagonal causal mask (phase B). Online softmax keeps both
// phases in one pass, so the two-segment attention of the reference (prefix keys, then
// suffix keys, one softmax) is reproduced exactly up to fp32 rounding.
//
// Tensor cores: mma.sync.m16n8k16 bf16 -> fp32 (4 warps x 16 rows). K/V tiles are staged
// with cp.async (zero-filled out of range) in a double-buffered smem ring.
#include "attention.cuh"
#include "common.cuh"
#include "sm100_ptx.cuh"

namespace sgc {
namespace {

constexpr int TQ = 64;   // query rows per CTA
constexpr int TK = 64;   // keys per block
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ void ldsm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                        const void* p) {
    uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(s));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                          const void* p) {
    uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(s));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t& r0, uint32_t& r1, const void* p) {
    uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "r"(s));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD>
struct Smem {
    static constexpr int LD = HD + 8;  // padded row (bf16 elements) -> conflict-free ldmatrix
    static constexpr int kTile = TK * LD;
    static constexpr int kQ = TQ * LD;
    static constexpr int kBytes = (kQ + 4 * kTile) * 2;
};

// load a [64 x HD] K or V block (rows kv0 .. kv0+63 of a [rows x d] bf16 matrix, head col c0)
template <int HD>
__device__ __forceinline__ void load_block(__nv_bfloat16* dst, const __nv_bfloat16* src, int d,
                                           int c0, int kv0, int nvalid) {
    constexpr int LD = Smem<HD>::LD;
    constexpr int CH = HD / 8;  // 16-byte chunks per row
    for (int i = threadIdx.x; i < TK * CH; i += kThreads) {
        int r = i / CH, c = i % CH;
        bool v = r < nvalid;
        const __nv_bfloat16* g = src + static_cast<size_t>(v ? kv0 + r : kv0) * d + c0 + c * 8;
        cp_async16(dst + r * LD + c * 8, g, v);
    }
}

template <int HD>
__global__ void __launch_bounds__(kThreads)
    cascade_attn_kernel(AttnParams p) {
    constexpr int LD = Smem<HD>::LD;
    constexpr int KC = HD / 16;  // k-chunks of the QK^T product
    constexpr int NO = HD / 8;   // n-tiles of the output
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
    __nv_bfloat16* const sK0 = sQ + Smem<HD>::kQ;                         // K ring: 2 blocks
    __nv_bfloat16* const sV0 = sQ + Smem<HD>::kQ + 2 * Smem<HD>::kTile;   // V ring: 2 blocks
#define sK(b) (sK0 + (b) * Smem<HD>::kTile)
#define sV(b) (sV0 + (b) * Smem<HD>::kTile)

    const AttnWork w = p.work[blockIdx.x];
    const int h = blockIdx.y;
    const int d = p.d;
    const int c0 = h * HD;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int g = lane / 4, t = lane % 4;

    // ---- Q tile -> registers (A fragments)
    for (int i = threadIdx.x; i < TQ * (HD / 8); i += kThreads) {
        int r = i / (HD / 8), c = i % (HD / 8);
        bool v = r < w.nrows;
        cp_async16(sQ + r * LD + c * 8, p.q + static_cast<size_t>(w.row0 + (v ? r : 0)) * d + c0 + c * 8, v);
    }
    cp_commit();

    // my two rows
    const int r_lo = warp * 16 + g, r_hi = r_lo + 8;
    const int row_lo = w.row0 + r_lo, row_hi = w.row0 + r_hi;
    const bool ok_lo = r_lo < w.nrows, ok_hi = r_hi < w.nrows;
    const int seg_lo_lo = ok_lo ? p.seg_lo[row_lo] : 0x7fffffff;
    const int seg_lo_hi = ok_hi ? p.seg_lo[row_hi] : 0x7fffffff;

    const float sl2 = p.scale * 1.4426950408889634f;  // softmax in base 2
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    float o[NO][4];
#pragma unroll
    for (int j = 0; j < NO; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;

    // key blocks: phase A = prefix blocks [0, nA), phase B = local blocks
    const int nA = (w.pfx_len + TK - 1) / TK;
    const int loc_first = p.seg_lo[w.row0];  // earliest key row any tile row can see
    const int loc_last = w.row0 + w.nrows - 1;
    const int nB = (loc_last - loc_first + TK) / TK;
    const int nblk = nA + nB;

    auto issue = [&](int b, int buf) {
        if (b < nA) {
            int k0 = b * TK;  // a 64-key block never straddles a 128-token page
            int nv = min(TK, w.pfx_len - k0);
            const int row = kv_row_of(p.bt, w.pfx_off, k0);
            load_block<HD>(sK(buf), p.k_pfx, d, c0, row, nv);
            load_block<HD>(sV(buf), p.v_pfx, d, c0, row, nv);
        } else {
            int k0 = loc_first + (b - nA) * TK;
            int nv = min(TK, loc_last + 1 - k0);
            const int row = w.loc_bt >= 0 ? kv_row_of(p.bt, w.loc_bt, (b - nA) * TK) : p.loc_kv0 + k0;
            load_block<HD>(sK(buf), p.k_loc, d, c0, row, nv);
            load_block<HD>(sV(buf), p.v_loc, d, c0, row, nv);
        }
        cp_commit();
    };

    if (nblk > 0) issue(0, 0);
    cp_wait<1>();
    __syncthreads();
    uint32_t qa[KC][4];
#pragma unroll
    for (int kc = 0; kc < KC; ++kc) {
        const __nv_bfloat16* ptr = sQ + (warp * 16 + (lane % 16)) * LD + kc * 16 + (lane / 16) * 8;
        ldsm_x4(qa[kc][0], qa[kc][1], qa[kc][2], qa[kc][3], ptr);
    }

    for (int b = 0; b < nblk; ++b) {
        const int buf = b & 1;
        if (b + 1 < nblk) {
            issue(b + 1, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();

        // S = Q K^T : 16 rows x 64 keys per warp
        float s[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) {
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) {  // two key n-tiles per ldmatrix.x4
                uint32_t b0, b1, b2, b3;
                const __nv_bfloat16* ptr =
                    sK(buf) + (jp * 16 + (lane / 16) * 8 + (lane % 8)) * LD + kc * 16 + ((lane / 8) % 2) * 8;
                ldsm_x4(b0, b1, b2, b3, ptr);
                mma16816(s[2 * jp], qa[kc], b0, b1);
                mma16816(s[2 * jp + 1], qa[kc], b2, b3);
            }
        }

        // masks
        const bool is_pfx = b < nA;
        int kbase;  // key index of column 0 in this block (prefix index or local row)
        int kvalid;
        if (is_pfx) {
            kbase = b * TK;
            kvalid = w.pfx_len;
        } else {
            kbase = loc_first + (b - nA) * TK;
            kvalid = 0;
        }
        float mx_lo = -INFINITY, mx_hi = -INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int key = kbase + j * 8 + 2 * t + e;
                bool v_lo, v_hi;
                if (is_pfx) {
                    v_lo = ok_lo && key < kvalid;
                    v_hi = ok_hi && key < kvalid;
                } else {
                    v_lo = key >= seg_lo_lo && key <= row_lo;
                    v_hi = key >= seg_lo_hi && key <= row_hi;
                }
                s[j][e] = v_lo ? s[j][e] * sl2 : -INFINITY;
                s[j][2 + e] = v_hi ? s[j][2 + e] * sl2 : -INFINITY;
                mx_lo = fmaxf(mx_lo, s[j][e]);
                mx_hi = fmaxf(mx_hi, s[j][2 + e]);
            }
        }
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffff, mx_lo, 1));
        mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffff, mx_lo, 2));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffff, mx_hi, 1));
        mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffff, mx_hi, 2));
        const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
        const float sh_lo = mn_lo == -INFINITY ? 0.f : mn_lo;
        const float sh_hi = mn_hi == -INFINITY ? 0.f : mn_hi;
        const float a_lo = exp2f(m_lo - sh_lo), a_hi = exp2f(m_hi - sh_hi);
        m_lo = mn_lo;
        m_hi = mn_hi;
        float rs_lo = 0.f, rs_hi = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            s[j][0] = exp2f(s[j][0] - sh_lo);
            s[j][1] = exp2f(s[j][1] - sh_lo);
            s[j][2] = exp2f(s[j][2] - sh_hi);
            s[j][3] = exp2f(s[j][3] - sh_hi);
            rs_lo += s[j][0] + s[j][1];
            rs_hi += s[j][2] + s[j][3];
        }
        l_lo = l_lo * a_lo + rs_lo;
        l_hi = l_hi * a_hi + rs_hi;
#pragma unroll
        for (int j = 0; j < NO; ++j) {
            o[j][0] *= a_lo;
            o[j][1] *= a_lo;
            o[j][2] *= a_hi;
            o[j][3] *= a_hi;
        }
        // O += P V  (P from the S accumulators, 16 keys per k-chunk)
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
            uint32_t pa[4];
            pa[0] = pack2(s[2 * kc][0], s[2 * kc][1]);
            pa[1] = pack2(s[2 * kc][2], s[2 * kc][3]);
            pa[2] = pack2(s[2 * kc + 1][0], s[2 * kc + 1][1]);
            pa[3] = pack2(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
            for (int jp = 0; jp < NO / 2; ++jp) {  // two hd n-tiles per ldmatrix.x4.trans
                uint32_t b0, b1, b2, b3;
                const __nv_bfloat16* ptr = sV(buf) + (kc * 16 + (lane % 8) + ((lane / 8) % 2) * 8) * LD +
                                           jp * 16 + (lane / 16) * 8;
                ldsm_x4_t(b0, b1, b2, b3, ptr);
                mma16816(o[2 * jp], pa, b0, b1);
                mma16816(o[2 * jp + 1], pa, b2, b3);
            }
            if constexpr (NO % 2 == 1) {
                uint32_t b0, b1;
                const __nv_bfloat16* ptr =
                    sV(buf) + (kc * 16 + (lane % 8) + ((lane / 8) % 2) * 8) * LD + (NO - 1) * 8;
                ldsm_x2_t(b0, b1, ptr);
                mma16816(o[NO - 1], pa, b0, b1);
            }
        }
        __syncthreads();  // buffer `buf` is refilled by the next iteration's issue()
    }

#undef sK
#undef sV
    // finalize: row sums across the quad, normalize, store bf16
    l_lo += __shfl_xor_sync(0xffffffff, l_lo, 1);
    l_lo += __shfl_xor_sync(0xffffffff, l_lo, 2);
    l_hi += __shfl_xor_sync(0xffffffff, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffff, l_hi, 2);
    const float il_lo = l_lo > 0.f ? 1.f / l_lo : 0.f;
    const float il_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
#pragma unroll
    for (int j = 0; j < NO; ++j) {
        const int col = c0 + j * 8 + 2 * t;
        if (ok_lo)
            *reinterpret_cast<uint32_t*>(p.out + static_cast<size_t>(row_lo) * d + col) =
                pack2(o[j][0] * il_lo, o[j][1] * il_lo);
        if (ok_hi)
            *reinterpret_cast<uint32_t*>(p.out + static_cast<size_t>(row_hi) * d + col) =
                pack2(o[j][2] * il_hi, o[j][3] * il_hi);
    }
}

template <int HD>
void launch(Ctx* c, const AttnParams& p, int n_work, int heads) {
    auto kfn = cascade_attn_kernel<HD>;
    static bool attr = false;
    if (!attr) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            Smem<HD>::kBytes));
        attr = true;
    }
    dim3 grid(n_work, heads);
    Ctx::Timed timer(c, "attention");
    kfn<<<grid, kThreads, Smem<HD>::kBytes, c->stream>>>(p);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace

void cascade_attention(Ctx* c, const AttnParams& p, int n_work, int heads, int hd) {
    if (n_work <= 0) return;
    switch (hd) {
        case 16: launch<16>(c, p, n_work, heads); break;
        case 32: launch<32>(c, p, n_work, heads); break;
        case 64: launch<64>(c, p, n_work, heads); break;
        case 128: launch<128>(c, p, n_work, heads); break;
        default: fail(SGC_DOMAIN, "attention: head_dim must be 16, 32, 64 or 128");
    }
}

// ---- decode step: each row's own keys (+ merge with the prefix partial) ------------------
// One warp per (row, head). Keys are visited 32 at a time, one key per lane: the lane's score
// is a full dot product (uint4 loads of its key row, q broadcast from shared memory), the chunk
// is folded into an online softmax in scaled-log2 units, and O += P V with lane i holding dims
// [i*DPL, i*DPL + DPL) (p_j broadcast by shuffle, V rows read coalesced). Ranges in order:
// the prefix (only when no tcgen05 partial is given), the question suffix, the generated
// tokens. Finally merged with the prefix partial:
//   out = (O1 2^(lse1 - M) + acc 2^(m2 - M)) / (2^(lse1 - M) + l2 2^(m2 - M)).
namespace {
#ifndef SGC_DECODE_LOCAL_MINB
#define SGC_DECODE_LOCAL_MINB 1
#endif
// warps per CTA of the own-key decode attention (consecutive heads of one row: a CTA reads
// SGC_DECODE_WPB x head_dim contiguous bytes of every key row). 32 = a whole 4096-wide key row
// per CTA at C3: 106-108 -> 88-90 ms per generation batch vs 8 (scripts/gpu_lib_gen_ab.sh)
#ifndef SGC_DECODE_WPB
#define SGC_DECODE_WPB 32
#endif
template <int HD>
__global__ void __launch_bounds__(32 * SGC_DECODE_WPB, SGC_DECODE_LOCAL_MINB) decode_local_kernel(DecodeAttnParams p) {
    constexpr int DPL = HD >= 32 ? HD / 32 : 1;
    __shared__ float qs[SGC_DECODE_WPB][HD];
    const int wib = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int wg = blockIdx.x * SGC_DECODE_WPB + wib;
    if (wg >= p.rows * p.heads) return;  // warp-uniform; only __syncwarp below
    const int r = wg / p.heads, h = wg % p.heads;
    const float sl2 = p.scale * 1.4426950408889634f;
    const __nv_bfloat16* qrow = p.q + static_cast<size_t>(r) * p.d + h * HD;
    for (int i = lane; i < HD; i += 32) qs[wib][i] = __bfloat162float(qrow[i]) * sl2;
    __syncwarp();
    const bool act = lane * DPL < HD;
    const size_t col = static_cast<size_t>(h) * HD + (act ? lane * DPL : 0);
    float m = -INFINITY, l = 0.f, acc[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] = 0.f;
    // keys [0, n) of a range at rows lo.. (bt == nullptr) or through the block table bt at offset
    // lo; a 32-key chunk never straddles a 128-token page
    auto run = [&](const __nv_bfloat16* K, const __nv_bfloat16* V, int lo, int n, const int32_t* bt) {
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int key = k0 + lane;
            const int row0 = kv_row_of(bt, lo, k0);
            float sc = -INFINITY;
            if (key < n) {
                const __nv_bfloat16* kr = K + static_cast<size_t>(row0 + lane) * p.d + h * HD;
                float a0 = 0.f, a1 = 0.f;
                // the key row in 32-byte loads (LDG.256): all of them in flight before the math
                uint32_t u[HD / 16][8];
#pragma unroll
                for (int c = 0; c < HD / 16; ++c) ptx::ld_nc_u8(kr + 16 * c, u[c]);
#pragma unroll
                for (int c = 0; c < HD / 16; ++c) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[c][e]));
                        a0 = fmaf(qs[wib][c * 16 + 2 * e], f.x, a0);
                        a1 = fmaf(qs[wib][c * 16 + 2 * e + 1], f.y, a1);
                    }
                }
                sc = a0 + a1;
            }
            float cm = sc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
            const float mn = fmaxf(m, cm);
            const float alpha = m == -INFINITY ? 0.f : exp2f(m - mn);
            const float pk = key < n ? exp2f(sc - mn) : 0.f;
            float ps = pk;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l = l * alpha + ps;
#pragma unroll
            for (int i = 0; i < DPL; ++i) acc[i] *= alpha;
            const int nk = min(32, n - k0);
            const __nv_bfloat16* vb = V + static_cast<size_t>(row0) * p.d + col;
#pragma unroll 8
            for (int j = 0; j < nk; ++j) {
                const float pj = __shfl_sync(0xffffffffu, pk, j);
                if (act) {
                    const __nv_bfloat16* vr = vb + static_cast<size_t>(j) * p.d;
                    if constexpr (DPL == 4) {
                        const uint2 u = *reinterpret_cast<const uint2*>(vr);
                        const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
                        const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
                        acc[0] = fmaf(pj, f0.x, acc[0]);
                        acc[1] = fmaf(pj, f0.y, acc[1]);
                        acc[2] = fmaf(pj, f1.x, acc[2]);
                        acc[3] = fmaf(pj, f1.y, acc[3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < DPL; ++i) acc[i] = fmaf(pj, __bfloat162float(vr[i]), acc[i]);
                    }
                }
            }
            m = mn;
        }
    };
    if (!p.part_o && p.p_n) run(p.k_p, p.v_p, p.p_lo[r], p.p_n[r], p.p_bt);
    if (p.q_n) run(p.k_q, p.v_q, p.q_lo[r], p.q_n[r], nullptr);
    if (p.g_n) run(p.k_g, p.v_g, p.g_lo[r], p.g_n[r], nullptr);
    float o1[DPL], w1 = 0.f, w2 = 1.f, den = l;
#pragma unroll
    for (int i = 0; i < DPL; ++i) o1[i] = 0.f;
    if (p.part_o) {
        const float lse1 = p.part_lse[static_cast<size_t>(r) * p.heads + h];
        const float M = fmaxf(lse1, m);
        w1 = lse1 == -INFINITY ? 0.f : exp2f(lse1 - M);
        w2 = m == -INFINITY ? 0.f : exp2f(m - M);
        den = w1 + l * w2;
#pragma unroll
        for (int i = 0; i < DPL; ++i) o1[i] = act ? p.part_o[static_cast<size_t>(r) * p.d + col + i] : 0.f;
    }
    const float inv = den > 0.f ? 1.f / den : 0.f;
    if (act) {
#pragma unroll
        for (int i = 0; i < DPL; ++i)
            p.out[static_cast<size_t>(r) * p.d + col + i] = __float2bfloat16_rn((o1[i] * w1 + acc[i] * w2) * inv);
    }
}
}  // namespace

void decode_attention_local(Ctx* c, const DecodeAttnParams& p) {
    if (p.rows <= 0) return;
    const int hd = p.d / p.heads;
    const int warps = p.rows * p.heads;
    const dim3 grid((warps + SGC_DECODE_WPB - 1) / SGC_DECODE_WPB);
    Ctx::Timed timer(c, "attn_decode");
    switch (hd) {
        case 16: decode_local_kernel<16><<<grid, 32 * SGC_DECODE_WPB, 0, c->stream>>>(p); break;
        case 32: decode_local_kernel<32><<<grid, 32 * SGC_DECODE_WPB, 0, c->stream>>>(p); break;
        case 64: decode_local_kernel<64><<<grid, 32 * SGC_DECODE_WPB, 0, c->stream>>>(p); break;
        case 128: decode_local_kernel<128><<<grid, 32 * SGC_DECODE_WPB, 0, c->stream>>>(p); break;
        default: fail(SGC_DOMAIN, "decode attention: head_dim must be 16, 32, 64 or 128");
    }
    SGC_LAUNCH_CHECK(c);
}

}  // namespace sgc
