// attention_sm100.cu -- tcgen05/TMEM/TMA cascade attention for sm_100a (head_dim 64 / 128).
//
// Same semantics as attention.cu (lm_core.cpp:246-274: one softmax over the sealed prefix keys
// followed by the row's own causal suffix keys), laid out for the 5th-gen tensor cores in the
// FlashAttention-4 style: one work unit = two 128-row query tiles (A, B) of ONE cluster and one
// head, so every K/V block fetched serves 256 member rows, and the two tiles ping-pong on the
// tensor core while the other tile's softmax runs:
//
//   warp 0      TMEM allocator + TMA: Q tiles (once per unit), K blocks (128 keys, 3-stage ring
//               released once both tiles' S = Q K^T consumed a slot) and V blocks (2-stage
//               ring released after both O += P V)
//   warp 1      MMA issuer (one thread), per block j:
//                 O_A += P_A(j) V_j ; S_A(j+1) = Q_A K_{j+1} ; O_B += P_B(j) V_j ; S_B(j+1) = ...
//               S_X lives in TMEM; P_X (bf16) is written back over S_X's first 64 columns and
//               consumed straight from TMEM by the PV MMA (A operand in TMEM, V MN-major in smem).
//               tcgen05 ops of one thread execute in order, so S_X(j+1) never overwrites P_X(j)
//               before PV_X(j) read it, and s_full_X(j+1) also certifies PV_X(j) completed.
//   TMEM: 512 columns S_A | S_B | O_A | O_B
//   warps 2-5   softmax of tile A, warps 6-9 softmax of tile B: thread r owns query row r
//               (TMEM lane r) -- one streaming pass over its S row against the running max
//               (double-buffered 32-column TMEM loads, P packed in registers, then stored back
//               to TMEM); the max only moves when a block overshoots it by > 2^8 (block
//               recomputed, O rescaled in place in TMEM, O is stable whenever S is ready);
//               ~30% of the exponentials on the FMA pipe (MUFU offload); final O / l epilogue.
//
// Persistent: CTAs loop over (unit, head) items; units never straddle clusters (members) or
// sequences (representative prefill).
#include <atomic>

#include "attention.cuh"
#include "common.cuh"
#include "sched.cuh"
#include "sm100_ptx.cuh"
#include "tma.cuh"

namespace sgc {
namespace {

constexpr int BQ = 128;   // rows per query tile (two tiles per unit)
constexpr int BKV = 128;  // keys per block
// threads: loader warp, MMA warp, 2 tiles x SPLIT softmax warpgroups (SPLIT = 1: 320, 2: 576)
bool g_attn_split = false;  // two softmax warpgroups per query tile (sgc_set_option "attn_split"; measured no faster)
#ifndef SGC_ATTN_KSTAGES
#define SGC_ATTN_KSTAGES 3
#endif
constexpr int kKStages = SGC_ATTN_KSTAGES;
constexpr int kVStages = 5 - SGC_ATTN_KSTAGES;  // the K + V rings share 5 stages of shared memory
// (K 3 / V 2 and K 2 / V 3 measured equal on the final kernel: 105.3-105.9 vs 105.2-106.0 ms per C3 step)
// SGC_POLY_NUM / SGC_POLY_DEN of the exponential pairs run as a polynomial on the FMA pipe
// (MUFU.EX2 offload, FA4-style); the rest on MUFU
// the row's reference max only moves when a block max exceeds it by more than this (log2
// units): P <= 2^SGC_LAZY_MAX in bf16 (same relative precision at any scale), O rescales rare
#ifndef SGC_LAZY_MAX
#define SGC_LAZY_MAX 8.f
#endif
#ifndef SGC_S3_VFIRST
#define SGC_S3_VFIRST 0
#endif
#ifndef SGC_S3_TOKEN_LATE
#define SGC_S3_TOKEN_LATE 0
#endif
// softmax ping-pong between the two tiles (named barriers around the exponentials): it helped
// while the MMA thread was the slow resource; with the convergent-warp MMA issue it costs ~1.3%
// (same box, 3 alternating runs: 108.1-108.6 vs 109.7-110.0 ms per C3 step), so it is off
// SGC_ATTN_SPLIT_S=1: S(j+1) issued in two N = 64 halves around PV(j) (the lower half as soon as
// the softmax has loaded S(j), P written over S's upper half) to shorten the per-tile chain;
// measured slower at C3 (114.5 vs 107.7 ms per step, same box): N = 64 QK^T MMAs re-read Q
#ifndef SGC_ATTN_SPLIT_S
#define SGC_ATTN_SPLIT_S 0
#endif
constexpr uint32_t kPCol = SGC_ATTN_SPLIT_S ? 64 : 0;  // TMEM column of P within a tile's S
#ifndef SGC_ATTN_PINGPONG
#define SGC_ATTN_PINGPONG 0
#endif
// share of the exponentials on the FMA pipe (pairs j with j % DEN < NUM): measured at C3 with the
// final kernels (scripts/gpu_lib_ab.sh, attention ms/step): 0 121, 1/8 113, 1/6 113, 1/5 109,
// 1/4 105-107, 1/3 107-108, 2/5 110, 1/2 120
#ifndef SGC_POLY_NUM
#define SGC_POLY_NUM 1
#define SGC_POLY_DEN 4
#endif

template <int HD>
struct TcCfg {
    static constexpr int kSub = HD / 64;  // 64-element (128 B) swizzle sub-tiles
    static constexpr int kQBytes = BQ * HD * 2;
    static constexpr int kKBytes = BKV * HD * 2;
    static constexpr int kVBytes = BKV * HD * 2;
    // + barriers (256 B) + the split-softmax exchange slots [2][2][BQ] fp32
    // + barriers (256 B) + the split-softmax exchange slots [2][2][BQ] fp32 + the item ring
    static constexpr int kSmem = 2 * kQBytes + kKStages * kKBytes + kVStages * kVBytes + 256 + 2 * 2 * BQ * 4 + 128 + 256;
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kS = 0;    // S_X at column X * 128
    static constexpr uint32_t kO = 256;  // O_X at column 256 + X * 128
};

// Compile with -DSGC_ATTN_PROF to accumulate per-phase clock64() cycles into a global
// [148][16] counter array (debug builds only; see scripts/attn_prof.py).
#ifdef SGC_ATTN_PROF
__device__ unsigned long long g_attn_prof[148 * 32];
#endif

struct TcParams {
    const AttnWork* work;
    int n_work, heads;
    // partial mode (decode, prefix segment only): no local blocks; the epilogue writes the
    // normalized fp32 O and the row's log2-sum-exp (scaled-log2 units) instead of bf16 O
    float* part_o;    // [rows x d] or nullptr
    float* part_lse;  // [rows x heads]
    const int32_t* seg_lo;
    __nv_bfloat16* out;
    int d;
    float scale_log2;
    uint32_t* sched;  // dynamic item counter (sched.cuh)
    const int32_t* bt;  // block table (AttnParams::bt)
};
using ItemRing = UnitRing<4>;
// what the producer resolved for a claimed item (published with the ring slot, so the MMA and
// softmax warps start an item from shared memory instead of two dependent global loads)
struct ItemInfo {
    AttnWork w;
    int nA, nb0, nb1, nrows0, nrows1, loc_first;
};

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

// ---- packed fp32x2 helpers (FFMA2 / FADD2 / FMNMX3 on sm_100a): the softmax is issue-bound,
// so every per-element op that has a paired or 3-input form uses it
__device__ __forceinline__ uint64_t f2pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// two ex2_poly lanes with packed arithmetic: 10 issue slots for 2 exponentials
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
    const uint64_t magic = f2pack(12582912.0f, 12582912.0f), nmagic = f2pack(-12582912.0f, -12582912.0f);
    const uint64_t x = f2pack(fmaxf(x0, -125.0f), fmaxf(x1, -125.0f));
    const uint64_t t = fadd2(x, magic);                        // round(x) in the low mantissa bits
    const uint64_t u = fadd2(t, nmagic);                       // round(x) (exact)
    const uint64_t f = ffma2(u, f2pack(-1.0f, -1.0f), x);      // x - round(x), exact
    uint64_t p = ffma2(f2pack(0.05508868f, 0.05508868f), f, f2pack(0.24260405f, 0.24260405f));
    p = ffma2(p, f, f2pack(0.69327623f, 0.69327623f));
    p = ffma2(p, f, f2pack(0.99992895f, 0.99992895f));
    float t0, t1, p0, p1;
    f2unpack(t, t0, t1);
    f2unpack(p, p0, p1);
    // (bits(t) << 23) == round(x) << 23 (mod 2^32): the magic's high bits shift out
    y0 = __int_as_float((__float_as_int(t0) << 23) + __float_as_int(p0));
    y1 = __int_as_float((__float_as_int(t1) << 23) + __float_as_int(p1));
}

// blocks of one unit: prefix blocks nA (shared), total blocks per tile, first local key row
struct UnitPlan {
    int nA, nb[2], nrows[2], loc_first;
};
__device__ __forceinline__ UnitPlan plan_unit(const AttnWork& w, const int32_t* seg_lo, bool partial) {
    UnitPlan u;
    u.nA = (w.pfx_len + BKV - 1) / BKV;
    if (partial) {
        u.loc_first = 0;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            u.nrows[x] = min(BQ, max(0, w.nrows - x * BQ));
            u.nb[x] = u.nrows[x] > 0 ? u.nA : 0;
        }
        return u;
    }
    u.loc_first = seg_lo[w.row0];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
        u.nrows[x] = min(BQ, max(0, w.nrows - x * BQ));
        const int last = w.row0 + x * BQ + u.nrows[x] - 1;
        u.nb[x] = u.nrows[x] > 0 ? u.nA + (last - u.loc_first + BKV) / BKV : 0;
    }
    return u;
}

template <int HD, int SPLIT>
__global__ void __launch_bounds__(64 + 256 * SPLIT, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKp,
                   const __grid_constant__ CUtensorMap tmVp, const __grid_constant__ CUtensorMap tmKl,
                   const __grid_constant__ CUtensorMap tmVl, TcParams p) {
    using C = TcCfg<HD>;
    static_assert(sizeof(ItemRing) <= 128 && 4 * sizeof(ItemInfo) <= 256, "item ring");
    // all shared memory is dynamic (no static arrays), so the base is 1024-byte aligned
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem;                                  // [2][BQ x HD]
    uint8_t* sK = sQ + 2 * C::kQBytes;                   // [kKStages][BKV x HD]
    uint8_t* sV = sK + kKStages * C::kKBytes;            // [kVStages][BKV x HD]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVStages * C::kVBytes);
    uint64_t* q_full = bars + 0;    // [2]
    uint64_t* q_empty = bars + 2;   // [2]
    uint64_t* k_full = bars + 4;                // [kKStages]
    uint64_t* k_empty = k_full + kKStages;      // [kKStages]
    uint64_t* v_full = k_empty + kKStages;      // [kVStages]
    uint64_t* v_empty = v_full + kVStages;      // [kVStages] (ends at bars + 14)
    uint64_t* s_full = bars + 14;   // [2] per tile
    uint64_t* p_full = bars + 16;   // [2] per tile
    uint64_t* o_full = bars + 18;   // [2] per tile
    uint64_t* s_read = bars + 20;   // [2] per tile: the softmax loaded S (its lower half may be reused)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);
    float* xm = reinterpret_cast<float*>(bars + 32);  // [2 tiles][SPLIT][BQ] row max / sum exchange
    // items (unit x head) claimed by the producer and handed to the MMA and softmax warps
    ItemRing* ring = reinterpret_cast<ItemRing*>(xm + 2 * 2 * BQ);
    ItemInfo* info = reinterpret_cast<ItemInfo*>(reinterpret_cast<uint8_t*>(ring) + 128);  // [4] per slot

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_items = p.n_work * p.heads;
    // consumer side: item k's slot -> (item, work, plan) in registers, then release the slot
    auto take_item = [&](uint32_t k, AttnWork& w, UnitPlan& u) -> uint32_t {
        const uint32_t iu = sched::wait(ring, k);
        if (iu < static_cast<uint32_t>(n_items)) {
            const ItemInfo& f = info[k % 4];
            w = f.w;
            u.nA = f.nA;
            u.nb[0] = f.nb0;
            u.nb[1] = f.nb1;
            u.nrows[0] = f.nrows0;
            u.nrows[1] = f.nrows1;
            u.loc_first = f.loc_first;
        }
        return iu;
    };

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmKp);
        ptx::tma_prefetch_desc(&tmVp);
        ptx::tma_prefetch_desc(&tmKl);
        ptx::tma_prefetch_desc(&tmVl);
        for (int i = 0; i < kKStages; ++i) {
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
        }
        for (int i = 0; i < kVStages; ++i) {
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&q_full[i], 1);
            ptx::mbar_init(&q_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&p_full[i], 128 * SPLIT);
            ptx::mbar_init(&o_full[i], 1);
            ptx::mbar_init(&s_read[i], 128 * SPLIT);
        }
        sched::init(ring, 1 + 8 * SPLIT);  // the MMA thread + every softmax warp
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // TMA loader: Q tiles once per unit, then K_b and V_b per block
        if (lane == 0) {
            uint32_t g = 0, qit[2] = {0, 0};
            for (uint32_t k = 0;; ++k) {
                // claim (when the slot frees: items are long, claiming ahead would only skew the
                // tail), resolve the item's plan, publish it with the slot
                const int sl = k % 4;
                ptx::mbar_wait(&ring->empty[sl], ((k / 4) & 1) ^ 1);
                const uint32_t iu = sched::claim(p.sched, n_items, gridDim.x, k);
                ring->unit[sl] = iu;
                AttnWork w{};
                UnitPlan u{};
                if (iu < static_cast<uint32_t>(n_items)) {
                    w = p.work[iu % p.n_work];
                    u = plan_unit(w, p.seg_lo, p.part_o != nullptr);
                    info[sl] = ItemInfo{w, u.nA, u.nb[0], u.nb[1], u.nrows[0], u.nrows[1], u.loc_first};
                }
                ptx::mbar_arrive(&ring->full[sl]);
                if (iu >= static_cast<uint32_t>(n_items)) break;
                const int h = static_cast<int>(iu) / p.n_work;
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    if (!u.nb[x]) continue;
                    ptx::mbar_wait(&q_empty[x], (qit[x] & 1) ^ 1);
                    ptx::mbar_expect_tx(&q_full[x], C::kQBytes);
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s)
                        ptx::tma_load_2d(sQ + x * C::kQBytes + s * (BQ * 128), &tmQ, &q_full[x],
                                         h * HD + s * 64, w.row0 + x * BQ);
                    ++qit[x];
                }
                const int nbu = max(u.nb[0], u.nb[1]);
                for (int b = 0; b < nbu; ++b, ++g) {
                    const bool pfx = b < u.nA;
                    // 128-key block == one page: prefix pages / the sequence's own pages
                    // (paged prefill) through the block table, or contiguous scratch rows
                    const int row = pfx ? kv_row_of(p.bt, w.pfx_off, b * BKV)
                                        : (w.loc_bt >= 0 ? kv_row_of(p.bt, w.loc_bt, (b - u.nA) * BKV)
                                                         : u.loc_first + (b - u.nA) * BKV);
                    const int ks = g % kKStages;
                    ptx::mbar_wait(&k_empty[ks], ((g / kKStages) & 1) ^ 1);
                    ptx::mbar_expect_tx(&k_full[ks], C::kKBytes);
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s)
                        ptx::tma_load_2d(sK + ks * C::kKBytes + s * (BKV * 128), pfx ? &tmKp : &tmKl,
                                         &k_full[ks], h * HD + s * 64, row);
                    const int vs = g % kVStages;
                    ptx::mbar_wait(&v_empty[vs], ((g / kVStages) & 1) ^ 1);
                    ptx::mbar_expect_tx(&v_full[vs], C::kVBytes);
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s)
                        ptx::tma_load_2d(sV + vs * C::kVBytes + s * (BKV * 128), pfx ? &tmVp : &tmVl,
                                         &v_full[vs], h * HD + s * 64, row);
                }
            }
        }
    } else if (warp == 1) {
        // the whole warp runs the issue loop (warp-uniform operands -> uniform datapath); one
        // elected lane issues each tcgen05.mma / commit
        {
#ifdef SGC_ATTN_PROF
            // MMA thread: cycles in each wait (slots 16..19) and in total (slot 22)
            const long long t_mma0 = clock64();
            auto mwait = [&](uint64_t* bar, uint32_t par, int slot) {
                const long long t0 = clock64();
                ptx::mbar_wait(bar, par);
                if (lane == 0) atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 32 + slot], (unsigned long long)(clock64() - t0));
            };
#else
            auto mwait = [&](uint64_t* bar, uint32_t par, int) { ptx::mbar_wait(bar, par); };
#endif
            constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
            constexpr uint32_t idO = ptx::idesc_bf16_f32_bmn(BQ, HD);
            uint32_t g = 0, gx[2] = {0, 0}, qit[2] = {0, 0};
            // descriptors built once per operand tile, then advanced by constants (the start
            // address field is bytes >> 4): fewer dependent instructions per tcgen05.mma for the
            // single issuing thread, which was busy ~70% of the kernel (scripts/attn_prof.py)
            auto issue_s = [&](int x, uint32_t kg) {  // S_X = Q_X K^T
                const uint64_t qd = ptx::umma_desc_sw128(ptx::smem_u32(sQ + x * C::kQBytes));
                const uint64_t kd = ptx::umma_desc_sw128(ptx::smem_u32(sK + (kg % kKStages) * C::kKBytes));
                const uint32_t dS = tmem_base + C::kS + x * BQ;
#pragma unroll
                for (int kc = 0; kc < HD / 16; ++kc) {
                    const uint64_t ad = qd + (((kc / 4) * (BQ * 128) + (kc % 4) * 32) >> 4);
                    const uint64_t bd = kd + (((kc / 4) * (BKV * 128) + (kc % 4) * 32) >> 4);
                    ptx::mma_bf16_elect(dS, ad, bd, idS, kc > 0 ? 1u : 0u);
                }
                ptx::mma_commit_elect(&s_full[x]);
            };
#if SGC_ATTN_SPLIT_S
            // S(j+1) in two N = 64 halves: the lower half (columns 0-63) as soon as the softmax has
            // loaded S(j) -- P(j) lives in columns 64-127 -- and the upper half after PV(j) read P(j)
            constexpr uint32_t idS64 = ptx::idesc_bf16_f32(BQ, 64);
            uint32_t sr[2] = {0, 0};
            auto issue_s_half = [&](int x, uint32_t kg, int half) {
                const uint64_t qd = ptx::umma_desc_sw128(ptx::smem_u32(sQ + x * C::kQBytes));
                const uint64_t kd = ptx::umma_desc_sw128(ptx::smem_u32(sK + (kg % kKStages) * C::kKBytes));
                const uint32_t dS = tmem_base + C::kS + x * BQ + half * 64;
#pragma unroll
                for (int kc = 0; kc < HD / 16; ++kc) {
                    const uint64_t ad = qd + (((kc / 4) * (BQ * 128) + (kc % 4) * 32) >> 4);
                    const uint64_t bd = kd + (((kc / 4) * (BKV * 128) + (kc % 4) * 32 + half * 64 * 128) >> 4);
                    ptx::mma_bf16_elect(dS, ad, bd, idS64, kc > 0 ? 1u : 0u);
                }
            };
#endif
            auto issue_pv = [&](int x, uint32_t kg, bool first) {  // O_X += P_X V
                mwait(&p_full[x], gx[x] & 1, 18);
                ptx::tc_fence_after();
                const uint64_t vd = ptx::umma_desc_sw128_lbo(ptx::smem_u32(sV + (kg % kVStages) * C::kVBytes), BKV * 128, 1024);
                const uint32_t dO = tmem_base + C::kO + x * 128, aP = tmem_base + C::kS + x * BQ + kPCol;
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk)
                    ptx::mma_bf16_ts_elect(dO, aP + kk * 8, vd + ((kk * 16 * 128) >> 4), idO, (!first || kk > 0) ? 1u : 0u);
                ++gx[x];
            };
            for (uint32_t k = 0;; ++k) {
                AttnWork w;
                UnitPlan u;
                const uint32_t iu = take_item(k, w, u);
                __syncwarp();
                if (lane == 0) sched::release(ring, k);
                if (iu >= static_cast<uint32_t>(n_items)) break;
                const int nbu = max(u.nb[0], u.nb[1]);
                for (int x = 0; x < 2; ++x)
                    if (u.nb[x]) mwait(&q_full[x], qit[x] & 1, 19);
                // prologue: S(0) of both tiles
                mwait(&k_full[g % kKStages], (g / kKStages) & 1, 16);
                ptx::tc_fence_after();
                for (int x = 0; x < 2; ++x)
                    if (u.nb[x]) issue_s(x, g);
                ptx::mma_commit_elect(&k_empty[g % kKStages]);
                for (int j = 0; j < nbu; ++j) {
                    const uint32_t kg = g + j;
                    mwait(&v_full[kg % kVStages], (kg / kVStages) & 1, 17);
                    bool waited_next_k = false;
#if SGC_ATTN_SPLIT_S
                    for (int x = 0; x < 2; ++x) {
                        if (j + 1 >= u.nb[x]) continue;
                        if (!waited_next_k) {
                            mwait(&k_full[(kg + 1) % kKStages], ((kg + 1) / kKStages) & 1, 16);
                            waited_next_k = true;
                        }
                        mwait(&s_read[x], sr[x] & 1, 16);
                        ++sr[x];
                        ptx::tc_fence_after();
                        issue_s_half(x, kg + 1, 0);
                    }
#endif
                    for (int x = 0; x < 2; ++x) {
                        if (j >= u.nb[x]) continue;
                        issue_pv(x, kg, j == 0);
                        if (j + 1 < u.nb[x]) {
                            if (!waited_next_k) {
                                mwait(&k_full[(kg + 1) % kKStages], ((kg + 1) / kKStages) & 1, 16);
                                ptx::tc_fence_after();
                                waited_next_k = true;
                            }
#if SGC_ATTN_SPLIT_S
                            issue_s_half(x, kg + 1, 1);
                            ptx::mma_commit_elect(&s_full[x]);
#else
                            issue_s(x, kg + 1);
#endif
                        } else {
                            ptx::mma_commit_elect(&o_full[x]);
                            ptx::mma_commit_elect(&q_empty[x]);
                        }
                    }
                    ptx::mma_commit_elect(&v_empty[kg % kVStages]);
                    if (j + 1 < nbu) ptx::mma_commit_elect(&k_empty[(kg + 1) % kKStages]);
                }
                g += nbu;
                for (int x = 0; x < 2; ++x)
                    if (u.nb[x]) ++qit[x];
            }
#ifdef SGC_ATTN_PROF
            if (lane == 0) atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 32 + 22], (unsigned long long)(clock64() - t_mma0));
#endif
        }
    } else {
        // softmax warps: tile x = 0 (A) / 1 (B); with SPLIT = 2 each tile has two warpgroups,
        // half 0 owning S columns 0-63 and half 1 columns 64-127 of every row (the row max is
        // exchanged through shared memory once per block). A warp may only touch TMEM lanes
        // 32 * (warp % 4) .. +31, so row = 32 * (warp % 4) + lane.
        constexpr int COLS = BKV / SPLIT;          // S columns per thread
        constexpr int OCOLS = HD / SPLIT;          // O columns per thread (rescale, epilogue)
        const int sw = warp - 2;
        const int x = sw / (4 * SPLIT);            // query tile handled by this warpgroup
        const int half = (sw / 4) % SPLIT;
        const int c0 = half * COLS;                // first S column (key) of this thread
        const int r = (warp & 3) * 32 + lane;      // row within the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tS = tmem_base + lane_base + C::kS + x * BQ;
        const uint32_t tO = tmem_base + lane_base + C::kO + x * 128;
        float* xch = xm + (x * SPLIT) * BQ;        // [SPLIT][BQ] exchange slots of this tile
        auto tile_sync = [&]() {
            if constexpr (SPLIT > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + x), "r"(128 * SPLIT) : "memory");
        };
        // Softmax ping-pong (FA3/FA4-style): while both tiles have block b, the two warpgroups
        // take turns on the exponentials (A(b), B(b), A(b+1), ...) through named barriers 3/4,
        // so each runs at the SM's full MUFU/FMA rate while the tensor pipe works on the other
        // tile's PV + next S, instead of both crawling side by side and stretching the chain
        // S(b) -> softmax(b) -> PV(b) -> S(b+1) of each tile.
        constexpr bool kPing = SPLIT == 1 && SGC_ATTN_PINGPONG;
        auto ping_wait = [&]() {
            if constexpr (kPing) asm volatile("bar.sync %0, 256;" ::"r"(3 + x) : "memory");
        };
        auto ping_pass = [&]() {
            if constexpr (kPing) asm volatile("bar.arrive %0, 256;" ::"r"(4 - x) : "memory");
        };
        uint32_t gs = 0, uit = 0;
#ifdef SGC_ATTN_PROF
        const bool prof_thr = threadIdx.x == 64;
        long long _pt = clock64();
#define SPROF(slot)                                                                            \
    if (prof_thr) {                                                                            \
        long long _n = clock64();                                                              \
        atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 32 + (slot)], (unsigned long long)(_n - _pt)); \
        _pt = _n;                                                                              \
    }
#else
#define SPROF(slot)
#endif
        for (uint32_t k = 0;; ++k) {
            AttnWork w;
            UnitPlan u;
            const uint32_t iu = take_item(k, w, u);
            __syncwarp();
            if (lane == 0) sched::release(ring, k);
            if (iu >= static_cast<uint32_t>(n_items)) break;
            const int item = static_cast<int>(iu);
            const int h = item / p.n_work;
            const int nb = u.nb[x];
            if (!nb) continue;
            const bool valid = r < u.nrows[x];
            const int row = w.row0 + x * BQ + r;
            const int seg = valid && !p.part_o ? p.seg_lo[row] : 0x7fffffff;
            // blocks both tiles have take turns; tile B hands tile A the first turn
            const int n_ping = min(u.nb[0], u.nb[1]);
            if (x == 1 && n_ping > 0) ping_pass();
            float m = -INFINITY, l = 0.f;
            for (int b = 0; b < nb; ++b, ++gs) {
                SPROF(0);
                ptx::mbar_wait(&s_full[x], gs & 1);
                ptx::tc_fence_after();
                SPROF(1);
                int k0, klo, khi;  // visible key window [klo, khi] in block-local index
                if (b < u.nA) {
                    k0 = b * BKV;
                    klo = 0;
                    khi = valid ? min(BKV, w.pfx_len - k0) - 1 : -1;
                } else {
                    k0 = u.loc_first + (b - u.nA) * BKV;
                    klo = max(0, seg - k0);
                    khi = valid ? min(BKV - 1, row - k0) : -1;
                }
                // warp-uniform: the tcgen05.ld/st below are .sync.aligned (whole warp, same path)
                const bool full = __all_sync(0xffffffffu, klo <= c0 && khi >= c0 + COLS - 1);
                // This thread's part of the S row (COLS fp32) is loaded into registers with
                // back-to-back tcgen05.ld (one wait), reduced to its max (with SPLIT = 2 combined
                // with the other half's through shared memory), exponentiated in place (P packed
                // as bf16 pairs) and stored over S's first 64 columns. The row's reference max m
                // is lazy: it only moves when the block max exceeds it by more than 2^8 (then O
                // is rescaled in place; P <= 2^8 otherwise), so the common case has no O traffic.
                const float sc = p.scale_log2;
                uint32_t sv[COLS];
#pragma unroll
                for (int c = 0; c < COLS / 32; ++c)
                    ptx::tmem_ld32(tS + c0 + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
                ptx::tmem_ld_wait();
#if SGC_ATTN_SPLIT_S
                if (b + 1 < nb) {  // S(b) is in registers: the MMA may compute S(b+1)'s lower half
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(&s_read[x]);
                }
#endif
                SPROF(7);
                // visibility bitmap of this thread's keys [klo, khi] (COLS / 32 words)
                uint32_t vw[COLS / 32];
#pragma unroll
                for (int wd = 0; wd < COLS / 32; ++wd) {
                    const int lo = klo - c0 - 32 * wd, hi = khi - c0 - 32 * wd;
                    const uint32_t mlo = lo <= 0 ? ~0u : (lo >= 32 ? 0u : ~0u << lo);
                    const uint32_t mhi = hi >= 31 ? ~0u : (hi < 0 ? 0u : ~0u >> (31 - hi));
                    vw[wd] = mlo & mhi;
                }
                if (!full) {
#pragma unroll
                    for (int j = 0; j < COLS; ++j)
                        if (!(vw[j / 32] & (1u << (j % 32)))) sv[j] = __float_as_uint(-INFINITY);
                }
                float bmax;
                {
                    // max over RAW scores (scale > 0): 3-input max, four independent chains
                    float q0 = -INFINITY, q1 = -INFINITY, q2 = -INFINITY, q3 = -INFINITY;
#pragma unroll
                    for (int j = 0; j < COLS; j += 8) {
                        q0 = fmax3(q0, __uint_as_float(sv[j]), __uint_as_float(sv[j + 1]));
                        q1 = fmax3(q1, __uint_as_float(sv[j + 2]), __uint_as_float(sv[j + 3]));
                        q2 = fmax3(q2, __uint_as_float(sv[j + 4]), __uint_as_float(sv[j + 5]));
                        q3 = fmax3(q3, __uint_as_float(sv[j + 6]), __uint_as_float(sv[j + 7]));
                    }
                    bmax = fmaxf(fmaxf(q0, q1), fmaxf(q2, q3));
                    if constexpr (SPLIT > 1) {
                        // every S load of the tile is complete once all its threads pass here,
                        // so P may overwrite S columns owned by the other half afterwards
                        xch[half * BQ + r] = bmax;
                        tile_sync();
                        bmax = fmaxf(bmax, xch[(1 - half) * BQ + r]);
                    }
                    bmax *= sc;  // scaled-log2 units
                }
                SPROF(8);
                // the turn covers the MUFU-heavy exponentials only: the S load and the max of one
                // tile overlap the other tile's exponentials
                if (b < n_ping) ping_wait();
                const float mnew = (m == -INFINITY || bmax > m + SGC_LAZY_MAX) ? bmax : m;
                const float nm = mnew == -INFINITY ? 0.f : -mnew;
                float rs;
                {
                    const uint64_t sc2 = f2pack(sc, sc), nm2 = f2pack(nm, nm);
                    uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;  // packed partial row sums
#pragma unroll
                    for (int j = 0; j < COLS / 2; ++j) {
                        float xa, xc;  // x = raw * scale_log2 - m: one FFMA2 per pair
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[2 * j]), __uint_as_float(sv[2 * j + 1])), sc2, nm2),
                                 xa, xc);
                        float a, cc;
                        if ((j % SGC_POLY_DEN) < SGC_POLY_NUM) {  // share of exponentials on the FMA pipe
                            // a masked key (-inf) comes out as 2^-125 instead of 0: < 1e-37 of the
                            // row sum (>= 1), below every fp32 ulp of l and O -- not worth the
                            // predicated selects in the hot loop
                            ex2_poly2(xa, xc, a, cc);
                        } else {
                            a = ex2_approx(xa);
                            cc = ex2_approx(xc);
                        }
                        const uint64_t pr = f2pack(a, cc);
                        if ((j & 3) == 0) r0 = fadd2(r0, pr);
                        else if ((j & 3) == 1) r1 = fadd2(r1, pr);
                        else if ((j & 3) == 2) r2 = fadd2(r2, pr);
                        else r3 = fadd2(r3, pr);
                        __nv_bfloat162 bv = __floats2bfloat162_rn(a, cc);
                        sv[j] = *reinterpret_cast<uint32_t*>(&bv);  // P pair j (j <= 2j: in place)
                    }
                    float x0, x1;
                    f2unpack(fadd2(fadd2(r0, r1), fadd2(r2, r3)), x0, x1);
                    rs = x0 + x1;
                }
                // A always passes the turn on; B only while A has another shared block
                if (b < n_ping && (x == 0 || b + 1 < n_ping)) ping_pass();
                SPROF(2);
                float alpha = 1.f;
                // the rescale is a per-row decision, but tcgen05.ld/st are .sync.aligned: the
                // whole warp enters when any lane needs it (the others scale by exactly 1)
                const bool resc = m != -INFINITY && mnew > m;
                if (__any_sync(0xffffffffu, resc)) {
                    // O is stable here: s_full certified the previous PV of this tile completed
                    alpha = resc ? ex2_approx(m - mnew) : 1.f;
#pragma unroll 1
                    for (int c = 0; c < OCOLS / 32; ++c) {
                        uint32_t o[32];
                        ptx::tmem_ld32(tO + half * OCOLS + c * 32, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                        ptx::tmem_st32(tO + half * OCOLS + c * 32, o);
                    }
                }
                m = mnew;
                SPROF(3);
                // P -> TMEM over S's first 64 columns (this thread's keys: columns c0/2 ..)
#pragma unroll
                for (int c = 0; c < COLS / 32; ++c)
                    ptx::tmem_st16(tS + kPCol + c0 / 2 + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
                l = l * alpha + rs;
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&p_full[x]);
                SPROF(4);
            }
            // epilogue: O / l -> bf16
            ptx::mbar_wait(&o_full[x], uit & 1);
            ptx::tc_fence_after();
            SPROF(5);
            if constexpr (SPLIT > 1) {
                // every thread of the tile read the last block's max before its p_full arrive,
                // and o_full follows all of them: the exchange slots are free for the row sums
                xch[half * BQ + r] = l;
                tile_sync();
                l += xch[(1 - half) * BQ + r];
                tile_sync();  // slots reused by the next item's first block
            }
            const float il = l > 0.f ? 1.f / l : 0.f;
            uint32_t o[OCOLS];
#pragma unroll
            for (int c = 0; c < OCOLS / 32; ++c)
                ptx::tmem_ld32(tO + half * OCOLS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
            ptx::tmem_ld_wait();
            if (valid && p.part_o) {
                float* dst = p.part_o + static_cast<size_t>(row) * p.d + h * HD + half * OCOLS;
#pragma unroll
                for (int q = 0; q < OCOLS / 8; ++q) {  // 32 B per store (STG.256)
                    uint32_t wv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) wv[e] = __float_as_uint(__uint_as_float(o[8 * q + e]) * il);
                    ptx::st_global_v8(dst + 8 * q, wv);
                }
                if (half == 0) p.part_lse[static_cast<size_t>(row) * p.heads + h] = l > 0.f ? m + __log2f(l) : -INFINITY;
            } else if (valid) {
                __nv_bfloat16* dst = p.out + static_cast<size_t>(row) * p.d + h * HD + half * OCOLS;
#pragma unroll
                for (int q = 0; q < OCOLS / 16; ++q) {  // 32 B per store (STG.256)
                    uint32_t wv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        __nv_bfloat162 bv = __floats2bfloat162_rn(__uint_as_float(o[16 * q + 2 * e]) * il,
                                                                  __uint_as_float(o[16 * q + 2 * e + 1]) * il);
                        wv[e] = *reinterpret_cast<uint32_t*>(&bv);
                    }
                    ptx::st_global_v8(dst + 16 * q, wv);
                }
            }
            ptx::tc_fence_before();
            ++uit;
            SPROF(6);
        }
#undef SPROF
    }
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// =============================================================================================
// attn_s3_kernel -- one 128-row query tile per item; S triple-buffered in TMEM; two softmax
// warpgroups taking alternate key blocks of the same rows.
//
// The two-tile kernel above runs two dependency chains S(b) -> softmax(b) -> PV(b) -> S(b+1) per
// CTA (P lives in S's columns, so S(b+1) of a tile waits for PV(b) of that tile) and shares the
// SM sub-partitions between the two tiles' softmaxes: the chain per block is softmax + S + PV +
// latencies (~3.7k cycles against 2 x 1024 of tensor work; 54% tensor-active, the softmax
// waiting a third of its time for its next S, scripts/attn_prof.py). Here:
//   * the MMA warp runs three blocks ahead: S(g+3) goes into buffer g % 3 as soon as PV(g) is
//     issued, so a block's S is ready long before its softmax starts;
//   * softmax warpgroup w takes the blocks g with g % 2 == w, so two blocks' softmaxes overlap
//     (one's exponentials on MUFU while the other loads S from TMEM / reduces its max) and each
//     warpgroup has two block periods per block;
//   * the rows' running max is shared (smem, lazy: it only moves when a block overshoots it by
//     more than 2^8): block g+1 reads the max block g decided (named-barrier token passed
//     between the warpgroups, after both computed their block max) before its exponentials;
//     each warpgroup keeps its own row sum relative to the max it last saw; the rare O rescale
//     waits for the previous PV; the epilogue combines the two row sums.
//
//   warp 0      TMEM allocator + TMA producer: claims tiles (skipping empty ones), Q per tile,
//               K blocks two ahead of V blocks in the global block stream
//   warp 10     S issuer: S(g) into buffer g % 3 once PV(g-3) read that buffer's P
//   warp 1      PV issuer: O += P(g) V(g) (one thread issuing both ran ~1.4k cycles per block
//               of 1024 tensor cycles: ~17 instructions per tcgen05.mma)
//   warps 2-5   softmax warpgroup 0 (even blocks), warps 6-9 warpgroup 1 (odd blocks)
//   TMEM: S_0 | S_1 | S_2 | O   (columns 0, 128, 256, 384)
// =============================================================================================
template <int HD>
struct S3Cfg {
    static constexpr int kSub = HD / 64;
    static constexpr int kQBytes = BQ * HD * 2;
    static constexpr int kKBytes = BKV * HD * 2;
    static constexpr int kVBytes = BKV * HD * 2;
    static constexpr int kQStages = 2, kKStages = 2, kVStages = 3;
    static constexpr int kTiles = kQStages * kQBytes + kKStages * kKBytes + kVStages * kVBytes;
    // + barriers (256 B) + shared row max and row-sum hand-over [2 tile parities][BQ] + item ring
    static constexpr int kSmem = kTiles + 256 + 2 * BQ * 4 + 2 * BQ * 4 + 160 + 8 * 44;
    static constexpr uint32_t kTmemCols = 512;
    static constexpr uint32_t kS = 0;    // S buffer s at column s * 128
    static constexpr uint32_t kO = 384;  // O (HD columns)
};

// a claimed 128-row tile, resolved by the producer and published with its ring slot
struct TileInfo {
    AttnWork w;
    int h, x, nA, nb, nrows, loc_first;
};
// eight slots: the MMA warp holds the tiles from its PV cursor to its S cursor (up to four
// one-block tiles) while the producer claims ahead
constexpr int kTileRing = 8;
using TileRing = UnitRing<kTileRing>;

__device__ __forceinline__ TileInfo plan_tile(const AttnWork& w, int h, int x, const int32_t* seg_lo, bool partial) {
    TileInfo t;
    t.w = w;
    t.h = h;
    t.x = x;
    t.nA = (w.pfx_len + BKV - 1) / BKV;
    t.nrows = min(BQ, max(0, w.nrows - x * BQ));
    if (partial) {
        t.loc_first = 0;
        t.nb = t.nrows > 0 ? t.nA : 0;
        return t;
    }
    // own keys: contiguous batch rows start at the tile's first member (keys before it are
    // never visible to the tile); paged sequences are read page by page from their start
    t.loc_first = t.nrows > 0 ? seg_lo[w.loc_bt >= 0 ? w.row0 : w.row0 + x * BQ] : 0;
    const int last = w.row0 + x * BQ + t.nrows - 1;
    t.nb = t.nrows > 0 ? t.nA + (last - t.loc_first + BKV) / BKV : 0;
    return t;
}

template <int HD>
__global__ void __launch_bounds__(352, 1)
    attn_s3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKp,
                   const __grid_constant__ CUtensorMap tmVp, const __grid_constant__ CUtensorMap tmKl,
                   const __grid_constant__ CUtensorMap tmVl, TcParams p) {
    using C = S3Cfg<HD>;
    static_assert(sizeof(TileRing) <= 160 && sizeof(TileInfo) <= 44, "tile ring");
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sQ = smem;                                  // [2][BQ x HD]
    uint8_t* sK = sQ + C::kQStages * C::kQBytes;         // [2][BKV x HD]
    uint8_t* sV = sK + C::kKStages * C::kKBytes;         // [3][BKV x HD]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + C::kVStages * C::kVBytes);
    uint64_t* q_full = bars + 0;    // [2]
    uint64_t* q_empty = bars + 2;   // [2]
    uint64_t* k_full = bars + 4;    // [2]
    uint64_t* k_empty = bars + 6;   // [2]
    uint64_t* v_full = bars + 8;    // [3]
    uint64_t* v_empty = bars + 11;  // [3]
    uint64_t* s_full = bars + 14;   // [3] per S buffer
    uint64_t* p_full = bars + 17;   // [3] per S buffer (P is written over S)
    uint64_t* o_full = bars + 20;   // the tile's last PV completed
    uint64_t* o_free = bars + 21;   // the tile's epilogue read O (the next tile's first PV may run)
    uint64_t* s_free = bars + 24;   // [3] PV(g) completed: S(g+3) may overwrite the buffer's P
                                    // (also what the rare O rescale of block g+1 waits for)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
    float* m_sh = reinterpret_cast<float*>(bars + 32);  // [2 tile parities][BQ] the rows' running max
    float* lx = m_sh + 2 * BQ;                          // [2 tile parities][BQ] row-sum hand-over
    TileRing* ring = reinterpret_cast<TileRing*>(lx + 2 * BQ);
    TileInfo* info = reinterpret_cast<TileInfo*>(reinterpret_cast<uint8_t*>(ring) + 160);  // [kTileRing]

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_items = 2 * p.n_work * p.heads;  // (head, unit, tile) with the tile fastest
    const bool partial = p.part_o != nullptr;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmQ);
        ptx::tma_prefetch_desc(&tmKp);
        ptx::tma_prefetch_desc(&tmVp);
        ptx::tma_prefetch_desc(&tmKl);
        ptx::tma_prefetch_desc(&tmVl);
        for (int i = 0; i < 3; ++i) {
            ptx::mbar_init(&v_full[i], 1);
            ptx::mbar_init(&v_empty[i], 1);
            ptx::mbar_init(&s_full[i], 1);
            ptx::mbar_init(&p_full[i], 128);
            ptx::mbar_init(&s_free[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&q_full[i], 1);
            ptx::mbar_init(&q_empty[i], 1);
            ptx::mbar_init(&k_full[i], 1);
            ptx::mbar_init(&k_empty[i], 1);
        }
        ptx::mbar_init(o_full, 1);
        ptx::mbar_init(o_free, 128);
        sched::init(ring, 2 + 8);  // the two MMA threads + every softmax warp
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

#ifdef SGC_ATTN_PROF
    // cycles the producer / MMA threads spend in each wait (slots 16..)
    auto pwait = [&](uint64_t* bar, uint32_t par, int slot) {
        const long long t0 = clock64();
        ptx::mbar_wait_park(bar, par);
        if ((threadIdx.x & 31) == 0)
            atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 32 + slot], (unsigned long long)(clock64() - t0));
    };
#else
    auto pwait = [&](uint64_t* bar, uint32_t par, int) { ptx::mbar_wait_park(bar, par); };
#endif
    // key row of block b of tile t: prefix pages, the sequence's own pages (paged prefill) or
    // contiguous scratch rows
    auto block_row = [&](const TileInfo& t, int b) -> int {
        if (b < t.nA) return kv_row_of(p.bt, t.w.pfx_off, b * BKV);
        return t.w.loc_bt >= 0 ? kv_row_of(p.bt, t.w.loc_bt, (b - t.nA) * BKV) : t.loc_first + (b - t.nA) * BKV;
    };

    if (warp == 0) {
        if (lane == 0) {
            // two cursors over the global block stream: K runs two blocks ahead of V
            uint32_t gk = 0, gv = 0;
            int ki = -1, kb = 0, knb = 0, vi = 0, vb = 0;
            bool kend = false;
            auto next_k = [&]() -> bool {
                if (kend) return false;
                while (kb >= knb) {
                    ++ki;
                    const int sl = ki % kTileRing;
                    pwait(&ring->empty[sl], ((ki / kTileRing) & 1) ^ 1, 27);
                    uint32_t iu;
                    TileInfo t{};
                    for (;;) {  // claim the next non-empty tile (one claim past the end per CTA)
                        iu = sched::claim(p.sched, n_items, gridDim.x, ki);
                        if (iu >= static_cast<uint32_t>(n_items)) break;
                        const int per_head = 2 * p.n_work;
                        const int h = static_cast<int>(iu) / per_head, rem = static_cast<int>(iu) % per_head;
                        t = plan_tile(p.work[rem >> 1], h, rem & 1, p.seg_lo, partial);
                        if (t.nb > 0) break;
                    }
                    ring->unit[sl] = iu;
                    if (iu < static_cast<uint32_t>(n_items)) info[sl] = t;
                    ptx::mbar_arrive(&ring->full[sl]);
                    if (iu >= static_cast<uint32_t>(n_items)) {
                        kend = true;
                        return false;
                    }
                    knb = t.nb;
                    kb = 0;
                    const int qs = ki & 1;
                    pwait(&q_empty[qs], ((ki >> 1) & 1) ^ 1, 26);
                    ptx::mbar_expect_tx(&q_full[qs], C::kQBytes);
#pragma unroll
                    for (int s = 0; s < C::kSub; ++s)
                        ptx::tma_load_2d(sQ + qs * C::kQBytes + s * (BQ * 128), &tmQ, &q_full[qs], t.h * HD + s * 64,
                                         t.w.row0 + t.x * BQ);
                }
                const TileInfo& t = info[ki % kTileRing];
                const bool pfx = kb < t.nA;
                const int row = block_row(t, kb);
                const int ks = gk % C::kKStages;
                pwait(&k_empty[ks], ((gk / C::kKStages) & 1) ^ 1, 24);
                ptx::mbar_expect_tx(&k_full[ks], C::kKBytes);
#pragma unroll
                for (int s = 0; s < C::kSub; ++s)
                    ptx::tma_load_2d(sK + ks * C::kKBytes + s * (BKV * 128), pfx ? &tmKp : &tmKl, &k_full[ks],
                                     t.h * HD + s * 64, row);
                ++kb;
                ++gk;
                return true;
            };
            auto next_v = [&]() {
                while (vb >= info[vi % kTileRing].nb) {  // the K cursor already claimed item vi (<= ki)
                    ++vi;
                    vb = 0;
                }
                const TileInfo& t = info[vi % kTileRing];
                const bool pfx = vb < t.nA;
                const int row = block_row(t, vb);
                const int vs = gv % C::kVStages;
                pwait(&v_empty[vs], ((gv / C::kVStages) & 1) ^ 1, 25);
                ptx::mbar_expect_tx(&v_full[vs], C::kVBytes);
#pragma unroll
                for (int s = 0; s < C::kSub; ++s)
                    ptx::tma_load_2d(sV + vs * C::kVBytes + s * (BKV * 128), pfx ? &tmVp : &tmVl, &v_full[vs],
                                     t.h * HD + s * 64, row);
                ++vb;
                ++gv;
            };
            // K(0), K(1), then K(g+2), V(g) (SGC_S3_VFIRST=1: V(g) first -- V(g) is due at PV(g),
            // K(g+2) at S(g+2); measured slower at C3, scripts/gpu_attn_ab.sh)
            bool more = next_k() && next_k();
            while (more || gv < gk) {
#if SGC_S3_VFIRST
                if (gv < gk) next_v();
                if (more) more = next_k();
#else
                if (more) more = next_k();
                if (gv < gk) next_v();
#endif
            }
        }
    } else if (warp == 1 || warp == 10) {
        // two MMA issuers (a single thread spends ~17 instructions per tcgen05.mma and was the
        // bottleneck issuing 16 MMAs per 1024 tensor cycles): warp 10 issues S, warp 1 PV.
        // S(g) overwrites buffer g % 3 only after PV(g - 3) read P(g - 3) from it (s_free).
        // each issuer warp runs its loop convergently; one elected lane issues (uniform datapath)
        if (warp == 10) {
            constexpr uint32_t idS = ptx::idesc_bf16_f32(BQ, BKV);
            uint32_t g = 0;
            for (uint32_t k = 0;; ++k) {
                const uint32_t iu = sched::wait(ring, k);
                const int nb = iu < static_cast<uint32_t>(n_items) ? info[k % kTileRing].nb : 0;
                __syncwarp();
                if (lane == 0) sched::release(ring, k);
                if (iu >= static_cast<uint32_t>(n_items)) break;
                pwait(&q_full[k & 1], (k >> 1) & 1, 20);
                const uint64_t qd = ptx::umma_desc_sw128(ptx::smem_u32(sQ + (k & 1) * C::kQBytes));
                for (int b = 0; b < nb; ++b, ++g) {
                    const int ks = g % C::kKStages;
                    const int sbuf = g % 3;
                    if (g >= 3) pwait(&s_free[sbuf], ((g - 3) / 3) & 1, 21);
                    pwait(&k_full[ks], (g / C::kKStages) & 1, 16);
                    ptx::tc_fence_after();
                    const uint64_t kd = ptx::umma_desc_sw128(ptx::smem_u32(sK + ks * C::kKBytes));
                    const uint32_t dS = tmem_base + C::kS + sbuf * 128;
#pragma unroll
                    for (int kc = 0; kc < HD / 16; ++kc) {
                        // descriptor start address field: bytes >> 4
                        const uint64_t ad = qd + (((kc / 4) * (BQ * 128) + (kc % 4) * 32) >> 4);
                        const uint64_t bd = kd + (((kc / 4) * (BKV * 128) + (kc % 4) * 32) >> 4);
                        ptx::mma_bf16_elect(dS, ad, bd, idS, kc > 0 ? 1u : 0u);
                    }
                    ptx::mma_commit_elect(&s_full[sbuf]);
                    ptx::mma_commit_elect(&k_empty[ks]);
                    if (b == nb - 1) ptx::mma_commit_elect(&q_empty[k & 1]);
                }
            }
        } else {
            constexpr uint32_t idO = ptx::idesc_bf16_f32_bmn(BQ, HD);
            uint32_t g = 0;
            for (uint32_t k = 0;; ++k) {
                const uint32_t iu = sched::wait(ring, k);
                const int nb = iu < static_cast<uint32_t>(n_items) ? info[k % kTileRing].nb : 0;
                __syncwarp();
                if (lane == 0) sched::release(ring, k);
                if (iu >= static_cast<uint32_t>(n_items)) break;
                if (k > 0) pwait(o_free, (k - 1) & 1, 19);  // the previous tile's epilogue read O
                for (int b = 0; b < nb; ++b, ++g) {
                    const int vs = g % C::kVStages;
                    const int pbuf = g % 3;
                    pwait(&v_full[vs], (g / C::kVStages) & 1, 17);
                    pwait(&p_full[pbuf], (g / 3) & 1, 18);
                    ptx::tc_fence_after();
                    const uint64_t vd = ptx::umma_desc_sw128_lbo(ptx::smem_u32(sV + vs * C::kVBytes), BKV * 128, 1024);
                    const uint32_t aP = tmem_base + C::kS + pbuf * 128;
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk)
                        ptx::mma_bf16_ts_elect(tmem_base + C::kO, aP + kk * 8, vd + ((kk * 16 * 128) >> 4), idO,
                                         (b > 0 || kk > 0) ? 1u : 0u);
                    ptx::mma_commit_elect(&v_empty[vs]);
                    ptx::mma_commit_elect(&s_free[pbuf]);
                    if (b == nb - 1) ptx::mma_commit_elect(o_full);
                }
            }
        }
    } else {
        const int wg = (warp - 2) / 4;            // softmax warpgroup: blocks with g % 2 == wg
        const int r = (warp & 3) * 32 + lane;     // row within the tile == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
        const uint32_t tO = tmem_base + lane_base + C::kO;
        // decision token (this warpgroup -> the other): named barriers 3 + wg / 4 - wg for even
        // tiles, 5 + wg / 6 - wg for odd ones (a warpgroup starts the next tile without waiting
        // for the other, so a tile's last token may still be pending when the next tile's first
        // is posted)
        uint32_t G = 0, uit = 0;  // first global block of the current tile, tiles done
#ifdef SGC_ATTN_PROF
        const bool prof_thr = threadIdx.x == 64 || threadIdx.x == 192;
        long long _pt = clock64();
#define SPROF(slot)                                                                                        \
    if (prof_thr) {                                                                                        \
        long long _n = clock64();                                                                          \
        atomicAdd(&g_attn_prof[(blockIdx.x % 148) * 32 + wg * 8 + (slot)], (unsigned long long)(_n - _pt)); \
        _pt = _n;                                                                                          \
    }
#else
#define SPROF(slot)
#endif
        for (uint32_t k = 0;; ++k) {
            const uint32_t iu = sched::wait(ring, k);
            TileInfo t;
            if (iu < static_cast<uint32_t>(n_items)) t = info[k % kTileRing];
            __syncwarp();
            if (lane == 0) sched::release(ring, k);
            if (iu >= static_cast<uint32_t>(n_items)) break;
            SPROF(7);
            const bool valid = r < t.nrows;
            const int row = t.w.row0 + t.x * BQ + r;
            const int seg = valid && !partial ? p.seg_lo[row] : 0x7fffffff;
            float m_w = -INFINITY, l_w = 0.f;  // this warpgroup's row sum, relative to m_w
            float m_prev = -INFINITY;            // the max the tile's last block started from
            float* m_shk = m_sh + (uit & 1) * BQ;
            const int bar_post = 3 + wg + 2 * (uit & 1), bar_take = 4 - wg + 2 * (uit & 1);
            for (int b = (static_cast<int>(G) + wg) & 1 ? 1 : 0; b < t.nb; b += 2) {
                const uint32_t g = G + b;
                const int sbuf = g % 3;
                const uint32_t tS = tmem_base + lane_base + C::kS + sbuf * 128;
                SPROF(0);
                ptx::mbar_wait(&s_full[sbuf], (g / 3) & 1);
                ptx::tc_fence_after();
                SPROF(1);
                int k0, klo, khi;  // visible key window [klo, khi] in block-local index
                if (b < t.nA) {
                    k0 = b * BKV;
                    klo = 0;
                    khi = valid ? min(BKV, t.w.pfx_len - k0) - 1 : -1;
                } else {
                    k0 = t.loc_first + (b - t.nA) * BKV;
                    klo = max(0, seg - k0);
                    khi = valid ? min(BKV - 1, row - k0) : -1;
                }
                const bool full = __all_sync(0xffffffffu, klo <= 0 && khi >= BKV - 1);
                const float sc = p.scale_log2;
                uint32_t sv[BKV];
#pragma unroll
                for (int c = 0; c < BKV / 32; ++c)
                    ptx::tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
                ptx::tmem_ld_wait();
                if (!full) {
                    uint32_t vw[BKV / 32];
#pragma unroll
                    for (int wd = 0; wd < BKV / 32; ++wd) {
                        const int lo = klo - 32 * wd, hi = khi - 32 * wd;
                        const uint32_t mlo = lo <= 0 ? ~0u : (lo >= 32 ? 0u : ~0u << lo);
                        const uint32_t mhi = hi >= 31 ? ~0u : (hi < 0 ? 0u : ~0u >> (31 - hi));
                        vw[wd] = mlo & mhi;
                    }
#pragma unroll
                    for (int j = 0; j < BKV; ++j)
                        if (!(vw[j / 32] & (1u << (j % 32)))) sv[j] = __float_as_uint(-INFINITY);
                }
                float bmax;
                {
                    float q0 = -INFINITY, q1 = -INFINITY, q2 = -INFINITY, q3 = -INFINITY;
#pragma unroll
                    for (int j = 0; j < BKV; j += 8) {
                        q0 = fmax3(q0, __uint_as_float(sv[j]), __uint_as_float(sv[j + 1]));
                        q1 = fmax3(q1, __uint_as_float(sv[j + 2]), __uint_as_float(sv[j + 3]));
                        q2 = fmax3(q2, __uint_as_float(sv[j + 4]), __uint_as_float(sv[j + 5]));
                        q3 = fmax3(q3, __uint_as_float(sv[j + 6]), __uint_as_float(sv[j + 7]));
                    }
                    bmax = fmaxf(fmaxf(q0, q1), fmaxf(q2, q3)) * sc;  // scaled-log2 units
                }
                SPROF(2);
                // the running max as the previous block of this tile left it (the other
                // warpgroup's decision, handed over through a named barrier)
                float m_cur = -INFINITY;
                if (b > 0) {
                    asm volatile("bar.sync %0, 256;" ::"r"(bar_take) : "memory");
                    m_cur = m_shk[r];
                }
                m_prev = m_cur;
                if (m_cur != m_w) {  // the other warpgroup moved the max: re-base this row sum
                    l_w = m_w == -INFINITY ? 0.f : l_w * ex2_approx(m_w - m_cur);
                    m_w = m_cur;
                }
                const float mnew = (m_cur == -INFINITY || bmax > m_cur + SGC_LAZY_MAX) ? bmax : m_cur;
                if (b == 0 || mnew != m_cur) m_shk[r] = mnew;
#if !SGC_S3_TOKEN_LATE
                if (b + 1 < t.nb) asm volatile("bar.arrive %0, 256;" ::"r"(bar_post) : "memory");
#endif
                const float nm = mnew == -INFINITY ? 0.f : -mnew;
                SPROF(3);
                float rs;
                {
                    const uint64_t sc2 = f2pack(sc, sc), nm2 = f2pack(nm, nm);
                    uint64_t r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
                    for (int j = 0; j < BKV / 2; ++j) {
                        float xa, xc;
                        f2unpack(ffma2(f2pack(__uint_as_float(sv[2 * j]), __uint_as_float(sv[2 * j + 1])), sc2, nm2),
                                 xa, xc);
                        float a, cc;
                        if ((j % SGC_POLY_DEN) < SGC_POLY_NUM) {
                            ex2_poly2(xa, xc, a, cc);
                        } else {
                            a = ex2_approx(xa);
                            cc = ex2_approx(xc);
                        }
                        const uint64_t pr = f2pack(a, cc);
                        if ((j & 3) == 0) r0 = fadd2(r0, pr);
                        else if ((j & 3) == 1) r1 = fadd2(r1, pr);
                        else if ((j & 3) == 2) r2 = fadd2(r2, pr);
                        else r3 = fadd2(r3, pr);
                        __nv_bfloat162 bv = __floats2bfloat162_rn(a, cc);
                        sv[j] = *reinterpret_cast<uint32_t*>(&bv);
                    }
                    float x0, x1;
                    f2unpack(fadd2(fadd2(r0, r1), fadd2(r2, r3)), x0, x1);
                    rs = x0 + x1;
                }
#if SGC_S3_TOKEN_LATE
                // hand the token on after the exponentials: the next block's exponentials start
                // when these end (the two warpgroups take turns on MUFU)
                if (b + 1 < t.nb) asm volatile("bar.arrive %0, 256;" ::"r"(bar_post) : "memory");
#endif
                SPROF(4);
                const bool resc = m_cur != -INFINITY && mnew > m_cur;
                if (__any_sync(0xffffffffu, resc)) {
                    // O holds PV(0 .. g-1) relative to m_cur: rescale once PV(g-1) completed.
                    // s_free[(g-1) % 3] phase (g-1)/3: its previous phase (PV(g-4)) is certified
                    // by s_full(g) (S(g) was issued after PV(g-3)), its next (PV(g+2)) needs this
                    // warpgroup's P(g+2) -- the parity is unambiguous
                    ptx::mbar_wait(&s_free[(g - 1) % 3], ((g - 1) / 3) & 1);
                    ptx::tc_fence_after();
                    const float alpha = resc ? ex2_approx(m_cur - mnew) : 1.f;
                    l_w *= alpha;
#pragma unroll 1
                    for (int c = 0; c < HD / 32; ++c) {
                        uint32_t o[32];
                        ptx::tmem_ld32(tO + c * 32, o);
                        ptx::tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
                        ptx::tmem_st32(tO + c * 32, o);
                    }
                }
                m_w = mnew;
                l_w += rs;
                // P -> TMEM over the buffer's first 64 columns
#pragma unroll
                for (int c = 0; c < BKV / 32; ++c)
                    ptx::tmem_st16(tS + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&sv[c * 16]));
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&p_full[sbuf]);
                SPROF(5);
            }
            const int last_wg = (G + t.nb - 1) & 1;  // the warpgroup of the tile's last block
            G += t.nb;
            // epilogue by the warpgroup of the tile's last block alone: the other hands over its
            // row sum (relative to the max the last block started from) and goes on with the next
            // tile's first block while this one waits for the last PV, reads O and frees it
            float* lxk = lx + (uit & 1) * BQ;
            const int bar_epi = 1 + (uit & 1);
            if (wg != last_wg) {
                lxk[r] = l_w;
                asm volatile("bar.arrive %0, 256;" ::"r"(bar_epi) : "memory");
            } else {
                asm volatile("bar.sync %0, 256;" ::"r"(bar_epi) : "memory");
                const float m_fin = m_w;
                const float lo = lxk[r];
                const float l = l_w + (m_prev == -INFINITY ? 0.f : lo * ex2_approx(m_prev - m_fin));
                ptx::mbar_wait(o_full, uit & 1);
                ptx::tc_fence_after();
                const float il = l > 0.f ? 1.f / l : 0.f;
#pragma unroll 1
                for (int hh = 0; hh < 2; ++hh) {  // two halves of the row (register budget)
                    constexpr int OCOLS = HD / 2;
                    uint32_t o[OCOLS];
#pragma unroll
                    for (int c = 0; c < OCOLS / 32; ++c)
                        ptx::tmem_ld32(tO + hh * OCOLS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&o[c * 32]));
                    ptx::tmem_ld_wait();
                    if (hh == 1) {
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(o_free);
                    }
                    if (valid && partial) {
                        float* dst = p.part_o + static_cast<size_t>(row) * p.d + t.h * HD + hh * OCOLS;
#pragma unroll
                        for (int q = 0; q < OCOLS / 8; ++q) {
                            uint32_t wv[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) wv[e] = __float_as_uint(__uint_as_float(o[8 * q + e]) * il);
                            ptx::st_global_v8(dst + 8 * q, wv);
                        }
                    } else if (valid) {
                        __nv_bfloat16* dst = p.out + static_cast<size_t>(row) * p.d + t.h * HD + hh * OCOLS;
#pragma unroll
                        for (int q = 0; q < OCOLS / 16; ++q) {
                            uint32_t wv[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                __nv_bfloat162 bv = __floats2bfloat162_rn(__uint_as_float(o[16 * q + 2 * e]) * il,
                                                                          __uint_as_float(o[16 * q + 2 * e + 1]) * il);
                                wv[e] = *reinterpret_cast<uint32_t*>(&bv);
                            }
                            ptx::st_global_v8(dst + 16 * q, wv);
                        }
                    }
                }
                if (valid && partial)
                    p.part_lse[static_cast<size_t>(row) * p.heads + t.h] = l > 0.f ? m_fin + __log2f(l) : -INFINITY;
            }
            ++uit;
            SPROF(6);
        }
#undef SPROF
    }
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// 0: two-tile kernel (attn_tc_kernel, default), 1: attn_s3_kernel (sgc_set_option "attn_kernel").
// Same-box A/B at C3 (scripts/gpu_attn_ab.sh): 112.4 / 112.3 vs 115.8 / 115.8 ms per step once the
// two-tile kernel's MMA thread built its descriptors once per operand tile (it was 115.6-118)
int g_attn_kernel = 0;
// the same choice for partial mode (decode steps: prefix keys only), sgc_set_option "attn_kernel_partial"
int g_attn_kernel_partial = 1;

template <int HD>
void launch_s3(Ctx* c, const AttnParams& a, int n_work, int heads, int q_rows, int pfx_rows, int loc_rows) {
    using Cf = S3Cfg<HD>;
    auto kfn = attn_s3_kernel<HD>;
    static std::atomic<uint64_t> attr_devices{0};
    if (!(attr_devices.load() >> c->device & 1)) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem));
        attr_devices |= 1ull << c->device;
    }
    const int d = a.d;
    CUtensorMap tq = make_map_2d(a.q, q_rows, d, BQ, 64);
    CUtensorMap tkp = make_map_2d(a.k_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tvp = make_map_2d(a.v_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tkl = make_map_2d(a.k_loc, loc_rows, d, BKV, 64);
    CUtensorMap tvl = make_map_2d(a.v_loc, loc_rows, d, BKV, 64);
    TcParams p{a.work, n_work, heads, a.part_o, a.part_lse, a.seg_lo, a.out, d, a.scale * 1.4426950408889634f,
               c->sched_counter(), a.bt};
    const int items = 2 * n_work * heads;
    const int grid = items < c->num_sms ? items : c->num_sms;
    Ctx::Timed timer(c, "attention");
    kfn<<<grid, 352, Cf::kSmem, c->stream>>>(tq, tkp, tvp, tkl, tvl, p);
    SGC_LAUNCH_CHECK(c);
}

template <int HD, int SPLIT>
void launch_tc(Ctx* c, const AttnParams& a, int n_work, int heads, int q_rows, int pfx_rows, int loc_rows) {
    using Cf = TcCfg<HD>;
    auto kfn = attn_tc_kernel<HD, SPLIT>;
    static std::atomic<uint64_t> attr_devices{0};  // function attributes are per device
    if (!(attr_devices.load() >> c->device & 1)) {
        SGC_CUDA_CHECK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::kSmem));
        attr_devices |= 1ull << c->device;
    }
    const int d = a.d;
    CUtensorMap tq = make_map_2d(a.q, q_rows, d, BQ, 64);
    CUtensorMap tkp = make_map_2d(a.k_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tvp = make_map_2d(a.v_pfx, pfx_rows, d, BKV, 64);
    CUtensorMap tkl = make_map_2d(a.k_loc, loc_rows, d, BKV, 64);
    CUtensorMap tvl = make_map_2d(a.v_loc, loc_rows, d, BKV, 64);
    TcParams p{a.work, n_work, heads, a.part_o, a.part_lse, a.seg_lo, a.out, d, a.scale * 1.4426950408889634f,
                c->sched_counter(), a.bt};
    const int items = n_work * heads;
    const int grid = items < c->num_sms ? items : c->num_sms;
    Ctx::Timed timer(c, "attention");
    kfn<<<grid, 64 + 256 * SPLIT, Cf::kSmem, c->stream>>>(tq, tkp, tvp, tkl, tvl, p);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace

#ifdef SGC_ATTN_PROF
void attn_prof_read(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, g_attn_prof, sizeof(unsigned long long) * 148 * 32);
}
void attn_prof_reset() {
    static unsigned long long z[148 * 32] = {};
    cudaMemcpyToSymbol(g_attn_prof, z, sizeof(z));
}
#endif

bool cascade_attention_tc(Ctx* c, const AttnParams& p, int n_work, int heads, int hd, int q_rows,
                          int pfx_rows, int loc_rows) {
    if (n_work <= 0) return true;
    if (p.loc_kv0 != 0) return false;
    if (p.part_o && !p.part_lse) return false;
    // decode (partial mode): a cluster's generating members rarely fill one 128-row tile, so the
    // two-tile kernel runs one tile per item with no second chain to overlap its softmax; the
    // one-tile kernel keeps two warpgroups busy on alternate key blocks of that tile
    const int kern = p.part_o ? g_attn_kernel_partial : g_attn_kernel;
    if (kern == 1) {
        switch (hd) {
            case 64: launch_s3<64>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows); return true;
            case 128: launch_s3<128>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows); return true;
            default: return false;
        }
    }
    const bool split = g_attn_split;
    switch (hd) {
        case 64:
            if (split) launch_tc<64, 2>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows);
            else launch_tc<64, 1>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows);
            return true;
        case 128:
            if (split) launch_tc<128, 2>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows);
            else launch_tc<128, 1>(c, p, n_work, heads, q_rows, pfx_rows, loc_rows);
            return true;
        default: return false;
    }
}

void attention_set_split(bool on) { g_attn_split = on; }
void attention_set_kernel(int k) { g_attn_kernel = k; }
void attention_set_kernel_partial(int k) { g_attn_kernel_partial = k; }

}  // namespace sgc
