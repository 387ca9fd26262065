// sched.cuh -- dynamic unit scheduling for the persistent tcgen05 kernels (GEMM, attention).
//
// A persistent kernel's CTAs (or CTA pairs) claim work units (output tiles, attention items) in
// increasing order from a global counter instead of a fixed blockIdx stride. Under the B200 power
// cap the SM clocks differ across GPCs by up to ~15% during one kernel (ncu gpc__cycles_elapsed
// .min/.max.per_second: 1.15 vs 1.37 GHz on the W2 GEMM) while every SM needs the same cycles per
// tile, so a static split waits for the slowest GPC's share; claiming units keeps every SM busy
// to the end. Claims stay in raster order, so the L2 grouping of concurrently running tiles holds.
//
// The counter pair [next unit, finished fetchers] lives in the Ctx (one per stream-ordered
// context). Every fetcher's loop ends with exactly one claim past the end; the last of those
// resets the pair, so the next kernel in the stream starts from zero without a host memset.
//
// Inside a CTA the fetcher publishes each claimed unit through a small smem ring (slot + full /
// empty mbarriers) to the warps that consume it (MMA issuer, epilogue / softmax warps). In a CTA
// pair the leader's fetcher also writes the peer's ring over DSMEM; the peer's consumers release
// the slot on the leader's `empty` barrier.
#pragma once
#include <stdint.h>

#include "sm100_ptx.cuh"

namespace sgc {

template <int R>
struct UnitRing {
    uint64_t full[R];
    uint64_t empty[R];
    uint32_t unit[R];
};

namespace sched {

// claim the next unit; a claim >= n_units ends the caller's loop (and, for the last fetcher to
// finish, resets the counter pair for the next kernel)
__device__ __forceinline__ uint32_t claim(uint32_t* ctr, uint32_t n_units, uint32_t n_fetchers, uint32_t k) {
#ifdef SGC_STATIC_SCHED
    // A/B builds only: the fixed stride it replaces (fetcher f takes f, f + n_fetchers, ...)
    (void)ctr;
    (void)n_units;
    return blockIdx.x / (gridDim.x / n_fetchers) + k * n_fetchers;
#else
    (void)k;
    const uint32_t t = atomicAdd(ctr, 1u);
    if (t >= n_units && atomicAdd(ctr + 1, 1u) == n_fetchers - 1) {
        atomicExch(ctr, 0u);
        atomicExch(ctr + 1, 0u);
    }
    return t;
#endif
}

template <int R>
__device__ __forceinline__ void init(UnitRing<R>* r, uint32_t consumers) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        ptx::mbar_init(&r->full[i], 1);
        ptx::mbar_init(&r->empty[i], consumers);
    }
}

// fetcher: publish unit t (claimed ahead: the next claim's atomic round trip overlaps the
// current unit's loads instead of stalling the operand pipeline at every unit boundary) as the
// k-th unit of this CTA (one thread)
template <int R>
__device__ __forceinline__ void publish(UnitRing<R>* r, uint32_t k, uint32_t t) {
    const int s = k % R;
    ptx::mbar_wait(&r->empty[s], ((k / R) & 1) ^ 1);
    r->unit[s] = t;
    ptx::mbar_arrive(&r->full[s]);
}

// CTA-pair leader's fetcher: also writes the peer's (rank 1) ring; the slot's empty barrier
// collects the peer's consumers too, so its wait acquires at cluster scope
template <int R>
__device__ __forceinline__ void publish_pair(UnitRing<R>* r, uint32_t k, uint32_t t) {
    const int s = k % R;
    ptx::mbar_wait_cluster(&r->empty[s], ((k / R) & 1) ^ 1);
    r->unit[s] = t;
    ptx::st_cluster_u32(&r->unit[s], 1, t);
    ptx::mbar_arrive(&r->full[s]);
    ptx::mbar_arrive_cluster(&r->full[s], 1);
}

// consumer: the k-th unit (every thread that calls it gets the value)
template <int R>
__device__ __forceinline__ uint32_t wait(UnitRing<R>* r, uint32_t k) {
    const int s = k % R;
    ptx::mbar_wait(&r->full[s], (k / R) & 1);
    return *reinterpret_cast<volatile uint32_t*>(&r->unit[s]);
}
// peer CTA's consumer: the slot was written over DSMEM by the leader
template <int R>
__device__ __forceinline__ uint32_t wait_remote(UnitRing<R>* r, uint32_t k) {
    const int s = k % R;
    ptx::mbar_wait_cluster(&r->full[s], (k / R) & 1);
    return *reinterpret_cast<volatile uint32_t*>(&r->unit[s]);
}
// release slot k (one arrive per consumer; `rank` = CTA of the ring's fetcher)
template <int R>
__device__ __forceinline__ void release(UnitRing<R>* r, uint32_t k) {
    ptx::mbar_arrive(&r->empty[k % R]);
}
template <int R>
__device__ __forceinline__ void release_to(UnitRing<R>* r, uint32_t k, uint32_t rank) {
    ptx::mbar_arrive_cluster(&r->empty[k % R], rank);
}

}  // namespace sched
}  // namespace sgc
