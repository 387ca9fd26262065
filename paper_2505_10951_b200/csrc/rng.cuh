// rng.cuh -- counter-form SplitMix64 (rng.hpp:12-34) for on-device weight generation.
#pragma once
#include <stdint.h>

namespace sgc {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// splitmix64_once (rng.hpp:36-39)
__host__ __device__ __forceinline__ uint64_t splitmix64_once(uint64_t x) { return mix64(x + kGamma); }

// Element i of a SplitMix64 stream seeded with state0 is mix(state0 + (i+1)*gamma);
// uniform(lo,hi) = lo + (hi - lo) * u with u = top 24 bits * 2^-24 (rng.hpp:25-28), no FMA.
__device__ __forceinline__ float uniform_at(uint64_t state0, uint64_t i, float lo, float hi) {
    uint64_t z = mix64(state0 + (i + 1) * kGamma);
    float u = __fmul_rn(static_cast<float>(z >> 40), 0x1.0p-24f);
    return __fadd_rn(lo, __fmul_rn(__fsub_rn(hi, lo), u));
}

}  // namespace sgc
