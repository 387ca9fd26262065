// cluster_kernels.cuh -- host interface of cluster_kernels.cu
#pragma once
#include <stdint.h>

namespace sgc {
struct Ctx;
// D [m x m] fp64 (zero diagonal); squared = ward/centroid (sqrt then square)
void pairwise_distances(Ctx* c, double* D, const float* emb, int m, int dim, bool squared);
// merge loop over D (destroyed); outputs are device pointers
void agglomerate(Ctx* c, double* D, int m, int clusters, int linkage, uint32_t* labels,
                 uint32_t* merge_left, uint32_t* merge_right, double* merge_dist);
// tests: keep the merge loop's per-row state in global memory at any m (the > ~8k-point path)
void agglomerate_set_global(bool on);
}  // namespace sgc
