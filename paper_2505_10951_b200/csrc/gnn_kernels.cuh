// gnn_kernels.cuh -- host interface of gnn_kernels.cu
#pragma once
#include <stdint.h>

namespace sgc {
struct Ctx;

struct GnnBatch {
    int layers, heads, d;
    int n_inst, n_sub;
    const uint32_t* inst_feat;     // [n_inst] feature row of the node
    const uint32_t* in_off;        // [n_inst+1] in-edges CSR by destination
    const uint32_t* in_src;        // source instance
    const uint32_t* in_gate;       // feature row of the edge text
    const uint32_t* sub_inst_off;  // [n_sub+1]
    const float* feat;             // text features [(nodes+edges) x d]
    const double* wbar;            // [layers x d x d]
    double* state;                 // [n_inst x d]
    double* agg;                   // [n_inst x d]
    float* out;                    // [n_sub x d]
};

void gnn_gen_wbar(Ctx* c, double* wbar, int layers, int heads, int d, uint64_t state0, float scale);
void gnn_encode_batch(Ctx* c, const GnnBatch& b);
}  // namespace sgc
