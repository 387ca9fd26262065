// gnn_kernels.cuh -- host interface of gnn_kernels.cu
#pragma once
#include <stdint.h>

namespace sgc {
struct Ctx;

// One message-passing layer over the layer's UNIQUE output states: group g aggregates
// state_prev[self_row[g]] + sum_{e} state_prev[in_src[e]] * feat[in_gate[e]] (ascending edge
// order) and maps it through the folded layer weights. Node instances of different subgraphs
// whose l-hop in-neighbourhood signatures agree share one group (bit-identical states).
struct GnnLayerPlan {
    int n_out;
    const uint32_t* self_row;
    const uint32_t* in_off;
    const uint32_t* in_src;
    const uint32_t* in_gate;
};

struct GnnPlan {
    int layers, heads, d;
    int n0;                    // layer-0 groups (distinct nodes)
    const uint32_t* g0_node;   // [n0] feature row of each layer-0 group
    GnnLayerPlan layer[8];
    int n_sub;
    const uint32_t* sub_off;   // [n_sub+1] into sub_rows
    const uint32_t* sub_rows;  // last-layer state row of every node of every subgraph
    const float* feat;         // text features [(nodes+edges) x d]
    const double* wbar;        // [layers x d x d]
    double* state[2];          // ping-pong [max groups x d]
    double* agg;               // [max groups x d]
    float* out;                // [n_sub x d]
};

void gnn_gen_wbar(Ctx* c, double* wbar, int layers, int heads, int d, uint64_t state0, float scale);
void gnn_encode_layers(Ctx* c, const GnnPlan& p);
void gather_rows(Ctx* c, float* out, const float* src, const uint32_t* idx, int n, int d);
// measured FP64 FMA throughput of this device (TFLOP/s, best of 5 short launches)
double fp64_probe_tflops(Ctx* c);
// the same for the FP64 tensor pipe (DMMA m16n8k4 chains)
double dmma_probe_tflops(Ctx* c);
}  // namespace sgc
