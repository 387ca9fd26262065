// gnn_kernels.cu -- GnnEncoder::encode (encoders.cpp:106-186) batched over all subgraphs of a
// batch, in fp64, over UNIQUE node states: the host plan (api.cu encode_subgraphs) groups node
// instances whose layer-l in-neighbourhood signatures agree, so each distinct state is computed
// once (C3: 18.5k instances -> 0.9k..2.3k states per layer) and results stay bit-identical.
//
//   aggregate : agg[g] = (s[self] + sum_{e: src->v, ascending e} s[src] * gate_e) * (1/fanin)
//               -- same operand order as the reference, mul/add rounded separately
//   layer map : s'[v] = tanh((Wbar . agg[v]) / heads), Wbar = sum_h W_h folded once in fp64
//               (register-tiled DFMA GEMM over [instances x dim] . [dim x dim]^T)
//   pool      : mean over v (ascending node id), L2 normalize (sequential), cast to float
#include "common.cuh"
#include "gnn_kernels.cuh"
#include "rng.cuh"

namespace sgc {
namespace {

// Wbar[l][r][c] = ((W0 + W1) + W2) + W3 in double; W_h from the GnnEncoder stream
// (encoders.cpp:95-104: index ((l*H + h)*d + r)*d + c)
__global__ void gen_wbar_kernel(double* wbar, int layers, int heads, int d, uint64_t state0,
                                float scale) {
    const uint64_t dd = static_cast<uint64_t>(d) * d;
    const uint64_t n = static_cast<uint64_t>(layers) * dd;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t l = i / dd, rc = i % dd;
        double s = 0.0;
        for (int h = 0; h < heads; ++h)
            s += static_cast<double>(uniform_at(state0, (l * heads + h) * dd + rc, -scale, scale));
        wbar[i] = s;
    }
}

// one CTA per output group; threads over the feature dim. The group's self row and in-edge
// list (ascending edge index) index the previous layer's unique states.
__global__ void gnn_aggregate_kernel(double* agg, const double* state, const uint32_t* self_row,
                                     const uint32_t* in_off, const uint32_t* in_src,
                                     const uint32_t* in_gate, const float* feat, int d) {
    const int v = blockIdx.x;
    const uint32_t e0 = in_off[v], e1 = in_off[v + 1];
    const double inv = __ddiv_rn(1.0, static_cast<double>(1 + (e1 - e0)));
    const size_t self = self_row[v];
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double a = state[self * d + k];
        for (uint32_t e = e0; e < e1; ++e) {
            double s = state[static_cast<size_t>(in_src[e]) * d + k];
            double g = static_cast<double>(feat[static_cast<size_t>(in_gate[e]) * d + k]);
            a = __dadd_rn(a, __dmul_rn(s, g));
        }
        agg[static_cast<size_t>(v) * d + k] = __dmul_rn(a, inv);
    }
}

// initial state: s[v] = double(text feature of the node)
__global__ void gnn_init_kernel(double* state, const uint32_t* inst_feat, const float* feat,
                                int n_inst, int d) {
    const uint64_t n = static_cast<uint64_t>(n_inst) * d;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t v = i / d, k = i % d;
        state[i] = static_cast<double>(feat[static_cast<size_t>(inst_feat[v]) * d + k]);
    }
}

constexpr int GM = 64, GN = 64, GK = 16;
// out[v][r] = tanh(sum_c W[r][c] * A[v][c] * inv_heads); 256 threads, 4x4 outputs each
__global__ void __launch_bounds__(256)
    gnn_layer_gemm(double* out, const double* A, const double* W, int n_inst, int d,
                   double inv_heads) {
    __shared__ double As[GK][GM + 1];
    __shared__ double Bs[GK][GN + 1];
    const int v0 = blockIdx.x * GM, r0 = blockIdx.y * GN;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < d; k0 += GK) {
        for (int idx = threadIdx.x; idx < GM * GK; idx += 256) {
            int r = idx / GK, kk = idx % GK;
            As[kk][r] = v0 + r < n_inst ? A[static_cast<size_t>(v0 + r) * d + k0 + kk] : 0.0;
            Bs[kk][r] = r0 + r < d ? W[static_cast<size_t>(r0 + r) * d + k0 + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = As[kk][ty + 16 * q];
                b[q] = Bs[kk][tx + 16 * q];
            }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int v = v0 + ty + 16 * p, r = r0 + tx + 16 * q;
            if (v < n_inst && r < d) out[static_cast<size_t>(v) * d + r] = tanh(acc[p][q] * inv_heads);
        }
}

// mean-pool over the subgraph's node states (ascending node id), sequential L2 norm, cast
// (encoders.cpp:170-185); rows index the last layer's unique states
__global__ void gnn_pool_kernel(float* out, const double* state, const uint32_t* sub_off,
                                const uint32_t* rows, int d) {
    extern __shared__ double pooled[];
    __shared__ double norm_s;
    const int u = blockIdx.x;
    const uint32_t v0 = sub_off[u], v1 = sub_off[u + 1];
    const double inv_n = __ddiv_rn(1.0, static_cast<double>(v1 - v0));
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double p = 0.0;
        for (uint32_t v = v0; v < v1; ++v) p = __dadd_rn(p, state[static_cast<size_t>(rows[v]) * d + k]);
        pooled[k] = __dmul_rn(p, inv_n);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double n = 0.0;
        for (int k = 0; k < d; ++k) n = __dadd_rn(n, __dmul_rn(pooled[k], pooled[k]));
        norm_s = __dsqrt_rn(n);
    }
    __syncthreads();
    const double nrm = norm_s;
    for (int k = threadIdx.x; k < d; k += blockDim.x)
        out[static_cast<size_t>(u) * d + k] = nrm > 0.0 ? static_cast<float>(__ddiv_rn(pooled[k], nrm)) : 0.0f;
}

__global__ void gather_rows_kernel(float* out, const float* src, const uint32_t* idx, int d) {
    const int i = blockIdx.x;
    const float* s = src + static_cast<size_t>(idx[i]) * d;
    for (int k = threadIdx.x; k < d; k += blockDim.x) out[static_cast<size_t>(i) * d + k] = s[k];
}

}  // namespace

void gnn_gen_wbar(Ctx* c, double* wbar, int layers, int heads, int d, uint64_t state0, float scale) {
    uint64_t n = static_cast<uint64_t>(layers) * d * d;
    unsigned g = ceil_div(n, 256);
    gen_wbar_kernel<<<g < 8192 ? g : 8192, 256, 0, c->stream>>>(wbar, layers, heads, d, state0, scale);
    SGC_LAUNCH_CHECK(c);
}

void gnn_encode_layers(Ctx* c, const GnnPlan& p) {
    const int d = p.d;
    const int threads = d >= 256 ? 256 : 64;
    Ctx::Timed timer(c, "gnn_encode");
    {
        uint64_t n = static_cast<uint64_t>(p.n0) * d;
        unsigned g = ceil_div(n, 256);
        gnn_init_kernel<<<g < 8192 ? g : 8192, 256, 0, c->stream>>>(p.state[0], p.g0_node, p.feat, p.n0, d);
        SGC_LAUNCH_CHECK(c);
    }
    for (int l = 0; l < p.layers; ++l) {
        const GnnLayerPlan& L = p.layer[l];
        double* prev = p.state[l & 1];
        double* next = p.state[(l + 1) & 1];
        gnn_aggregate_kernel<<<L.n_out, threads, 0, c->stream>>>(p.agg, prev, L.self_row, L.in_off, L.in_src,
                                                                 L.in_gate, p.feat, d);
        SGC_LAUNCH_CHECK(c);
        dim3 grid(ceil_div(L.n_out, GM), ceil_div(d, GN));
        gnn_layer_gemm<<<grid, 256, 0, c->stream>>>(next, p.agg, p.wbar + static_cast<size_t>(l) * d * d,
                                                     L.n_out, d, 1.0 / p.heads);
        SGC_LAUNCH_CHECK(c);
    }
    size_t smem = static_cast<size_t>(d) * sizeof(double);
    if (smem > 48 * 1024)
        SGC_CUDA_CHECK(cudaFuncSetAttribute(gnn_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
    gnn_pool_kernel<<<p.n_sub, threads, smem, c->stream>>>(p.out, p.state[p.layers & 1], p.sub_off,
                                                          p.sub_rows, d);
    SGC_LAUNCH_CHECK(c);
}

void gather_rows(Ctx* c, float* out, const float* src, const uint32_t* idx, int n, int d) {
    if (n <= 0) return;
    gather_rows_kernel<<<n, d >= 256 ? 256 : 64, 0, c->stream>>>(out, src, idx, d);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace sgc
