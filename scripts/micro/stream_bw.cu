// stream_bw.cu -- weight-streaming microbenchmark (decode-step GEMM operand path, no MMA):
// every CTA streams its share of a [N x K] bf16 matrix through a STAGES-deep smem ring, either
// as 2D TMA boxes of 128 rows x 128 B (row-major weights, the GEMM's B-operand loads) or as 1D
// bulk copies of 16 KB contiguous blocks (the same bytes pre-tiled). Prints GB/s of each.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw stream_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

#ifndef STAGES
#define STAGES 6
#endif
constexpr int TILE = 16384;  // bytes per operand tile (128 rows x 128 B)
constexpr int STAGE = 2 * TILE;  // B tile + (MODE 2) an A tile

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(s32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(s32(b)),
        "r"(ph)
        : "memory");
}

template <int MODE>  // 0 = 2D TMA boxes, 1 = 1D bulk 16 KB, 2 = 2D TMA B + the activation (A) tile of the k-block
__global__ void __launch_bounds__(32) stream_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap ta,
                                                    const uint8_t* src, int rows,
                                                    int kb_per_row, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * STAGE);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int row_tiles = rows / 128;
    const int total = row_tiles * kb_per_row;  // 16 KB units
    const int per = (total + gridDim.x - 1) / gridDim.x;
    const int u0 = blockIdx.x * per, u1 = min(total, u0 + per);
    unsigned long long acc = 0;
    int issued = u0, done = u0;
    auto issue = [&](int u) {
        const int s = (u - u0) % STAGES;
        expect_tx(&full[s], MODE == 2 ? 2 * TILE : TILE);
        if (MODE != 1) {
            const int rt = u / kb_per_row, kb = u % kb_per_row;  // units along K first (as the GEMM)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                    s32(sm + s * STAGE)),
                "l"(&tm), "r"(s32(&full[s])), "r"(kb * 64), "r"(rt * 128)
                : "memory");
            if (MODE == 2)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                        s32(sm + s * STAGE + TILE)),
                    "l"(&ta), "r"(s32(&full[s])), "r"(kb * 64), "r"((blockIdx.x & 1) * 128)
                    : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             s32(sm + s * STAGE)),
                         "l"(src + static_cast<size_t>(u) * TILE), "r"(TILE), "r"(s32(&full[s]))
                         : "memory");
        }
    };
    while (issued < u1 && issued - u0 < STAGES) issue(issued++);
    while (done < u1) {
        const int s = (done - u0) % STAGES;
        wait(&full[s], ((done - u0) / STAGES) & 1);
        acc += sm[s * STAGE + (done & 1023)];
        ++done;
        if (issued < u1) issue(issued++);
    }
    atomicAdd(sink, acc);
}

int main() {
    const int N = 12288, K = 4096;  // the C3 QKV weights
    const size_t bytes = static_cast<size_t>(N) * K * 2;
    const int copies = 4;  // rotate > L2
    uint8_t* buf;
    cudaMalloc(&buf, bytes * copies);
    cudaMemset(buf, 1, bytes * copies);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm[copies];
    for (int c = 0; c < copies; ++c) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
        cuuint64_t str[1] = {static_cast<cuuint64_t>(K) * 2};
        cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        enc(&tm[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf + c * bytes, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    // activations: 256 rows x K (L2-resident, read by every CTA)
    uint8_t* act;
    cudaMalloc(&act, 256ull * K * 2);
    cudaMemset(act, 1, 256ull * K * 2);
    CUtensorMap ta;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), 256};
        cuuint64_t str[1] = {static_cast<cuuint64_t>(K) * 2};
        cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        enc(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int smem = STAGES * STAGE + 1024;
    cudaFuncSetAttribute(stream_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(stream_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(stream_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int grid : {96, 148, 296}) {
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                const int iters = 40;
                cudaEventRecord(e0);
                for (int i = 0; i < iters; ++i) {
                    const int c = i % copies;
                    if (mode == 0) stream_kernel<0><<<grid, 32, smem>>>(tm[c], ta, buf + c * bytes, N, K / 64, sink);
                    else if (mode == 1) stream_kernel<1><<<grid, 32, smem>>>(tm[c], ta, buf + c * bytes, N, K / 64, sink);
                    else stream_kernel<2><<<grid, 32, smem>>>(tm[c], ta, buf + c * bytes, N, K / 64, sink);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep) printf("grid %3d %-10s %7.1f us/launch  %6.0f GB/s\n", grid, mode == 2 ? "tma-2d+A" : mode ? "bulk-1d" : "tma-2d",
                                ms * 1e3 / iters, bytes / (ms * 1e-3 / iters) / 1e9);
            }
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
