// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM for 4 / 8 / 12 warps, and
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_bw scripts/micro/tmem_bw.cu
// tcgen05.st. Prints cycles per warp-load and bytes/clk/SM.
#include <cstdio>
#include <cstdint>
#include "../../paper_2505_10951_b200/csrc/sm100_ptx.cuh"
using namespace sgc;

template <int NW, bool ST>
__global__ void __launch_bounds__(NW * 32) bench(unsigned long long* out, float* sink, int iters) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp / 4) * 128;
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            if (ST) {
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(acc + j);
                ptx::tmem_st32(base + c * 32, v);
            } else {
                ptx::tmem_ld32(base + c * 32, v);
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += __uint_as_float(v[j]);
            }
        }
        if (ST) ptx::tmem_st_wait();
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<512>(slot);
}

template <int NW, bool ST>
void run(const char* name) {
    unsigned long long* d;
    float* s;
    cudaMalloc(&d, 148 * 8);
    cudaMalloc(&s, 148 * NW * 32 * 4);
    const int iters = 2000;
    bench<NW, ST><<<148, NW * 32>>>(d, s, iters);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    const double bytes = static_cast<double>(iters) * 4 * NW * 32 * 32 * 4;
    printf("%-10s warps=%2d: %.1f cycles per warp-op (x32), %.1f B/clk/SM\n", name, NW,
           cyc / (iters * 4.0), bytes / cyc);
    cudaFree(d);
    cudaFree(s);
}

int main() {
    run<4, false>("ld");
    run<8, false>("ld");
    run<12, false>("ld");
    run<4, true>("st");
    run<8, true>("st");
    return 0;
}
