// common.cuh -- shared host/device plumbing for the sm_100a SubGCache library.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgc_b200.h"
#include "comm.cuh"

namespace sgc {

// ---- error taxonomy (mirrors include/subgcache/errors.hpp:9-32) ---------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

#define SGC_CUDA_CHECK(x)                                                                    \
    do {                                                                                     \
        cudaError_t _e = (x);                                                                \
        if (_e != cudaSuccess)                                                               \
            ::sgc::fail(SGC_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e) + " @" +   \
                                      __FILE__ + ":" + std::to_string(__LINE__));            \
    } while (0)

#define SGC_LAUNCH_CHECK(ctx)                                                                \
    do {                                                                                     \
        cudaError_t _e = cudaGetLastError();                                                 \
        if (_e != cudaSuccess)                                                               \
            ::sgc::fail(SGC_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e) +  \
                                      " @" + __FILE__ + ":" + std::to_string(__LINE__));     \
        (ctx)->launches++;                                                                   \
        if (::sgc::trace_launches()) ::sgc::trace_launch(ctx, __FILE__, __LINE__);           \
    } while (0)

// SGC_TRACE=1: synchronize after every launch and log its site (hang / fault triage)
inline bool trace_launches() {
    static const int on = [] {
        const char* e = std::getenv("SGC_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}
struct Ctx;
void trace_launch(Ctx* c, const char* file, int line);

// ---- device scratch arena: grow-only buffers keyed by name -------------------------------
struct Buffer {
    void* ptr = nullptr;
    size_t bytes = 0;
};

struct KernelTiming {
    double ms = 0;
    uint64_t launches = 0;
};

struct Ctx {
    int device = 0;
    int num_sms = 148;
    // generation: a wave decodes on its own until fewer than this % of its queries are still
    // generating; the stragglers of all waves then finish in one shared loop
    uint32_t decode_defer_pct = 25;
    // last GNN encode: unique node states computed (all layers) / the reference's node instances
    uint64_t gnn_state_rows = 0, gnn_node_instances = 0;
    int gnn_tile = 3;  // GNN layer-map GEMM: DFMA register tiles 0 = 64x64, 1 = 64x128, 2 = 128x128; 3 = DMMA (FP64 tensor pipe)
    // GNN node-state dedup (identical subgraphs / identical per-layer in-neighbourhood signatures
    // computed once; exact): 0 computes every node instance as the reference does (bench.py
    // reports the embedding stage both ways)
    int gnn_dedup = 1;
    cudaStream_t own_stream = nullptr;
    cudaStream_t side = nullptr;  // overlapped side work (sealed-prefix digests), created on first use
    cudaStream_t side_stream() {
        if (!side) SGC_CUDA_CHECK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        return side;
    }
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    std::map<std::string, Buffer> scratch;
    bool timing = false;
    std::map<std::string, KernelTiming> timings;
    // pending (name, start, stop) event triples, resolved when the timings are read
    std::vector<std::pair<std::string, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<cudaEvent_t> event_pool;

    // device free / total memory for the planners, cached: cudaMemGetInfo takes a driver lock
    // that an nvidia-smi / NVML poller holds now and then, and a step that called it stalled its
    // host planning for 10-65 ms (scripts/host_trace.py). Refreshed after a minute or when the
    // KV page pool (the one large allocator) changed size.
    size_t mem_free = 0, mem_total = 0;
    std::chrono::steady_clock::time_point mem_at{};
    bool mem_valid = false;
    void mem_info(size_t* free_b, size_t* total_b) {
        const auto now = std::chrono::steady_clock::now();
        if (!mem_valid || now - mem_at > std::chrono::seconds(60)) {
            SGC_CUDA_CHECK(cudaMemGetInfo(&mem_free, &mem_total));
            mem_at = now;
            mem_valid = true;
        }
        *free_b = mem_free;
        *total_b = mem_total;
    }
    void mem_changed() { mem_valid = false; }

    template <typename T>
    T* buf(const std::string& name, size_t count) {
        Buffer& b = scratch[name];
        size_t need = count * sizeof(T);
        if (need == 0) need = 16;
        if (b.bytes < need) {
            if (b.ptr) SGC_CUDA_CHECK(cudaFreeAsync(b.ptr, stream));
            size_t cap = need + need / 8;
            SGC_CUDA_CHECK(cudaMallocAsync(&b.ptr, cap, stream));
            b.bytes = cap;
        }
        return reinterpret_cast<T*>(b.ptr);
    }

    cudaEvent_t event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        SGC_CUDA_CHECK(cudaEventCreate(&e));
        return e;
    }
    // bracket a launch with events when timing is on
    struct Timed {
        Ctx* c;
        std::string name;
        cudaEvent_t a = nullptr, b = nullptr;
        Timed(Ctx* ctx, const char* n) : c(ctx), name(n) {
            if (c->timing) {
                a = c->event();
                b = c->event();
                cudaEventRecord(a, c->stream);
            }
        }
        ~Timed() {
            if (a) {
                cudaEventRecord(b, c->stream);
                c->pending.push_back({name, {a, b}});
            }
        }
    };
    void resolve_timings() {
        for (auto& p : pending) {
            float ms = 0;
            cudaEventSynchronize(p.second.second);
            cudaEventElapsedTime(&ms, p.second.first, p.second.second);
            KernelTiming& t = timings[p.first];
            t.ms += ms;
            t.launches++;
            event_pool.push_back(p.second.first);
            event_pool.push_back(p.second.second);
        }
        pending.clear();
    }
    // pending event pairs are resolved when the timings are read (or the list grows large), not
    // at every sync: resolving ~1000 pairs right after a sync kept the GPU idle for milliseconds
    void sync() {
        SGC_CUDA_CHECK(cudaStreamSynchronize(stream));
        if (pending.size() > 16384) resolve_timings();
    }
    // grow-only PINNED host buffers keyed by name (asynchronous device -> host copies)
    std::map<std::string, Buffer> pinned_bufs;
    template <typename T>
    T* pinned(const std::string& name, size_t count) {
        Buffer& b = pinned_bufs[name];
        size_t need = std::max<size_t>(16, count * sizeof(T));
        if (b.bytes < need) {
            if (b.ptr) {
                SGC_CUDA_CHECK(cudaStreamSynchronize(stream));  // no copy may still target it
                SGC_CUDA_CHECK(cudaFreeHost(b.ptr));
            }
            SGC_CUDA_CHECK(cudaMallocHost(&b.ptr, need + need / 8));
            b.bytes = need + need / 8;
        }
        return reinterpret_cast<T*>(b.ptr);
    }
    // Pinned staging ring for host -> device plan uploads (row maps, block tables, work lists):
    // cudaMemcpyAsync from pageable memory synchronizes the stream first, so every per-wave /
    // per-decode-step upload used to drain the GPU while the host kept planning. Copies out of the
    // ring are truly asynchronous. The ring is 4 segments; an event recorded when the head leaves
    // a segment guards its reuse, so the host only ever waits for copies enqueued a lap ago.
    static constexpr int kRingSegs = 4;
    uint8_t* ring_base = nullptr;
    size_t ring_seg = 0, ring_head = 0;  // segment bytes; head offset in the whole ring
    cudaEvent_t ring_ev[kRingSegs] = {};
    bool ring_ev_live[kRingSegs] = {};
    void* stage(const void* src, size_t bytes) {
        const size_t need = (bytes + 255) & ~size_t(255);
        if (need > ring_seg) {  // (re)allocate: nothing may still read the old ring
            SGC_CUDA_CHECK(cudaStreamSynchronize(stream));
            if (ring_base) SGC_CUDA_CHECK(cudaFreeHost(ring_base));
            ring_seg = std::max<size_t>(need, 16ull << 20);
            SGC_CUDA_CHECK(cudaMallocHost(&ring_base, ring_seg * kRingSegs));
            for (int i = 0; i < kRingSegs; ++i) {
                if (!ring_ev[i]) SGC_CUDA_CHECK(cudaEventCreateWithFlags(&ring_ev[i], cudaEventDisableTiming));
                ring_ev_live[i] = false;
            }
            ring_head = 0;
        }
        const int seg = static_cast<int>(ring_head / ring_seg);
        if (ring_head + need > static_cast<size_t>(seg + 1) * ring_seg) {  // move to the next segment
            SGC_CUDA_CHECK(cudaEventRecord(ring_ev[seg], stream));
            ring_ev_live[seg] = true;
            const int nxt = (seg + 1) % kRingSegs;
            if (ring_ev_live[nxt]) SGC_CUDA_CHECK(cudaEventSynchronize(ring_ev[nxt]));
            ring_ev_live[nxt] = false;
            ring_head = static_cast<size_t>(nxt) * ring_seg;
        }
        void* dst = ring_base + ring_head;
        std::memcpy(dst, src, bytes);
        ring_head += need;
        return dst;
    }
    // [next unit, finished fetchers] of the persistent kernels' dynamic scheduler (sched.cuh):
    // zeroed once, every kernel leaves it zeroed for the next one in the stream
    uint32_t* sched_ptr = nullptr;
    uint32_t* sched_counter() {
        if (!sched_ptr) {
            sched_ptr = buf<uint32_t>("unit_sched", 4);
            SGC_CUDA_CHECK(cudaMemsetAsync(sched_ptr, 0, 4 * sizeof(uint32_t), stream));
        }
        return sched_ptr;
    }
    // stream-K GEMM ready flags (one per CTA of the largest grid, zeroed once) and the launch
    // sequence number they are compared against
    uint32_t* sk_flags = nullptr;
    uint32_t sk_seq = 0;
    // device [0, 1, ..., n-1] (grown on demand, filled on the device: no host round trip)
    int32_t* iota(int n);
    int iota_n = 0;
    int32_t* iota_ptr = nullptr;
    // error flags raised by kernels: copied (stream-ordered) into pinned host memory and OR-ed
    // there; take_flag() is valid after the next stream sync
    int* h_flags = nullptr;
    int n_flags = 0;
    void flag_readback(const int* d_flag) {
        if (!h_flags) SGC_CUDA_CHECK(cudaMallocHost(&h_flags, 64 * sizeof(int)));
        if (n_flags == 64) {  // rare: fold the pending flags first
            sync();
            int any = 0;
            for (int i = 0; i < n_flags; ++i) any |= h_flags[i];
            h_flags[0] = any;
            n_flags = 1;
        }
        SGC_CUDA_CHECK(cudaMemcpyAsync(h_flags + n_flags, d_flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
        ++n_flags;
    }
    bool take_flag() {
        int any = 0;
        for (int i = 0; i < n_flags; ++i) any |= h_flags[i];
        n_flags = 0;
        return any != 0;
    }
};

// copy helpers that accept host or device pointers (cudaMemcpyDefault under UVA)
template <typename T>
inline void copy_in(Ctx* c, T* dst_dev, const T* src, size_t n) {
    if (n) SGC_CUDA_CHECK(cudaMemcpyAsync(dst_dev, src, n * sizeof(T), cudaMemcpyDefault, c->stream));
}
// host (pageable) -> device through the context's pinned staging ring: no stream drain
template <typename T>
inline void copy_in_staged(Ctx* c, T* dst_dev, const T* src_host, size_t n) {
    if (n)
        SGC_CUDA_CHECK(cudaMemcpyAsync(dst_dev, c->stage(src_host, n * sizeof(T)), n * sizeof(T),
                                       cudaMemcpyDefault, c->stream));
}
template <typename T>
inline void copy_out(Ctx* c, T* dst, const T* src_dev, size_t n) {
    if (n && dst) SGC_CUDA_CHECK(cudaMemcpyAsync(dst, src_dev, n * sizeof(T), cudaMemcpyDefault, c->stream));
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace sgc

// opaque handle definitions
struct sgc_ctx {
    sgc::Ctx c;
    std::unique_ptr<sgc::Comm> comm;  // multi-GPU transport (comm.cuh), null = single GPU
};
