// cluster_kernels.cu -- exact fp64 pairwise distances and the Lance-Williams agglomeration
// (clustering.cpp:33-174) on the device, bit-identical to the reference.
//
// Exactness rules: direct-form sum over k in sequential order with every
// mul/add rounded separately (__dmul_rn/__dadd_rn, no FMA), sqrt then square for
// ward/centroid, the same Lance-Williams operand order, and the (value, i, j) lexicographic
// argmin -- which equals the reference's tie rule because an alive slot's index is always its
// min member (clustering.cpp:113).
#include "cluster_kernels.cuh"
#include "common.cuh"

namespace sgc {
namespace {

constexpr int PK = 16;   // k chunk

// encoders.cpp:40-48 euclidean_distance for all i<j (thread = PP x PP pairs, k sequential).
// PT = 32 (2 x 2 pairs per thread): at m = 1024 that is 528 tiles instead of the 136 of a
// 64-pair tile, so every SM gets several CTAs; the per-pair arithmetic and order are unchanged.
template <int PT>
__global__ void __launch_bounds__(256)
    pairwise_kernel(double* D, const float* emb, int m, int dim, const int2* tiles, int squared) {
    constexpr int PP = PT / 16;
    __shared__ float As[PK][PT + 1];
    __shared__ float Bs[PK][PT + 1];
    const int2 tile = tiles[blockIdx.x];
    const int i0 = tile.x * PT, j0 = tile.y * PT;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[PP][PP];
#pragma unroll
    for (int a = 0; a < PP; ++a)
#pragma unroll
        for (int b = 0; b < PP; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < dim; k0 += PK) {
        for (int idx = threadIdx.x; idx < PT * PK; idx += 256) {
            int r = idx / PK, kk = idx % PK;
            int gi = i0 + r, gj = j0 + r, gk = k0 + kk;
            As[kk][r] = (gi < m && gk < dim) ? emb[static_cast<size_t>(gi) * dim + gk] : 0.f;
            Bs[kk][r] = (gj < m && gk < dim) ? emb[static_cast<size_t>(gj) * dim + gk] : 0.f;
        }
        __syncthreads();
        const int kn = min(PK, dim - k0);
        for (int kk = 0; kk < kn; ++kk) {
            double a[PP], b[PP];
#pragma unroll
            for (int q = 0; q < PP; ++q) {
                a[q] = static_cast<double>(As[kk][ty + 16 * q]);
                b[q] = static_cast<double>(Bs[kk][tx + 16 * q]);
            }
#pragma unroll
            for (int p = 0; p < PP; ++p)
#pragma unroll
                for (int q = 0; q < PP; ++q) {
                    double v = __dsub_rn(a[p], b[q]);
                    acc[p][q] = __dadd_rn(acc[p][q], __dmul_rn(v, v));
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int q = 0; q < PP; ++q) {
            int i = i0 + ty + 16 * p, j = j0 + tx + 16 * q;
            if (i < m && j < m && i <= j) {
                double v = i == j ? 0.0 : __dsqrt_rn(acc[p][q]);
                if (squared) v = __dmul_rn(v, v);  // clustering.cpp:72-74 squares the sqrt
                D[static_cast<size_t>(i) * m + j] = v;
                D[static_cast<size_t>(j) * m + i] = v;
            }
        }
}

struct Best {
    double v;
    int j;
};
__device__ __forceinline__ bool better(double v, int j, double bv, int bj) {
    return v < bv || (v == bv && j < bj);
}

// merge-loop CTA size (C3, m = 1024: 1024 threads 6.9 ms, 512 7.4-7.8, 256 9.1-9.5 per step)
#ifndef SGC_AGG_THREADS
#define SGC_AGG_THREADS 1024
#endif
constexpr int kAggThreads = SGC_AGG_THREADS;

// One CTA runs the whole merge loop. Per alive row i a cached (value, j) minimum over alive
// j > i is maintained; after a merge only rows whose cached argmin touched keep/kill (or row
// keep itself) are rescanned, every other row gets an O(1) update against the new D[i][keep].
// The per-row state (25 B per point) lives in shared memory up to m ~ 8k points; larger batches
// (`state` != nullptr) keep it in global memory (L1/L2-resident, same code and results).
__global__ void __launch_bounds__(kAggThreads)
    agglomerate_kernel(double* D, int m, int c, int linkage, uint32_t* labels, uint32_t* merge_left,
                       uint32_t* merge_right, double* merge_dist, uint8_t* state) {
    extern __shared__ uint8_t smem_state[];
    uint8_t* sm = state ? state : smem_state;
    double* rv = reinterpret_cast<double*>(sm);                 // [m] row-min value
    int* rj = reinterpret_cast<int*>(rv + m);                   // [m] row-min column
    int* size = rj + m;                                         // [m]
    int* owner = size + m;                                      // [m] point -> slot
    int* rescan = owner + m;                                    // [m] rows to rescan
    unsigned char* alive = reinterpret_cast<unsigned char*>(rescan + m);
    __shared__ double red_v[32];
    __shared__ int red_i[32], red_j[32];
    __shared__ int n_rescan;
    __shared__ int s_keep, s_kill;
    constexpr int kRescanRows = kAggThreads / 32 / 8;  // rows rescanned 8 warps each
    __shared__ double part_v[kAggThreads / 32];
    __shared__ int part_j[kAggThreads / 32];

    const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32, nwarps = blockDim.x / 32;
    for (int i = tid; i < m; i += blockDim.x) {
        alive[i] = 1;
        size[i] = 1;
        owner[i] = i;
    }
    __syncthreads();

    // warp-cooperative min over alive j in [j_lo, j_hi), j != skip, of (D[i][j], j); every lane
    // returns the result. 8 independent L2 loads in flight per lane per round (a rescan was a
    // chain of m/32 dependent round trips); the (value, j) minimum does not depend on the
    // visiting order
    auto scan_range = [&](int i, int j_lo, int j_hi, int skip, double& bv, int& bj) {
        bv = INFINITY;
        bj = 0x7fffffff;
        const double* row = D + static_cast<size_t>(i) * m;
        constexpr int U = 8;
        for (int j0 = j_lo + lane; j0 < j_hi; j0 += 32 * U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + 32 * u;
                v[u] = j < j_hi ? row[j] : INFINITY;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + 32 * u;
                if (j < j_hi && j != skip && alive[j] && better(v[u], j, bv, bj)) {
                    bv = v[u];
                    bj = j;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffff, bv, o);
            int oj = __shfl_xor_sync(0xffffffff, bj, o);
            if (better(ov, oj, bv, bj)) {
                bv = ov;
                bj = oj;
            }
        }
    };
    auto scan_row = [&](int i, int skip) {
        double bv;
        int bj;
        scan_range(i, i + 1, m, skip, bv, bj);
        if (lane == 0) {
            rv[i] = bv;
            rj[i] = bj;
        }
    };
    for (int i = warp; i < m; i += nwarps) scan_row(i, -1);
    __syncthreads();

    const int steps = m - c;
    for (int step = 0; step < steps; ++step) {
        // ---- global argmin over rows, key (value, i, j)
        double bv = INFINITY;
        int bi = 0x7fffffff, bj = 0x7fffffff;
        for (int i = tid; i < m; i += blockDim.x) {
            if (!alive[i] || rj[i] == 0x7fffffff) continue;
            double v = rv[i];
            if (v < bv || (v == bv && (i < bi || (i == bi && rj[i] < bj)))) {
                bv = v;
                bi = i;
                bj = rj[i];
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffff, bv, o);
            int oi = __shfl_xor_sync(0xffffffff, bi, o);
            int oj = __shfl_xor_sync(0xffffffff, bj, o);
            if (ov < bv || (ov == bv && (oi < bi || (oi == bi && oj < bj)))) {
                bv = ov;
                bi = oi;
                bj = oj;
            }
        }
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
            red_j[warp] = bj;
        }
        __syncthreads();
        if (warp == 0) {
            bv = lane < nwarps ? red_v[lane] : INFINITY;
            bi = lane < nwarps ? red_i[lane] : 0x7fffffff;
            bj = lane < nwarps ? red_j[lane] : 0x7fffffff;
            for (int o = 16; o > 0; o >>= 1) {
                double ov = __shfl_xor_sync(0xffffffff, bv, o);
                int oi = __shfl_xor_sync(0xffffffff, bi, o);
                int oj = __shfl_xor_sync(0xffffffff, bj, o);
                if (ov < bv || (ov == bv && (oi < bi || (oi == bi && oj < bj)))) {
                    bv = ov;
                    bi = oi;
                    bj = oj;
                }
            }
        }
        if (tid == 0) {
            s_keep = bi;  // slot index == min member, bi < bj
            s_kill = bj;
            merge_left[step] = bi;
            merge_right[step] = bj;
            merge_dist[step] = linkage == SGC_WARD ? __ddiv_rn(bv, 2.0)
                               : linkage == SGC_CENTROID ? __dsqrt_rn(bv)
                                                         : bv;
            n_rescan = 0;
        }
        __syncthreads();
        const int keep = s_keep, kill = s_kill;
        const double na = size[keep], nb = size[kill];
        double* Dk = D + static_cast<size_t>(keep) * m;
        const double* Dl = D + static_cast<size_t>(kill) * m;
        const double dab = Dk[kill];
        // ---- one pass per k: Lance-Williams update (clustering.cpp:128-148, same operand order,
        // no FMA), owner relabel, and row k's cached minimum against its new D[k][keep] (the
        // value this thread just computed); rows whose cached argmin was keep / kill are rescanned
        for (int k = tid; k < m; k += blockDim.x) {
            if (owner[k] == kill) owner[k] = keep;
            if (!alive[k] || k == kill) continue;
            double v = 0.0;
            if (k != keep) {
                const double dak = Dk[k], dbk = Dl[k];
                const double nk = size[k];
                switch (linkage) {
                    case SGC_SINGLE: v = dak < dbk ? dak : dbk; break;
                    case SGC_COMPLETE: v = dak > dbk ? dak : dbk; break;
                    case SGC_AVERAGE:
                        v = __ddiv_rn(__dadd_rn(__dmul_rn(na, dak), __dmul_rn(nb, dbk)), __dadd_rn(na, nb));
                        break;
                    case SGC_CENTROID: {
                        double s = __dadd_rn(na, nb);
                        double t1 = __ddiv_rn(__dadd_rn(__dmul_rn(na, dak), __dmul_rn(nb, dbk)), s);
                        double t2 = __ddiv_rn(__dmul_rn(__dmul_rn(na, nb), dab), __dmul_rn(s, s));
                        v = __dsub_rn(t1, t2);
                        break;
                    }
                    default: {  // ward
                        double t = __dadd_rn(__dmul_rn(__dadd_rn(na, nk), dak), __dmul_rn(__dadd_rn(nb, nk), dbk));
                        t = __dsub_rn(t, __dmul_rn(nk, dab));
                        v = __ddiv_rn(t, __dadd_rn(__dadd_rn(na, nb), nk));
                    }
                }
                Dk[k] = v;
                D[static_cast<size_t>(k) * m + keep] = v;
            }
            // row-min maintenance of row k (rows > kill never cached keep or kill)
            if (k < kill) {
                bool need = false;
                if (k == keep) need = true;
                else if (rj[k] == kill) need = true;
                else if (k < keep) {
                    if (rj[k] == keep) need = true;
                    else if (better(v, keep, rv[k], rj[k])) {
                        rv[k] = v;
                        rj[k] = keep;
                    }
                }
                if (need) rescan[atomicAdd(&n_rescan, 1)] = k;
            }
        }
        __syncthreads();
        // rescans skip `kill` explicitly: thread 0 retires it concurrently (read again only after
        // the closing barrier)
        if (tid == 0) {
            alive[kill] = 0;
            size[keep] += size[kill];
        }
        const int nr = n_rescan;
        if (nr <= kRescanRows) {
            // few rows (the common case): 8 warps per row, one contiguous j segment each, then one
            // thread per row merges the 8 partial minima -- one L2 round trip instead of m/256
            const int rr = warp / 8, sg = warp % 8;
            if (rr < nr) {
                const int i = rescan[rr];
                const int len = m - i - 1, seg_len = (len + 7) / 8;
                const int lo = i + 1 + sg * seg_len, hi = min(m, lo + seg_len);
                double pv;
                int pj;
                scan_range(i, lo, hi, kill, pv, pj);
                if (lane == 0) {
                    part_v[warp] = pv;
                    part_j[warp] = pj;
                }
            }
            __syncthreads();
            if (tid < nr) {
                double bv2 = INFINITY;
                int bj2 = 0x7fffffff;
                for (int q = 0; q < 8; ++q)
                    if (better(part_v[tid * 8 + q], part_j[tid * 8 + q], bv2, bj2)) {
                        bv2 = part_v[tid * 8 + q];
                        bj2 = part_j[tid * 8 + q];
                    }
                rv[rescan[tid]] = bv2;
                rj[rescan[tid]] = bj2;
            }
        } else {
            for (int r = warp; r < nr; r += nwarps) scan_row(rescan[r], kill);
        }
        __syncthreads();
    }
    // ---- labels by ascending min member (clustering.cpp:162-172): alive slot i == min member
    if (tid == 0) {
        int next = 0;
        for (int i = 0; i < m; ++i)
            if (alive[i]) rescan[i] = next++;
    }
    __syncthreads();
    for (int p = tid; p < m; p += blockDim.x) labels[p] = rescan[owner[p]];
}

}  // namespace

void pairwise_distances(Ctx* c, double* D, const float* emb, int m, int dim, bool squared) {
    constexpr int PT = 32;
    int nt = (m + PT - 1) / PT;
    std::vector<int2> tiles;
    for (int a = 0; a < nt; ++a)
        for (int b = a; b < nt; ++b) tiles.push_back(make_int2(a, b));
    int2* dt = c->buf<int2>("pairwise_tiles", tiles.size());
    copy_in_staged(c, dt, tiles.data(), tiles.size());  // pinned staging: no stream drain
    Ctx::Timed timer(c, "pairwise");
    pairwise_kernel<PT><<<tiles.size(), 256, 0, c->stream>>>(D, emb, m, dim, dt, squared ? 1 : 0);
    SGC_LAUNCH_CHECK(c);
}

size_t agglomerate_smem(int m) { return static_cast<size_t>(m) * (8 + 4 * 4 + 1) + 16; }
// tests: force the global-memory row state at any m (the large-batch path)
bool g_agglomerate_global = false;
void agglomerate_set_global(bool on) { g_agglomerate_global = on; }

void agglomerate(Ctx* c, double* D, int m, int clusters, int linkage, uint32_t* labels,
                 uint32_t* merge_left, uint32_t* merge_right, double* merge_dist) {
    const size_t bytes = agglomerate_smem(m);
    const bool on_chip = bytes <= 200 * 1024 && !g_agglomerate_global;
    uint8_t* state = on_chip ? nullptr : c->buf<uint8_t>("agglomerate_state", bytes);
    const int smem = on_chip ? static_cast<int>(bytes) : 0;
    if (on_chip)
        SGC_CUDA_CHECK(cudaFuncSetAttribute(agglomerate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    Ctx::Timed timer(c, "agglomerate");
    agglomerate_kernel<<<1, kAggThreads, smem, c->stream>>>(D, m, clusters, linkage, labels, merge_left,
                                                            merge_right, merge_dist, state);
    SGC_LAUNCH_CHECK(c);
}

}  // namespace sgc
