// Query reranking on the GPU: the greedy nearest-neighbour chain of
// proj/src/rerank.cpp:55-94, bit-exact with the host version (rerank_packed, csrc/host/rerank.cpp).
//
// The host first reduces the batch to distinct table sets (rerank_classes: identical sets are
// consumed back to back, so the chain over class representatives expanded class by class is the
// reference chain). The class chain runs on ONE thread-block cluster of C CTAs (C = 1..16): each
// CTA keeps its slice of the class rows in shared memory; per step every CTA takes the argmin of
// (distance, slot) over its unused rows (slot = the class index, so ties go to the lowest slot
// exactly like the reference's strict `<` over ascending slots, rerank.cpp:82), and pushes its
// candidate's key AND row into every CTA's exchange slot through distributed shared memory; one
// cluster barrier later every thread reduces the C candidates itself and already holds the
// winner's row for the next step. One __syncthreads and one cluster barrier per step.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "common.cuh"
#include "serve.cuh"
#include "tablekv/rerank.hpp"

namespace tkv {

namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxWords = 64;    // tables up to 4096
constexpr int kMaxCluster = 16;  // non-portable cluster size (opted in below)
constexpr int kMaxRowsPerThread = 32;  // used-bits live in one register per thread
constexpr size_t kSmemRowsCap = 200 * 1024;

struct Xch {  // one CTA's candidate for one step
    unsigned long long key;
    uint64_t row[kMaxWords];
};
constexpr size_t kFixedSmem = sizeof(Xch) * 2 * kMaxCluster + 32 * 8 + kMaxWords * 8;

__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x < v ? x : v;
    }
    return v;
}

// W = compile-time bound on the words per row (cur is held in registers); rows in shared memory
// are word-major ([word][row]) so a warp's 32 lanes read 32 consecutive rows' word w at once
// (conflict-free, 256 bytes per request); rows left in global memory stay row-major.
template <int W>
__global__ void __launch_bounds__(kThreads, 1)
    rerank_cluster_kernel(const uint64_t* __restrict__ g_inc, int n, int words, int first, int per, int rows_in_smem,
                          int32_t* __restrict__ order) {
    cg::cluster_group cl = cg::this_cluster();
    const int rank = int(cl.block_rank()), C = int(cl.num_blocks());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) uint64_t sm[];
    Xch* xch = reinterpret_cast<Xch*>(sm);                                                 // [2][kMaxCluster]
    unsigned long long* red = reinterpret_cast<unsigned long long*>(xch + 2 * kMaxCluster);  // [32]
    uint64_t* cur0 = reinterpret_cast<uint64_t*>(red + 32);                                 // [kMaxWords]
    uint64_t* s_rows = cur0 + kMaxWords;                                                    // [words][per]
    const int r0 = rank * per;
    const int n_loc = max(0, min(n - r0, per));
    if (rows_in_smem)
        for (long i = tid; i < long(n_loc) * words; i += kThreads) {
            const long r = i / words, w = i % words;
            s_rows[w * per + r] = g_inc[long(r0) * words + i];
        }
    if (tid < words) cur0[tid] = g_inc[long(first) * words + tid];
    // used bits of this thread's rows: bit j <-> local row tid + j * kThreads
    uint32_t used = 0;
    if (first >= r0 && first < r0 + n_loc && (first - r0) % kThreads == tid) used |= 1u << ((first - r0) / kThreads);
    if (rank == 0 && tid == 0) order[0] = first;
    cl.sync();  // every CTA's exchange area and rows exist before the first remote store
    const uint64_t* cur = cur0;
    for (int step = 1; step < n; ++step) {
        uint64_t cw[W];
#pragma unroll
        for (int w = 0; w < W; ++w) cw[w] = w < words ? cur[w] : 0ull;
        unsigned long long best = ~0ull;
        int j = 0;
        for (int i = tid; i < n_loc; i += kThreads, ++j) {
            if ((used >> j) & 1u) continue;
            uint32_t d = 0;
            if (rows_in_smem) {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    if (w < words) d += __popcll(s_rows[long(w) * per + i] ^ cw[w]);
            } else {
                const uint64_t* row = g_inc + long(r0 + i) * words;
#pragma unroll
                for (int w = 0; w < W; ++w)
                    if (w < words) d += __popcll(__ldg(row + w) ^ cw[w]);
            }
            const unsigned long long key = (static_cast<unsigned long long>(d) << 32) | uint32_t(r0 + i);
            best = key < best ? key : best;
        }
        best = warp_min(best);
        if (lane == 0) red[warp] = best;
        __syncthreads();
        const int par = step & 1;
        if (warp == 0) {
            best = warp_min(lane < kWarps ? red[lane] : ~0ull);
            const bool has = best != ~0ull;
            const long li = has ? long(uint32_t(best)) - r0 : 0;
            // this CTA's candidate -> slot [par][rank] of every CTA: lane w carries row word w
            uint64_t rw = 0;
            if (has && lane < words)
                rw = rows_in_smem ? s_rows[long(lane) * per + li] : g_inc[(r0 + li) * long(words) + lane];
            for (int dst = 0; dst < C; ++dst) {
                Xch* x = cl.map_shared_rank(&xch[par * kMaxCluster + rank], dst);
                if (lane == 0) x->key = best;
                if (has)
                    for (int w = lane; w < words; w += 32)
                        x->row[w] = w == lane ? rw : (rows_in_smem ? s_rows[long(w) * per + li] : g_inc[(r0 + li) * long(words) + w]);
            }
        }
        cl.sync();
        unsigned long long win = ~0ull;
        int wr = 0;
        for (int r = 0; r < C; ++r) {
            const unsigned long long k = xch[par * kMaxCluster + r].key;
            if (k < win) win = k, wr = r;
        }
        cur = xch[par * kMaxCluster + wr].row;  // read during the next step; rewritten two steps later
        const int ls = int(uint32_t(win)) - r0;
        if (ls >= 0 && ls < n_loc && ls % kThreads == tid) used |= 1u << (ls / kThreads);
        if (rank == 0 && tid == 0) order[step] = int32_t(uint32_t(win));
    }
}

thread_local RerankStats g_stats;

// per-thread device scratch, grown on demand and kept (no allocator traffic per batch)
struct Scratch {
    int device = -1;
    uint64_t* inc = nullptr;
    int32_t* order = nullptr;
    size_t cap_inc = 0, cap_order = 0;
};

}  // namespace

std::vector<size_t> rerank_chain_device(const uint64_t* rows, size_t m, size_t words, size_t first, cudaStream_t s) {
    if (m == 0) return {};
    if (words > size_t(kMaxWords)) throw std::invalid_argument("device rerank supports up to 4096 tables");
    if (m > size_t(kMaxCluster) * kThreads * kMaxRowsPerThread) throw std::invalid_argument("device rerank: batch too large");
    // smallest cluster whose slices fit shared memory with at most 4 rows per thread; beyond 16
    // CTAs the rows stay in global memory (L2) instead
    int C = 1;
    auto fits = [&](int c) {
        const size_t per = (m + size_t(c) - 1) / size_t(c);
        return per * words * 8 <= kSmemRowsCap && per <= size_t(4 * kThreads);
    };
    while (C < kMaxCluster && !fits(C)) C *= 2;
    const size_t per = (m + size_t(C) - 1) / size_t(C);
    const bool in_smem = per * words * 8 <= kSmemRowsCap;
    if (per > size_t(kThreads) * kMaxRowsPerThread) throw std::invalid_argument("device rerank: batch too large");
    const size_t smem = kFixedSmem + (in_smem ? per * words * 8 : 0);

    static thread_local Scratch sc;
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    if (sc.device != dev) sc = Scratch{}, sc.device = dev;  // (a previous device's buffers are left to it)
    if (sc.cap_inc < m * words) {
        cudaFree(sc.inc);
        sc.cap_inc = std::max<size_t>(m * words, 1 << 16);
        TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&sc.inc), sc.cap_inc * 8));
    }
    if (sc.cap_order < m) {
        cudaFree(sc.order);
        sc.cap_order = std::max<size_t>(m, 1 << 14);
        TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&sc.order), sc.cap_order * 4));
    }
    TKV_CUDA_CHECK(cudaMemcpyAsync(sc.inc, rows, m * words * 8, cudaMemcpyHostToDevice, s));
    using KernelFn = void (*)(const uint64_t*, int, int, int, int, int, int32_t*);
    const KernelFn kern = words <= 4 ? rerank_cluster_kernel<4> : words <= 8 ? rerank_cluster_kernel<8>
                          : words <= 16 ? rerank_cluster_kernel<16> : rerank_cluster_kernel<kMaxWords>;
    ensure_smem_optin(reinterpret_cast<const void*>(kern), int(smem));
    static thread_local std::vector<const void*> nonportable;  // (kernel, device) pairs opted in
    const void* key = reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(kern) ^ uintptr_t(dev));
    if (std::find(nonportable.begin(), nonportable.end(), key) == nonportable.end()) {
        TKV_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        nonportable.push_back(key);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    static thread_local int ev_dev = -1;
    if (ev_dev != dev) {
        TKV_CUDA_CHECK(cudaEventCreate(&ev[0]));
        TKV_CUDA_CHECK(cudaEventCreate(&ev[1]));
        ev_dev = dev;
    }
    TKV_CUDA_CHECK(cudaEventRecord(ev[0], s));
    TKV_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, static_cast<const uint64_t*>(sc.inc), int(m), int(words), int(first),
                                      int(per), int(in_smem), sc.order));
    TKV_CUDA_CHECK(cudaEventRecord(ev[1], s));
    std::vector<int32_t> ord(m);
    TKV_CUDA_CHECK(cudaMemcpyAsync(ord.data(), sc.order, m * 4, cudaMemcpyDeviceToHost, s));
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0;
    TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    g_stats.kernel_ms = ms;
    g_stats.n_classes = double(m);
    g_stats.cluster = C;
    return std::vector<size_t>(ord.begin(), ord.end());
}

std::vector<size_t> rerank_device(const uint64_t* inc, size_t n, size_t words, uint64_t seed, tablekv::AnchorMode mode,
                                  cudaStream_t s) {
    if (words > size_t(kMaxWords)) throw std::invalid_argument("device rerank supports up to 4096 tables");
    const auto t0 = std::chrono::steady_clock::now();
    g_stats = RerankStats{};
    const tablekv::RerankClasses rc = tablekv::rerank_classes(inc, n, words, seed, mode);
    g_stats.classes_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rc.n_classes() == 0) return rc.empty;
    auto out = tablekv::expand_class_chain(rc, rerank_chain_device(rc.rows.data(), rc.n_classes(), words, rc.anchor_class, s));
    g_stats.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

RerankStats last_rerank_stats() { return g_stats;
}

}  // namespace tkv
