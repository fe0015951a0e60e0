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
#include <cstring>
#include <chrono>
#include <vector>

#include "common.cuh"
#include "serve.cuh"
#include "tablekv/rerank.hpp"

namespace tkv {

namespace {

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
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

// Compact chain on ONE CTA (no cluster barrier per step): when every distinct table set fits a
// 128-bit window of two consecutive incidence words (a query's tables come from one database), a
// row is (w0, bits of words w0 and w0 + 1, popcount) — 19 bytes — so 10k classes fit one SM's
// shared memory. distance(cur, row) = |cur| + |row| - 2 |cur & row|, the intersection read off the
// overlap of the two windows: the same integer as the XOR popcount, the same (distance, slot) key.
constexpr int kCompactThreads = 1024;
constexpr size_t kCompactRowBytes = 16 + 2 + 1;

__global__ void __launch_bounds__(kCompactThreads, 1)
    rerank_compact_kernel(const ulonglong2* __restrict__ g_bits, const uint16_t* __restrict__ g_w0,
                          const uint8_t* __restrict__ g_pc, int n, int first, int32_t* __restrict__ order) {
    extern __shared__ __align__(16) uint8_t csm[];
    ulonglong2* s_bits = reinterpret_cast<ulonglong2*>(csm);
    uint16_t* s_w0 = reinterpret_cast<uint16_t*>(s_bits + n);
    uint8_t* s_pc = reinterpret_cast<uint8_t*>(s_w0 + n);
    __shared__ unsigned long long red[32];
    __shared__ unsigned long long win_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += kCompactThreads) s_bits[i] = g_bits[i], s_w0[i] = g_w0[i], s_pc[i] = g_pc[i];
    uint32_t used = 0;
    if (first % kCompactThreads == tid) used |= 1u << (first / kCompactThreads);
    if (tid == 0) order[0] = first;
    __syncthreads();
    int cw = s_w0[first], cpc = s_pc[first];
    ulonglong2 cb = s_bits[first];
    for (int step = 1; step < n; ++step) {
        unsigned long long best = ~0ull;
        int j = 0;
        for (int i = tid; i < n; i += kCompactThreads, ++j) {
            if ((used >> j) & 1u) continue;
            const ulonglong2 b = s_bits[i];
            const int w = s_w0[i];
            const uint64_t x0 = w == cw ? cb.x : (w == cw + 1 ? cb.y : 0ull);  // cur's words w, w + 1
            const uint64_t x1 = w + 1 == cw ? cb.x : (w == cw ? cb.y : 0ull);
            const uint32_t d = uint32_t(cpc + s_pc[i] - 2 * (__popcll(x0 & b.x) + __popcll(x1 & b.y)));
            const unsigned long long key = (static_cast<unsigned long long>(d) << 32) | uint32_t(i);
            best = key < best ? key : best;
        }
        best = warp_min(best);
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (warp == 0) {
            best = warp_min(red[lane]);
            if (lane == 0) win_s = best;
        }
        __syncthreads();
        const int wi = int(uint32_t(win_s));
        cw = s_w0[wi], cpc = s_pc[wi], cb = s_bits[wi];
        if (wi % kCompactThreads == tid) used |= 1u << (wi / kCompactThreads);
        if (tid == 0) order[step] = wi;
    }
}

// Window chain on ONE CTA with the rows in REGISTERS: when every distinct table set lies within 64
// consecutive table ids (one database's tables), a row is (first id b0, 64 bits from b0, popcount)
// and thread t keeps rows t + 1024 j for j < R in registers, so the per-step scan reads no shared
// memory at all; the intersection with the current row is a funnel of the two windows. Keys are
// 32-bit: (distance << 14) | slot, so the argmin is the same (distance, lowest slot) order.
constexpr int kWinThreads = 1024;

template <int R>
__global__ void __launch_bounds__(kWinThreads, 1)
    rerank_window_kernel(const uint64_t* __restrict__ g_bits, const uint16_t* __restrict__ g_b0,
                         const uint8_t* __restrict__ g_pc, int n, int first, int32_t* __restrict__ order) {
    extern __shared__ __align__(16) uint8_t wsm[];
    uint64_t* s_bits = reinterpret_cast<uint64_t*>(wsm);
    uint16_t* s_b0 = reinterpret_cast<uint16_t*>(s_bits + n);
    uint8_t* s_pc = reinterpret_cast<uint8_t*>(s_b0 + n);
    __shared__ uint32_t red[32];
    __shared__ uint32_t win_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += kWinThreads) s_bits[i] = g_bits[i], s_b0[i] = g_b0[i], s_pc[i] = g_pc[i];
    uint64_t rb[R];
    int rs[R];  // b0 | popcount << 16
    uint32_t used = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int i = tid + j * kWinThreads;
        rb[j] = i < n ? g_bits[i] : 0ull;
        rs[j] = i < n ? int(g_b0[i]) | (int(g_pc[i]) << 16) : 0;
        if (i >= n || i == first) used |= 1u << j;
    }
    if (tid == 0) order[0] = first;
    __syncthreads();
    uint64_t cb = s_bits[first];
    int cb0 = s_b0[first], cpc = s_pc[first];
    for (int step = 1; step < n; ++step) {
        uint32_t best = ~0u;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int sh = (rs[j] & 0xffff) - cb0;
            const uint64_t x = sh >= 64 || sh <= -64 ? 0ull : (sh >= 0 ? cb >> sh : cb << -sh);  // cur's bits at the row's window
            const uint32_t d = uint32_t(cpc + (rs[j] >> 16) - 2 * __popcll(x & rb[j]));
            const uint32_t key = (used >> j) & 1u ? ~0u : (d << 14) | uint32_t(tid + j * kWinThreads);
            best = min(best, key);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (warp == 0) {
            best = red[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (lane == 0) win_s = best;
        }
        __syncthreads();
        const int wi = int(win_s & 0x3fffu);
        cb = s_bits[wi], cb0 = s_b0[wi], cpc = s_pc[wi];
        if (wi % kWinThreads == tid) used |= 1u << (wi / kWinThreads);
        if (tid == 0) order[step] = wi;
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

std::vector<size_t> rerank_window_device(const std::vector<uint64_t>& bits, const std::vector<uint16_t>& b0,
                                         const std::vector<uint8_t>& pc, size_t first, cudaStream_t s) {
    const size_t m = bits.size();
    static thread_local int dev_cached = -1;
    static thread_local uint8_t* buf = nullptr;
    static thread_local int32_t* ord_d = nullptr;
    static thread_local size_t cap = 0;
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    const size_t bytes = m * 8 + m * 2 + m;
    if (dev_cached != dev || cap < m) {  // (a previous device's buffers are left to it)
        if (dev_cached == dev) cudaFree(buf), cudaFree(ord_d);
        cap = std::max<size_t>(m, 4096);
        TKV_CUDA_CHECK(cudaMalloc(&buf, cap * 11 + 64));
        TKV_CUDA_CHECK(cudaMalloc(&ord_d, cap * 4));
        dev_cached = dev;
    }
    std::vector<uint8_t> host(bytes);
    std::memcpy(host.data(), bits.data(), m * 8);
    std::memcpy(host.data() + m * 8, b0.data(), m * 2);
    std::memcpy(host.data() + m * 10, pc.data(), m);
    TKV_CUDA_CHECK(cudaMemcpyAsync(buf, host.data(), bytes, cudaMemcpyHostToDevice, s));
    const size_t smem = bytes + 16;
    using KernelFn = void (*)(const uint64_t*, const uint16_t*, const uint8_t*, int, int, int32_t*);
    const KernelFn kern = m <= 4 * size_t(kWinThreads) ? rerank_window_kernel<4>
                          : m <= 8 * size_t(kWinThreads) ? rerank_window_kernel<8>
                          : m <= 12 * size_t(kWinThreads) ? rerank_window_kernel<12> : rerank_window_kernel<16>;
    ensure_smem_optin(reinterpret_cast<const void*>(kern), int(smem));
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    static thread_local int ev_dev = -1;
    if (ev_dev != dev) {
        TKV_CUDA_CHECK(cudaEventCreate(&ev[0]));
        TKV_CUDA_CHECK(cudaEventCreate(&ev[1]));
        ev_dev = dev;
    }
    TKV_CUDA_CHECK(cudaEventRecord(ev[0], s));
    kern<<<1, kWinThreads, smem, s>>>(reinterpret_cast<const uint64_t*>(buf), reinterpret_cast<const uint16_t*>(buf + m * 8),
                                      buf + m * 10, int(m), int(first), ord_d);
    TKV_CUDA_CHECK(cudaGetLastError());
    TKV_CUDA_CHECK(cudaEventRecord(ev[1], s));
    std::vector<int32_t> ord(m);
    TKV_CUDA_CHECK(cudaMemcpyAsync(ord.data(), ord_d, m * 4, cudaMemcpyDeviceToHost, s));
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0;
    TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    g_stats.kernel_ms = ms;
    g_stats.n_classes = double(m);
    g_stats.cluster = -1;  // register-window single-CTA chain
    return std::vector<size_t>(ord.begin(), ord.end());
}

std::vector<size_t> rerank_compact_device(const std::vector<ulonglong2>& bits, const std::vector<uint16_t>& w0,
                                          const std::vector<uint8_t>& pc, size_t first, cudaStream_t s) {
    const size_t m = bits.size();
    static thread_local int dev_cached = -1;
    static thread_local uint8_t* buf = nullptr;
    static thread_local int32_t* ord_d = nullptr;
    static thread_local size_t cap = 0;
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    const size_t bytes = m * 16 + m * 2 + m + 64;
    if (dev_cached != dev || cap < m) {  // (a previous device's buffers are left to it)
        if (dev_cached == dev) cudaFree(buf), cudaFree(ord_d);
        cap = std::max<size_t>(m, 4096);
        TKV_CUDA_CHECK(cudaMalloc(&buf, cap * 19 + 64));
        TKV_CUDA_CHECK(cudaMalloc(&ord_d, cap * 4));
        dev_cached = dev;
    }
    std::vector<uint8_t> host(bytes);
    std::memcpy(host.data(), bits.data(), m * 16);
    std::memcpy(host.data() + m * 16, w0.data(), m * 2);
    std::memcpy(host.data() + m * 18, pc.data(), m);
    TKV_CUDA_CHECK(cudaMemcpyAsync(buf, host.data(), bytes, cudaMemcpyHostToDevice, s));
    const size_t smem = m * kCompactRowBytes + 16;
    ensure_smem_optin(reinterpret_cast<const void*>(rerank_compact_kernel), int(smem));
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    static thread_local int ev_dev = -1;
    if (ev_dev != dev) {
        TKV_CUDA_CHECK(cudaEventCreate(&ev[0]));
        TKV_CUDA_CHECK(cudaEventCreate(&ev[1]));
        ev_dev = dev;
    }
    TKV_CUDA_CHECK(cudaEventRecord(ev[0], s));
    rerank_compact_kernel<<<1, kCompactThreads, smem, s>>>(reinterpret_cast<const ulonglong2*>(buf),
                                                            reinterpret_cast<const uint16_t*>(buf + m * 16), buf + m * 18,
                                                            int(m), int(first), ord_d);
    TKV_CUDA_CHECK(cudaGetLastError());
    TKV_CUDA_CHECK(cudaEventRecord(ev[1], s));
    std::vector<int32_t> ord(m);
    TKV_CUDA_CHECK(cudaMemcpyAsync(ord.data(), ord_d, m * 4, cudaMemcpyDeviceToHost, s));
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
    float ms = 0;
    TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    g_stats.kernel_ms = ms;
    g_stats.n_classes = double(m);
    g_stats.cluster = 0;  // compact single-CTA chain
    return std::vector<size_t>(ord.begin(), ord.end());
}

}  // namespace

std::vector<size_t> rerank_chain_device(const uint64_t* rows, size_t m, size_t words, size_t first, cudaStream_t s) {
    if (m == 0) return {};
    // register-window chain when every row's tables span < 64 consecutive ids (and < 16384 rows)
    if (m <= 16 * size_t(kWinThreads) && m * 11 + 16 <= kSmemRowsCap) {
        std::vector<uint64_t> bits(m);
        std::vector<uint16_t> b0(m);
        std::vector<uint8_t> pc(m);
        bool ok = true;
        for (size_t i = 0; i < m && ok; ++i) {
            const uint64_t* r = rows + i * words;
            long lo = -1, hi = -1;
            int p = 0;
            for (size_t w = 0; w < words; ++w)
                if (r[w]) {
                    if (lo < 0) lo = long(w) * 64 + __builtin_ctzll(r[w]);
                    hi = long(w) * 64 + 63 - __builtin_clzll(r[w]);
                    p += __builtin_popcountll(r[w]);
                }
            if (lo < 0) lo = hi = 0;
            ok = hi - lo < 64 && lo < 65536;
            if (!ok) break;
            const size_t w = size_t(lo) >> 6, o = size_t(lo) & 63;
            const uint64_t a = r[w], b = w + 1 < words ? r[w + 1] : 0ull;
            bits[i] = o ? (a >> o) | (b << (64 - o)) : a;
            b0[i] = uint16_t(lo);
            pc[i] = uint8_t(p);
        }
        if (ok) return rerank_window_device(bits, b0, pc, first, s);
    }
    // compact single-CTA chain when every row lives in two consecutive words and the rows fit smem
    if (m * kCompactRowBytes <= kSmemRowsCap && m <= size_t(kCompactThreads) * kMaxRowsPerThread) {
        std::vector<ulonglong2> bits(m);
        std::vector<uint16_t> w0(m);
        std::vector<uint8_t> pc(m);
        bool ok = true;
        for (size_t i = 0; i < m && ok; ++i) {
            const uint64_t* r = rows + i * words;
            size_t lo = words, hi = 0;
            int p = 0;
            for (size_t w = 0; w < words; ++w)
                if (r[w]) lo = std::min(lo, w), hi = w, p += __builtin_popcountll(r[w]);
            if (lo == words) lo = hi = 0;
            ok = hi <= lo + 1 && p < 256;
            w0[i] = uint16_t(lo);
            pc[i] = uint8_t(p);
            bits[i] = make_ulonglong2(r[lo], lo + 1 < words ? r[lo + 1] : 0ull);
        }
        if (ok) return rerank_compact_device(bits, w0, pc, first, s);
    }
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
