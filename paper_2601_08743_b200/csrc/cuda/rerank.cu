// Query reranking on the GPU: the greedy nearest-neighbour chain of
// proj/src/rerank.cpp:55-94, bit-exact with the host version (rerank_packed, csrc/host/rerank.cpp).
//
// One CTA of 1024 threads runs the whole chain: the live queries' packed incidence rows stay in
// shared memory when they fit (else they are read from L2), a bitmask marks chosen rows, and each
// step is one XOR-popcount distance per remaining row followed by a block argmin on
// (distance, slot) — slot = the row's index among live queries, so ties go to the lowest slot
// exactly like the reference's strict `<` over ascending slots (rerank.cpp:82).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tablekv/rerank.hpp"
#include "tablekv/rng.hpp"

namespace tkv {

namespace {

constexpr int kThreads = 1024;
constexpr int kMaxWords = 64;  // tables up to 4096

// the chosen-row bitmask, in 8-byte units so everything after it stays 8-byte aligned
__host__ __device__ inline int used_u64(int m) { return (m + 63) / 64; }

__global__ void __launch_bounds__(kThreads, 1)
    rerank_chain_kernel(const uint64_t* __restrict__ g_inc, int m, int words, int first, int in_smem, int32_t* __restrict__ order) {
    extern __shared__ uint64_t sm[];
    uint64_t* cur_row = sm;                                       // [words]
    uint32_t* used = reinterpret_cast<uint32_t*>(sm + kMaxWords);  // [ceil(m/32)]
    unsigned long long* red = reinterpret_cast<unsigned long long*>(sm + kMaxWords + used_u64(m));  // [32]
    uint64_t* s_inc = reinterpret_cast<uint64_t*>(red + 32);      // [m][words] when in_smem
    const uint64_t* inc = in_smem ? s_inc : g_inc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 2 * used_u64(m); i += kThreads) used[i] = 0;
    if (in_smem)
        for (long i = tid; i < long(m) * words; i += kThreads) s_inc[i] = g_inc[i];
    __syncthreads();
    int cur = first;
    if (tid == 0) {
        order[0] = first;
        used[first >> 5] |= 1u << (first & 31);
    }
    for (int step = 1; step < m; ++step) {
        if (tid < words) cur_row[tid] = inc[long(cur) * words + tid];
        __syncthreads();
        // key = distance << 32 | slot: the minimum key is the lowest slot among the nearest rows
        unsigned long long best = ~0ull;
        for (int i = tid; i < m; i += kThreads) {
            if (used[i >> 5] & (1u << (i & 31))) continue;
            const uint64_t* row = inc + long(i) * words;
            uint32_t d = 0;
            for (int w = 0; w < words; ++w) d += __popcll(row[w] ^ cur_row[w]);
            const unsigned long long key = (static_cast<unsigned long long>(d) << 32) | uint32_t(i);
            best = key < best ? key : best;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
            best = other < best ? other : best;
        }
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (warp == 0) {
            best = red[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
                best = other < best ? other : best;
            }
            if (lane == 0) {
                const int pick = int(uint32_t(best));
                order[step] = pick;
                used[pick >> 5] |= 1u << (pick & 31);
                red[0] = best;
            }
        }
        __syncthreads();
        cur = int(uint32_t(red[0]));
    }
}

}  // namespace

std::vector<size_t> rerank_device(const uint64_t* inc, size_t n, size_t words, uint64_t seed, tablekv::AnchorMode mode,
                                  cudaStream_t s) {
    if (n == 0) throw tablekv::Error(tablekv::Errc::empty_batch, "rerank needs at least one query");
    if (words > size_t(kMaxWords)) throw std::invalid_argument("device rerank supports up to 4096 tables");
    std::vector<size_t> live, empty;
    for (size_t i = 0; i < n; ++i) {
        bool any = false;
        for (size_t w = 0; w < words && !any; ++w) any = inc[i * words + w] != 0;
        (any ? live : empty).push_back(i);
    }
    std::vector<size_t> out;
    out.reserve(n);
    if (!live.empty()) {
        const size_t m = live.size();
        size_t first = 0;
        if (mode == tablekv::AnchorMode::seeded) {  // rerank.cpp:68-71
            tablekv::SeededRng r(seed);
            first = size_t(r.next_below(m));
        }
        std::vector<uint64_t> packed(m * words);
        for (size_t k = 0; k < m; ++k) std::copy(inc + live[k] * words, inc + (live[k] + 1) * words, packed.begin() + long(k * words));
        // per-thread device scratch, grown on demand and kept (no allocator traffic per batch)
        struct Scratch {
            int device = -1;
            uint64_t* inc = nullptr;
            int32_t* order = nullptr;
            size_t cap = 0;
        };
        static thread_local Scratch sc;
        int dev = 0;
        TKV_CUDA_CHECK(cudaGetDevice(&dev));
        if (sc.device != dev || sc.cap < m * (words + 1)) {
            if (sc.device == dev) {
                cudaFree(sc.inc);
                cudaFree(sc.order);
            }
            sc.device = dev;
            sc.cap = std::max<size_t>(m * (words + 1), 1 << 16);
            TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&sc.inc), sc.cap * 8));
            TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&sc.order), sc.cap * 4));
            TKV_CUDA_CHECK(cudaFuncSetAttribute(rerank_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 4096));
        }
        TKV_CUDA_CHECK(cudaMemcpyAsync(sc.inc, packed.data(), packed.size() * 8, cudaMemcpyHostToDevice, s));
        const size_t base = (kMaxWords + size_t(used_u64(int(m))) + 32) * 8;
        const size_t full = base + packed.size() * 8;
        const bool in_smem = full <= 200 * 1024;
        const size_t smem = in_smem ? full : base;
        if (smem > 200 * 1024 + 4096) throw std::invalid_argument("device rerank: batch too large for one CTA's bitmask");
        rerank_chain_kernel<<<1, kThreads, smem, s>>>(sc.inc, int(m), int(words), int(first), int(in_smem), sc.order);
        TKV_CUDA_CHECK(cudaGetLastError());
        std::vector<int32_t> ord(m);
        TKV_CUDA_CHECK(cudaMemcpyAsync(ord.data(), sc.order, m * 4, cudaMemcpyDeviceToHost, s));
        TKV_CUDA_CHECK(cudaStreamSynchronize(s));
        for (int32_t k : ord) out.push_back(live[size_t(k)]);
    }
    out.insert(out.end(), empty.begin(), empty.end());  // rerank.cpp:92
    return out;
}

}  // namespace tkv
