// Slow tier -> HBM pool page copies (the SlowTier::load of the B200 build,
// proj/include/tablekv/tiered_cache.hpp:24-29, proj/src/tiered_cache.cpp:49-59).
//
// The pinned host arena holds each table's image contiguously; the pool holds it in
// fixed-size pages that need not be contiguous. The SM-driven path reads the arena through
// its mapped device pointer with 16-byte vector loads, UNROLL requests in flight per thread,
// and stores 16 bytes per lane into the destination page: every warp access is a fully
// coalesced 512-byte run (pages are multiples of 16 bytes, so no vector straddles a page).
#include "common.cuh"
#include "kernels.cuh"

namespace tkv {

namespace {

constexpr int kUnroll = 8;

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__global__ void h2d_pages_kernel(const uint4* __restrict__ src, long n_vec, uint8_t* __restrict__ pool,
                                 long page_vecs, PageList pages) {
    const long stride = long(gridDim.x) * blockDim.x;
    long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n_vec; i += kUnroll * stride) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const long j = i + u * stride;
            const long pg = j / page_vecs;
            reinterpret_cast<uint4*>(pool)[long(pages.page[pg]) * page_vecs + (j - pg * page_vecs)] = v[u];
        }
    }
    for (; i < n_vec; i += stride) {
        const long pg = i / page_vecs;
        reinterpret_cast<uint4*>(pool)[long(pages.page[pg]) * page_vecs + (i - pg * page_vecs)] = ld_stream(src + i);
    }
}

}  // namespace

void launch_h2d_pages(const void* src_mapped, size_t bytes, uint8_t* pool, size_t page_bytes, const PageList& pages,
                      int n_ctas, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes % 16 || page_bytes % 16) throw std::invalid_argument("h2d_pages: sizes must be multiples of 16 bytes");
    const long n_vec = long(bytes / 16);
    const int threads = 512;
    const int blocks = std::max(1, std::min(n_ctas, ceil_div(n_vec, threads)));
    h2d_pages_kernel<<<blocks, threads, 0, s>>>(static_cast<const uint4*>(src_mapped), n_vec, pool,
                                                long(page_bytes / 16), pages);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
