// NVLink peer KV fetch: residency directory + reader/owner kernels (see peer.cuh).
#include <cuda/atomic>

#include <algorithm>

#include "common.cuh"
#include "peer.cuh"

namespace tkv {

namespace {

constexpr uint32_t kBlobMagic = 0x544b5650u;  // "PVKT"
// bounded spins: a peer that died mid-copy must not hang this GPU (about a second of polling)
constexpr long kMaxSpin = 1L << 24;

using sys_ref = cuda::atomic_ref<uint32_t, cuda::thread_scope_system>;

__device__ void revoke(DirEntry* e) {
    sys_ref(e->state).store(0u, cuda::memory_order_seq_cst);
    sys_ref readers(e->readers);
    for (long spin = 0; spin < kMaxSpin && readers.load(cuda::memory_order_seq_cst) != 0u; ++spin) __nanosleep(256);
}

__global__ void dir_publish_kernel(DirEntry* e, PageList pages) {
    // every lane writes part of the page list; lane 0 owns the state word
    if (threadIdx.x == 0) revoke(e);
    __syncthreads();
    for (int i = threadIdx.x; i < pages.n; i += blockDim.x) e->page[i] = pages.page[i];
    if (threadIdx.x == 0) e->n_pages = pages.n;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        sys_ref(e->state).store(1u, cuda::memory_order_seq_cst);
    }
}

__global__ void dir_revoke_kernel(DirEntry* e) { revoke(e); }

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Each CTA copies one contiguous chunk of the table image. Source per CTA: the first peer in
// `order` whose directory entry is valid while this CTA is registered as a reader, else the
// mapped host arena. Peer pages are read with volatile-free 16-byte loads (the entry cannot be
// revoked while we are registered, so the bytes are stable).
__global__ void __launch_bounds__(512) peer_fetch_kernel(PeerView v, PeerOrder order, int t, const uint4* __restrict__ host,
                                                         long n_vec, uint8_t* __restrict__ dst_pool, long page_vecs,
                                                         PageList dst, unsigned long long* stats) {
    __shared__ int s_src;
    __shared__ int32_t s_pages[kMaxPagesPerCopy];
    const long per_cta = (n_vec + gridDim.x - 1) / gridDim.x;
    const long lo = blockIdx.x * per_cta, hi = min(n_vec, lo + per_cta);
    if (lo >= hi) return;
    if (threadIdx.x == 0) {
        int src = -1;
        for (int i = 0; i < kMaxPeers && src < 0; ++i) {
            const int p = order.p[i];
            if (p < 0 || p >= v.n || t >= v.dir_entries) continue;
            DirEntry* e = v.dir[p] + t;
            sys_ref readers(e->readers);
            readers.fetch_add(1u, cuda::memory_order_seq_cst);
            if (sys_ref(e->state).load(cuda::memory_order_seq_cst) == 1u)
                src = p;
            else
                readers.fetch_sub(1u, cuda::memory_order_seq_cst);
        }
        s_src = src;
    }
    __syncthreads();
    const int src = s_src;
    if (src >= 0) {
        const DirEntry* e = v.dir[src] + t;
        const long p0 = lo / page_vecs, p1 = (hi - 1) / page_vecs;
        for (long p = p0 + threadIdx.x; p <= p1; p += blockDim.x) s_pages[p] = e->page[p];
        __syncthreads();
        const uint4* pool = reinterpret_cast<const uint4*>(v.pool[src]);
        for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const long pg = i / page_vecs, off = i - pg * page_vecs;
            reinterpret_cast<uint4*>(dst_pool)[long(dst.page[pg]) * page_vecs + off] = ld_stream(pool + long(s_pages[pg]) * page_vecs + off);
        }
    } else {
        for (long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            const long pg = i / page_vecs;
            reinterpret_cast<uint4*>(dst_pool)[long(dst.page[pg]) * page_vecs + (i - pg * page_vecs)] = ld_stream(host + i);
        }
    }
    __syncthreads();  // every load of this CTA has retired (its value was stored)
    if (threadIdx.x == 0) {
        if (src >= 0) sys_ref(v.dir[src][t].readers).fetch_sub(1u, cuda::memory_order_seq_cst);
        atomicAdd(stats + (src >= 0 ? 0 : 1), (unsigned long long)(hi - lo) * 16ull);
    }
}

}  // namespace

PeerMesh::PeerMesh(uint8_t* local_pool, size_t page_bytes, int n_pages, int dir_entries)
    : pool_(local_pool), page_bytes_(page_bytes), n_pages_(n_pages), dir_entries_(dir_entries) {
    TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&dir_), sizeof(DirEntry) * size_t(dir_entries)));
    TKV_CUDA_CHECK(cudaMemset(dir_, 0, sizeof(DirEntry) * size_t(dir_entries)));
    TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&stats_), 2 * sizeof(unsigned long long)));
    TKV_CUDA_CHECK(cudaMemset(stats_, 0, 2 * sizeof(unsigned long long)));
    view_.n = 0;
    view_.dir_entries = dir_entries;
}

PeerMesh::~PeerMesh() {
    cudaDeviceSynchronize();
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    cudaFree(dir_);
    cudaFree(stats_);
}

PeerBlob PeerMesh::blob() const {
    PeerBlob b{};
    b.magic = kBlobMagic;
    TKV_CUDA_CHECK(cudaGetDevice(&b.device));
    b.page_bytes = page_bytes_;
    b.n_pages = n_pages_;
    b.dir_entries = dir_entries_;
    TKV_CUDA_CHECK(cudaIpcGetMemHandle(&b.pool, pool_));
    TKV_CUDA_CHECK(cudaIpcGetMemHandle(&b.dir, dir_));
    return b;
}

void PeerMesh::attach(const std::vector<PeerBlob>& peers) {
    if (view_.n) throw std::logic_error("peers already attached");
    if (int(peers.size()) > kMaxPeers) throw std::invalid_argument("at most 8 peers");
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    for (const PeerBlob& b : peers) {
        if (b.magic != kBlobMagic) throw std::invalid_argument("not a peer blob");
        if (b.page_bytes != page_bytes_) throw std::invalid_argument("peers must use the same page size");
        if (b.device != dev) {
            int can = 0;
            TKV_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, dev, b.device));
            if (!can) throw std::runtime_error("no peer access from device " + std::to_string(dev) + " to " + std::to_string(b.device));
        }
        void *pool = nullptr, *dir = nullptr;
        TKV_CUDA_CHECK(cudaIpcOpenMemHandle(&pool, b.pool, cudaIpcMemLazyEnablePeerAccess));
        opened_.push_back(pool);
        TKV_CUDA_CHECK(cudaIpcOpenMemHandle(&dir, b.dir, cudaIpcMemLazyEnablePeerAccess));
        opened_.push_back(dir);
        view_.pool[view_.n] = static_cast<const uint8_t*>(pool);
        view_.dir[view_.n] = static_cast<DirEntry*>(dir);
        view_.dir_entries = std::min(view_.dir_entries, b.dir_entries);
        ++view_.n;
    }
}

void launch_dir_publish(const PeerMesh& m, int t, const PageList& pages, cudaStream_t s) {
    if (t < 0 || t >= m.dir_entries()) throw std::out_of_range("peer directory: table " + std::to_string(t) + " outside it");
    if (pages.n < 0 || pages.n > kMaxPagesPerCopy) throw std::invalid_argument("peer directory: page list too long");
    dir_publish_kernel<<<1, 128, 0, s>>>(m.local_dir() + t, pages);
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_dir_revoke(const PeerMesh& m, int t, cudaStream_t s) {
    if (t < 0 || t >= m.dir_entries()) throw std::out_of_range("peer directory: table " + std::to_string(t) + " outside it");
    dir_revoke_kernel<<<1, 1, 0, s>>>(m.local_dir() + t);
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_peer_fetch(const PeerView& v, const PeerOrder& order, int t, const uint8_t* host_src, size_t bytes,
                       uint8_t* dst_pool, size_t page_bytes, const PageList& dst_pages, unsigned long long* stats,
                       int n_ctas, cudaStream_t s) {
    if (bytes == 0) return;
    if (bytes % 16 || page_bytes % 16) throw std::invalid_argument("peer fetch: sizes must be multiples of 16 bytes");
    const long n_vec = long(bytes / 16);
    const int blocks = std::max(1, std::min(n_ctas, ceil_div(n_vec, 512 * 4)));
    peer_fetch_kernel<<<blocks, 512, 0, s>>>(v, order, t, reinterpret_cast<const uint4*>(host_src), n_vec, dst_pool,
                                             long(page_bytes / 16), dst_pages, stats);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
