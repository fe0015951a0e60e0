// Pinned host arena + paged HBM pool (see runtime.cuh).
#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>

#include "common.cuh"
#include "runtime.cuh"

namespace tkv {

void ensure_smem_optin(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;  // (device, kernel) -> opted-in bytes
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int& have = done[{dev, func}];
    if (bytes <= have) return;
    TKV_CUDA_CHECK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
}

int device_sm_count() {
    static std::mutex mu;
    static std::map<int, int> n;
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int& c = n[dev];
    if (!c) TKV_CUDA_CHECK(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev));
    return c;
}

// ------------------------------------------------------------------ Arena
Arena::~Arena() {
    for (auto& c : chunks_) cudaFreeHost(c.host);
}

uint8_t* Arena::reserve(size_t bytes) {
    const size_t need = (bytes + 255) & ~size_t(255);
    if (chunks_.empty() || chunks_.back().cap - chunks_.back().used < need) {
        const size_t cap = std::max<size_t>(need, size_t(256) << 20);
        Chunk c{};
        TKV_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c.host), cap, cudaHostAllocMapped | cudaHostAllocPortable));
        TKV_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.mapped), c.host, 0));
        c.cap = cap;
        c.used = 0;
        chunks_.push_back(c);
    }
    Chunk& c = chunks_.back();
    uint8_t* p = c.host + c.used;
    c.used += need;
    return p;
}

const TableImage& Arena::put(int table_id, int tokens, int layers, int kv_dim, int local_offset, DType dt,
                             const void* payload) {
    if (tables_.count(table_id)) throw std::invalid_argument("arena already holds table " + std::to_string(table_id));
    TableImage img;
    img.table_id = table_id;
    img.tokens = tokens;
    img.layers = layers;
    img.kv_dim = kv_dim;
    img.local_offset = local_offset;
    img.dtype = dt;
    img.bytes = size_t(2) * layers * tokens * kv_dim * dtype_size(dt);
    img.host = reserve(img.bytes);
    const Chunk& c = chunks_.back();
    img.mapped = c.mapped + (img.host - c.host);
    if (payload) std::memcpy(img.host, payload, img.bytes);
    total_ += img.bytes;
    return tables_.emplace(table_id, img).first->second;
}

const TableImage* Arena::find(int table_id) const {
    auto it = tables_.find(table_id);
    return it == tables_.end() ? nullptr : &it->second;
}

// ------------------------------------------------------------------ PagePool
PagePool::PagePool(size_t page_bytes, int n_pages) : page_bytes_(page_bytes), n_pages_(n_pages) {
    if (page_bytes % 256) throw std::invalid_argument("page size must be a multiple of 256 bytes");
    TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&base_), page_bytes * size_t(n_pages)));
    free_.reserve(n_pages);
    for (int i = n_pages - 1; i >= 0; --i) free_.push_back(i);
}

PagePool::~PagePool() {
    cudaDeviceSynchronize();
    for (auto& d : deferred_) cudaEventDestroy(d.ev);
    cudaFree(base_);
}

void PagePool::reclaim() {
    while (!deferred_.empty() && cudaEventQuery(deferred_.front().ev) == cudaSuccess) {
        // pushed highest id first: alloc() pops from the back, so a freed run comes back out in
        // ascending order and a table's copy stays one contiguous run (LIFO order would hand out
        // every other batch descending, one copy per page)
        std::vector<int32_t>& pg = deferred_.front().pages;
        std::sort(pg.begin(), pg.end(), std::greater<int32_t>());
        for (int32_t p : pg) free_.push_back(p);
        cudaEventDestroy(deferred_.front().ev);
        deferred_.pop_front();
    }
}

std::vector<int32_t> PagePool::alloc(int n) {
    if (n > n_pages_) throw std::runtime_error("table larger than the whole page pool");
    reclaim();
    while (int(free_.size()) < n) {
        if (deferred_.empty()) throw std::runtime_error("page pool exhausted (pool too small for the resident set)");
        TKV_CUDA_CHECK(cudaEventSynchronize(deferred_.front().ev));
        reclaim();
    }
    std::vector<int32_t> out(free_.rbegin(), free_.rbegin() + n);  // lowest ids first => adjacent runs
    free_.resize(free_.size() - n);
    return out;
}

void PagePool::release(const std::vector<int32_t>& pages, cudaStream_t readers) {
    if (pages.empty()) return;
    cudaEvent_t ev;
    TKV_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TKV_CUDA_CHECK(cudaEventRecord(ev, readers));  // everything already queued on `readers` may read them
    deferred_.push_back({pages, ev});
}

// ------------------------------------------------------------------ copies
void copy_table_to_pages(const TableImage& img, PagePool& pool, const std::vector<int32_t>& pages, CopyEngine eng,
                         int sm_ctas, cudaStream_t s) {
    const size_t P = pool.page_bytes();
    if (pages.size() * P < img.bytes) throw std::logic_error("not enough pages for table image");
    if (eng == CopyEngine::sm && img.bytes % 16 == 0 && int(pages.size()) <= kMaxPagesPerCopy) {
        PageList pl;
        pl.n = int(pages.size());
        for (size_t i = 0; i < pages.size(); ++i) pl.page[i] = pages[i];
        launch_h2d_pages(img.mapped, img.bytes, pool.base(), P, pl, sm_ctas, s);
        return;
    }
    // DMA: one copy-engine transfer per page, merged across physically adjacent pages
    size_t off = 0;
    size_t i = 0;
    while (off < img.bytes) {
        size_t run = 1;
        while (i + run < pages.size() && pages[i + run] == pages[i] + int32_t(run) && off + run * P < img.bytes) ++run;
        const size_t n = std::min(run * P, img.bytes - off);
        TKV_CUDA_CHECK(cudaMemcpyAsync(pool.base() + size_t(pages[i]) * P, img.host + off, n, cudaMemcpyHostToDevice, s));
        off += n;
        i += run;
    }
}

void copy_image_range_to_pages(const TableImage& img, PagePool& pool, const std::vector<int32_t>& pages, size_t off,
                               size_t bytes, cudaStream_t s) {
    const size_t P = pool.page_bytes();
    if (off + bytes > img.bytes || pages.size() * P < img.bytes) throw std::logic_error("image range outside the table pages");
    const size_t end = off + bytes;
    while (off < end) {  // one DMA transfer per run of physically adjacent pages
        size_t i = off / P;
        size_t stop = std::min(end, (i + 1) * P);
        while (stop < end && i + 1 < pages.size() && pages[i + 1] == pages[i] + 1) ++i, stop = std::min(end, (i + 1) * P);
        TKV_CUDA_CHECK(cudaMemcpyAsync(pool.base() + size_t(pages[off / P]) * P + off % P, img.host + off, stop - off,
                                       cudaMemcpyHostToDevice, s));
        off = stop;
    }
}

}  // namespace tkv
