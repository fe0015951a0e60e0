// Memory tiers of the B200 build: pinned host arena (the slow tier) and the paged HBM pool
// (the fast tier's physical storage). Bookkeeping of WHICH tables are resident is the
// reference's TieredCache policy (host, tiered_cache.cpp); this file only owns bytes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <deque>
#include <unordered_map>
#include <vector>

#include "kernels.cuh"

namespace tkv {

// Per-table KV image in the .kv layout (table_kv.hpp:45-48) minus the 24-byte header:
// [K: L][T][kv_dim] then [V: L][T][kv_dim], element type f32 (reference files) or bf16.
struct TableImage {
    int table_id = -1, tokens = 0, layers = 0, kv_dim = 0, local_offset = 0;
    DType dtype = DType::f32;
    size_t bytes = 0;
    uint8_t* host = nullptr;        // pinned
    const uint8_t* mapped = nullptr;  // device-visible alias of `host`
};

class Arena {
   public:
    Arena() = default;
    ~Arena();
    Arena(const Arena&) = delete;
    Arena& operator=(const Arena&) = delete;
    // copies `bytes` of payload into pinned memory
    const TableImage& put(int table_id, int tokens, int layers, int kv_dim, int local_offset, DType dt, const void* payload);
    const TableImage* find(int table_id) const;
    size_t total_bytes() const { return total_; }
    size_t size() const { return tables_.size(); }
    int max_table_id() const {
        int m = -1;
        for (const auto& kv : tables_) m = std::max(m, kv.first);
        return m;
    }

   private:
    uint8_t* reserve(size_t bytes);
    struct Chunk {
        uint8_t* host;
        uint8_t* mapped;
        size_t cap, used;
    };
    std::vector<Chunk> chunks_;
    std::unordered_map<int, TableImage> tables_;
    size_t total_ = 0;
};

// Fixed-size pages carved from one HBM slab. Freed pages become reusable only after the
// work queued on the reader stream at free time (the last compute that may read them) is done.
class PagePool {
   public:
    PagePool(size_t page_bytes, int n_pages);
    ~PagePool();
    PagePool(const PagePool&) = delete;
    PagePool& operator=(const PagePool&) = delete;
    uint8_t* base() const { return base_; }
    size_t page_bytes() const { return page_bytes_; }
    int n_pages() const { return n_pages_; }
    int free_pages() const { return int(free_.size()); }
    // blocks (host) on the oldest deferred frees if needed
    std::vector<int32_t> alloc(int n);
    // pages become reusable once all work queued so far on `readers` has completed
    void release(const std::vector<int32_t>& pages, cudaStream_t readers);
    void reclaim();  // non-blocking sweep of completed deferred frees

   private:
    struct Deferred {
        std::vector<int32_t> pages;
        cudaEvent_t ev;
    };
    uint8_t* base_ = nullptr;
    size_t page_bytes_;
    int n_pages_;
    std::vector<int32_t> free_;
    std::deque<Deferred> deferred_;
};

enum class CopyEngine : int { dma = 0, sm = 1 };

// Enqueue the copy of a table image into `pages` on `s`.
void copy_table_to_pages(const TableImage& img, PagePool& pool, const std::vector<int32_t>& pages, CopyEngine eng,
                         int sm_ctas, cudaStream_t s);
// DMA copy of image bytes [off, off + bytes) into their place in `pages` (layer-ordered loads)
void copy_image_range_to_pages(const TableImage& img, PagePool& pool, const std::vector<int32_t>& pages, size_t off,
                               size_t bytes, cudaStream_t s);

}  // namespace tkv
