// NVLink peer KV fetch: a table already resident in a peer GPU's HBM pool is
// copied from that pool over NVLink instead of from the pinned host arena over PCIe.
//
// Each rank's pool owns a device-resident residency directory, one entry per table id, exported
// with its pool slab through CUDA IPC. The owner publishes an entry (page list, then state=valid)
// once the table's bytes have landed and revokes it (state=invalid, then waits for in-flight
// readers to drain) before those pages can be recycled. A reader CTA registers itself in the
// entry's reader count, then checks the state (seq_cst on both sides: either the owner sees the
// reader and waits, or the reader sees the revoke and falls back to the host arena). Bytes are
// identical from either source, so every CTA chooses its source independently and no reader ever
// waits on anything: the protocol cannot deadlock and changes only the SOURCE of a miss, never the
// reference's per-GPU hit/miss/evict trace.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "kernels.cuh"

namespace tkv {

constexpr int kMaxPeers = 8;

struct DirEntry {
    uint32_t state;    // 0 invalid, 1 valid
    uint32_t readers;  // reader CTAs currently copying from this entry's pages
    int32_t n_pages;
    int32_t pad;
    int32_t page[kMaxPagesPerCopy];
};

// Opaque blob one rank hands to its peers (cudaIpcMemHandle of the pool slab and the directory).
struct PeerBlob {
    uint32_t magic;
    int32_t device;
    uint64_t page_bytes;
    int32_t n_pages;
    int32_t dir_entries;
    cudaIpcMemHandle_t pool;
    cudaIpcMemHandle_t dir;
};

struct PeerOrder {  // peer slots to try, in order; -1 = none
    int8_t p[kMaxPeers];
};

struct PeerView {  // kernel argument: the attached peers
    const uint8_t* pool[kMaxPeers];
    DirEntry* dir[kMaxPeers];
    int32_t n;
    int32_t dir_entries;
};

class PeerMesh {
   public:
    PeerMesh(uint8_t* local_pool, size_t page_bytes, int n_pages, int dir_entries);
    ~PeerMesh();
    PeerMesh(const PeerMesh&) = delete;
    PeerMesh& operator=(const PeerMesh&) = delete;
    PeerBlob blob() const;
    // peers[i] = blob of peer slot i (the local rank's own blob is skipped by the caller)
    void attach(const std::vector<PeerBlob>& peers);
    int n_peers() const { return view_.n; }
    int dir_entries() const { return dir_entries_; }
    DirEntry* local_dir() const { return dir_; }
    const PeerView& view() const { return view_; }
    unsigned long long* stats() const { return stats_; }  // [0] bytes from peers, [1] bytes from host fallback

   private:
    uint8_t* pool_;
    size_t page_bytes_;
    int n_pages_, dir_entries_;
    DirEntry* dir_ = nullptr;
    unsigned long long* stats_ = nullptr;
    PeerView view_{};
    std::vector<void*> opened_;
};

// owner side (stream-ordered): publish table `t` at `pages`; revoke `t`
// (bounds-checked against the mesh's directory size and kMaxPagesPerCopy)
void launch_dir_publish(const PeerMesh& m, int t, const PageList& pages, cudaStream_t s);
void launch_dir_revoke(const PeerMesh& m, int t, cudaStream_t s);
// reader side: copy table `t` (`bytes`) into local `dst_pages`, each CTA from the first peer in
// `order` holding a valid entry, else from the mapped host arena image `host_src`
void launch_peer_fetch(const PeerView& v, const PeerOrder& order, int t, const uint8_t* host_src, size_t bytes,
                       uint8_t* dst_pool, size_t page_bytes, const PageList& dst_pages, unsigned long long* stats,
                       int n_ctas, cudaStream_t s);

}  // namespace tkv
