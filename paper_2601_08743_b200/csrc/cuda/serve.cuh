// GPU executor of the online path: rerank -> schedule -> canonical cache trace (host, exact
// reference decisions) -> per window: H2D/peer page copies for every miss/prefetch on copy
// streams, prefix gather+RoPE and the batched suffix prefill + first-token head on the compute
// stream, events for TTFT. proj/src/pipeline.cpp:310-342 (run_batch) is the reference caller.
#pragma once

#include <array>

#include <cuda_runtime.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "model.cuh"
#include "peer.cuh"
#include "runtime.cuh"
#include "tablekv/pipeline.hpp"

namespace tkv {

struct ServeQuery {
    std::string id;
    std::vector<int> tables;       // matched tables in assembly (PK-FK topological) order
    std::vector<int32_t> suffix;   // remainder tokens (engine.cpp:133-151)
};

struct ServeOptions {
    tablekv::RunOptions run;
    tablekv::CostModel cost;
    CopyEngine engine = CopyEngine::dma;
    int sm_copy_ctas = 16;
    bool keep_logits = false;      // copy first-token logits back (parity tests)
    bool time_kernels = false;     // per-GEMM events (bench roofline)
    bool peer_fetch = false;       // misses predicted resident on an attached peer come over NVLink
    int peer_ctas = 64;            // CTAs per peer-fetch copy
};

// A peer's upcoming batch, as it will serve it (its queries' tables; same run options). Every
// rank's trace is deterministic, so replaying it here predicts in which of the peer's windows a
// table is resident — the host-side residency directory that routes a miss to the peer.
struct PeerPlan {
    std::vector<std::vector<int>> tables;
    std::vector<int> suffix_len;
};

struct TraceEvent {  // one cache decision that moved bytes (or a boundary hit)
    int window, kind;   // kind 0 boundary, 1 prefetch, 2 emergency
    long query;         // plan-order query index for emergency records, else -1
    int table, evicted;
    bool miss;
    size_t bytes;       // KV bytes copied into HBM for this record
};

struct ServeResult {
    std::vector<size_t> order;             // served order (indices into the input)
    std::vector<double> ttft_ms;           // per served query: batch submission -> first-token logits
    std::vector<int32_t> argmax;           // per served query: first generated token
    std::vector<float> logits;             // [served][vocab_padded] when keep_logits
    std::vector<int> window_of;            // per served query
    std::vector<double> window_end_ms;
    std::vector<std::array<double, 4>> window_timeline;  // demand copy start / end, compute ready, end
    std::vector<TraceEvent> trace;
    tablekv::CacheCounters counters;
    size_t h2d_bytes = 0, meta_bytes = 0;
    size_t h2d_demand_bytes = 0;           // boundary + emergency loads (demand copy stream)
    size_t peer_routed_bytes = 0;          // misses routed to the NVLink peer-fetch path
    unsigned long long peer_bytes = 0, peer_fallback_bytes = 0;  // ... served by a peer / by the host arena
    double copy_busy_ms = 0;               // sum of per-window copy spans (both copy streams)
    double copy_demand_ms = 0;             // demand stream only (its copies run back to back)
    double makespan_ms = 0, host_ms = 0;
    double wall_ms = 0;                    // serve() entry to return on the host clock
    long launches = 0;
    double gemm_ms = 0, gemm_flops = 0;    // time_kernels only
    double gather_ms = 0, gather_bytes = 0;
    double attn_ms = 0;
    long total_ctx_tokens = 0, total_suffix_tokens = 0;
};

// host half of the executor: rerank -> schedule -> canonical trace over a metadata-only tier
struct BatchTrace {
    std::vector<size_t> order;
    tablekv::BatchPlan plan;
    tablekv::Trace trace;
    tablekv::CacheCounters counters;
    bool managed = true;
};
BatchTrace plan_batch(const std::vector<std::vector<int>>& tables, const std::vector<int>& suffix_len,
                      const ServeOptions& opts, const Arena& arena, cudaStream_t s = nullptr);
// rerank_packed (csrc/host/rerank.cpp) on the GPU: identical permutation, one CTA runs the chain
std::vector<size_t> rerank_device(const uint64_t* inc, size_t n, size_t words, uint64_t seed, tablekv::AnchorMode mode,
                                  cudaStream_t s);
// the calling thread's last rerank_device: host class reduction, chain kernel (CUDA events), whole call
struct RerankStats {
    double classes_ms = 0, kernel_ms = 0, total_ms = 0, n_classes = 0;
    int cluster = 0;
};
RerankStats last_rerank_stats();
constexpr size_t kDeviceRerankMin = 512;  // batches at least this large rerank on the GPU
// table -> [first, last] windows during which the executor keeps it published for peers
std::unordered_map<int, std::vector<std::pair<int, int>>> residency_intervals(const BatchTrace& bt);

class Server {
   public:
    Server(Model& model, Arena& arena, PagePool& pool);
    ~Server();
    // table_tokens: token ids per table id (needed only by the no-cache baseline)
    void set_table_tokens(std::vector<std::vector<int32_t>> tt, std::vector<int> group_of);
    ServeResult serve(const std::vector<ServeQuery>& queries, const ServeOptions& opts);
    // baseline: full block-masked prefill of [tables ; suffix] per query, no cache, same windows
    ServeResult serve_nocache(const std::vector<ServeQuery>& queries, const ServeOptions& opts);
    cudaStream_t compute_stream() const { return cs_; }
    // NVLink peer fetch: the mesh (owned by the store) and the peers' upcoming batches
    void set_mesh(PeerMesh* m) { mesh_ = m; }
    void set_peer_plan(int slot, PeerPlan plan);

   private:
    void ensure_ctx(size_t bytes);
    void ensure_out(size_t n_argmax, size_t n_logits);
    Model& model_;
    Arena& arena_;
    PagePool& pool_;
    cudaStream_t cs_ = nullptr, ds_ = nullptr, ps_ = nullptr;  // compute, demand copies, prefetch copies
    cudaStream_t xs_ = nullptr;                                 // peer (NVLink) copies
    PeerMesh* mesh_ = nullptr;
    std::unordered_map<int, PeerPlan> peer_plans_;
    void* ctx_buf_ = nullptr;
    size_t ctx_cap_ = 0;
    int32_t* argmax_buf_ = nullptr;
    float* logits_buf_ = nullptr;
    size_t argmax_cap_ = 0, logits_cap_ = 0;
    std::vector<std::vector<int32_t>> table_tokens_;
    std::vector<int> group_of_;
};

}  // namespace tkv
