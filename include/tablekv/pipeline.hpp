// tablekv B200 build — computation loading pipeline (drop-in for proj/include/tablekv/pipeline.hpp).
//
// schedule() cuts the served order into b_c windows with the next b_m queries' tables as
// prefetch candidates; build_trace() is the canonical cache trajectory (boundary demand gets,
// prefetch admissions with the deferral rule, per-query emergency reloads,
// pipeline.cpp:44-116) — exposed here because on the B200 it DRIVES every copy the executor
// issues. simulate() keeps the reference's virtual two-timeline clock as the predicted
// timeline next to measured GPU TTFTs.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "tablekv/errors.hpp"
#include "tablekv/rerank.hpp"
#include "tablekv/tiered_cache.hpp"

namespace tablekv {

struct CostModel {
    double compute_per_token = 0.01;
    double load_per_token = 1.0;
    double switch_overhead = 5.0;
    void validate() const {
        if (compute_per_token < 0 || load_per_token < 0 || switch_overhead < 0)
            throw Error(Errc::bad_config, "cost model parameters must be non-negative");
    }
};

struct SimQuery {
    std::string query_id;
    std::vector<int> tables;  // assembly order
    int query_tokens = 0;
};

struct BatchPlan {
    struct Window {
        size_t begin = 0;
        size_t end = 0;
        std::vector<int> demand;
        std::vector<int> prefetch;
    };
    int b_c = 0;
    int b_m = 0;
    std::vector<SimQuery> queries;
    std::vector<Window> windows;
    std::unordered_map<int, size_t> last_use;
};

BatchPlan schedule(std::vector<SimQuery> queries, int b_c, int b_m);

enum class SimMode { overlapped, serial };

struct SimReport {
    std::vector<std::string> query_ids;
    std::vector<double> ttft;
    double total_ttft = 0;
    double makespan = 0;
    double total_compute = 0;
    double total_transfer = 0;
    double serial_baseline_ttft = 0;
    std::uint64_t hits = 0;
    std::uint64_t misses = 0;
    std::uint64_t swaps = 0;
    std::uint64_t prefetch_loads = 0;

    std::string to_json() const;
    std::string to_csv() const;
};

// ---- canonical trace (B200 extension: public, consumed by the GPU executor) ----------------
struct LoadRec {
    int table = -1;
    bool miss = false;
    int evicted = -1;
    double size = 0;  // cost-model transfer units (0 for hits)
};

struct WindowTrace {
    std::vector<LoadRec> boundary;
    std::vector<LoadRec> prefetch;
    std::vector<std::vector<LoadRec>> emergency;  // per query of the window
};

struct Trace {
    std::vector<WindowTrace> windows;
    std::vector<double> compute;
};

// Per-record hook, called in trace order right after the cache decision it describes;
// kind: 0 boundary, 1 prefetch, 2 emergency (query = index in plan order, else -1).
struct TraceSink {
    virtual ~TraceSink() = default;
    virtual void on_window_begin(size_t window) { (void)window; }
    virtual void on_record(size_t window, int kind, long query, const LoadRec& r) = 0;
    virtual void on_query_ready(size_t window, size_t query) { (void)window, (void)query; }
};

Trace build_trace(const BatchPlan& plan, const CostModel& cost, TieredCache& cache, TraceSink* sink = nullptr);

SimReport simulate(const BatchPlan& plan, const CostModel& cost, TieredCache& cache, SimMode mode);

struct RunOptions {
    bool rerank_on = true;
    bool pipeline_on = true;
    size_t capacity = 8;
    EvictionPolicy policy = EvictionPolicy::lru;
    int b_c = 100;
    int b_m = 10;
    std::uint64_t seed = 1;
    AnchorMode anchor = AnchorMode::seeded;
};

SimReport run_batch(const std::vector<QueryRecord>& queries, const RunOptions& opts, const CostModel& cost,
                    std::shared_ptr<SlowTier> slow);

// order produced by run_batch's optional rerank (identity when off)
std::vector<size_t> serving_order(const std::vector<QueryRecord>& queries, const RunOptions& opts);

}  // namespace tablekv
