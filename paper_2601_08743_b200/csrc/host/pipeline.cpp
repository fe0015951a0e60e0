// Computation loading pipeline: schedule (proj/src/pipeline.cpp:147-174), the canonical cache
// trajectory build_trace (:44-116) with a per-record sink the GPU executor hooks, the virtual
// two-timeline clock simulate (:176-308) and run_batch (:310-342). Same decisions, new code.
#include <algorithm>
#include <cmath>
#include <limits>
#include <unordered_set>

#include <json.hpp>

#include "tablekv/pipeline.hpp"

namespace tablekv {

namespace {

// first-occurrence distinct append
struct Distinct {
    std::vector<int>& out;
    std::unordered_set<int> seen;
    void add(int t) {
        if (seen.insert(t).second) out.push_back(t);
    }
};

}  // namespace

BatchPlan schedule(std::vector<SimQuery> queries, int b_c, int b_m) {
    if (queries.empty()) throw Error(Errc::empty_batch, "cannot schedule an empty batch");
    if (b_c < 1 || b_m < 1) throw Error(Errc::bad_config, "b_c and b_m must be at least 1");
    BatchPlan plan;
    plan.b_c = b_c;
    plan.b_m = b_m;
    plan.queries = std::move(queries);
    const size_t n = plan.queries.size();
    for (size_t i = 0; i < n; ++i)
        for (int t : plan.queries[i].tables) plan.last_use[t] = i;
    for (size_t b = 0; b < n; b += size_t(b_c)) {
        BatchPlan::Window w;
        w.begin = b;
        w.end = std::min(n, b + size_t(b_c));
        Distinct dem{w.demand, {}};
        for (size_t i = w.begin; i < w.end; ++i)
            for (int t : plan.queries[i].tables) dem.add(t);
        Distinct pre{w.prefetch, {}};
        for (size_t i = w.end; i < std::min(n, w.end + size_t(b_m)); ++i)
            for (int t : plan.queries[i].tables) pre.add(t);
        plan.windows.push_back(std::move(w));
    }
    return plan;
}

Trace build_trace(const BatchPlan& plan, const CostModel& cost, TieredCache& cache, TraceSink* sink) {
    Trace tr;
    tr.windows.reserve(plan.windows.size());
    tr.compute.assign(plan.queries.size(), 0.0);
    const bool managed = cache.capacity() > 0;
    std::unordered_map<int, int> tokens;  // table -> token count, learned from loads
    std::vector<int> deferred;             // prefetch candidates postponed to the next window
    auto transfer = [&](int tok, bool swapped) { return cost.load_per_token * tok + (swapped ? cost.switch_overhead : 0.0); };

    for (size_t wi = 0; wi < plan.windows.size(); ++wi) {
        const auto& w = plan.windows[wi];
        if (sink) sink->on_window_begin(wi);
        WindowTrace wt;
        wt.emergency.resize(w.end - w.begin);
        const std::unordered_set<int> needed(w.demand.begin(), w.demand.end());
        if (managed) {
            // 1. demand gets at the window boundary
            for (int t : w.demand) {
                const GetResult g = cache.get(t);
                tokens[t] = g.kv->token_count;
                wt.boundary.push_back({t, !g.hit, g.evicted_id, g.hit ? 0.0 : transfer(g.kv->token_count, g.evicted_id >= 0)});
                if (sink) sink->on_record(wi, 0, -1, wt.boundary.back());
            }
            // 2. prefetch candidates: deferred ones first, then the next b_m queries' tables
            std::vector<int> cand;
            Distinct cd{cand, {}};
            for (int t : deferred) cd.add(t);
            for (int t : w.prefetch) cd.add(t);
            deferred.clear();
            for (int t : cand) {
                const auto lu = plan.last_use.find(t);
                if (lu == plan.last_use.end() || lu->second < w.begin) continue;  // nobody needs it any more
                const int one[1] = {t};
                if (cache.resident(t)) {
                    cache.prefetch(one);  // recency/frequency refresh only
                    continue;
                }
                int victim = -1;
                if (cache.size() == cache.capacity()) {
                    victim = cache.evict_candidate();
                    if (needed.count(victim)) {  // would evict a table this window still needs
                        deferred.push_back(t);
                        continue;
                    }
                }
                cache.prefetch(one);
                const int tok = cache.peek(t)->token_count;
                tokens[t] = tok;
                wt.prefetch.push_back({t, true, victim, transfer(tok, victim >= 0)});
                if (sink) sink->on_record(wi, 1, -1, wt.prefetch.back());
            }
        }
        // 3. per query: reload anything evicted inside the window, then its compute cost
        for (size_t qi = w.begin; qi < w.end; ++qi) {
            const SimQuery& q = plan.queries[qi];
            auto& em = wt.emergency[qi - w.begin];
            for (int t : q.tables) {
                if (managed && cache.resident(t)) continue;
                const GetResult g = cache.get(t);
                tokens[t] = g.kv->token_count;
                em.push_back({t, true, g.evicted_id, transfer(g.kv->token_count, g.evicted_id >= 0)});
                if (sink) sink->on_record(wi, 2, long(qi), em.back());
            }
            double ctx = 0;
            for (int t : q.tables) ctx += tokens.at(t);
            const double nq = q.query_tokens;
            tr.compute[qi] = cost.compute_per_token * (ctx * nq + nq * nq / 2.0);
            if (sink) sink->on_query_ready(wi, qi);
        }
        tr.windows.push_back(std::move(wt));
    }
    return tr;
}

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

// Background (prefetch) transfer: uses only gaps of the demand timeline, FIFO among jobs,
// cancelled if its table is evicted before completion.
struct Job {
    double size = 0, issue = 0, cancel = kInf, end = 0, wire = 0;
    bool placed = false;
};

class Timelines {
   public:
    double demand(double issue, double size) {
        const double s = std::max(issue, clock_);
        clock_ = s + size;
        if (size > 0) busy_.push_back({s, clock_});
        demand_total_ += size;
        return clock_;
    }
    double clock() const { return clock_; }
    double demand_total() const { return demand_total_; }

    size_t add_job(double size, double issue) {
        jobs_.push_back({size, issue});
        return jobs_.size() - 1;
    }
    Job& job(size_t i) { return jobs_[i]; }
    size_t jobs() const { return jobs_.size(); }

    // place jobs [next_, through] into the demand gaps (exact: all demand intervals that can
    // precede a job's completion are known when its table is first awaited)
    void place_through(size_t through) {
        for (; next_ <= through; ++next_) {
            Job& j = jobs_[next_];
            double at = std::max(cursor_, j.issue), left = j.size;
            while (left > 0 && at < j.cancel) {
                const double bs = bi_ < busy_.size() ? busy_[bi_].first : kInf;
                const double be = bi_ < busy_.size() ? busy_[bi_].second : kInf;
                if (be <= at) {
                    ++bi_;
                    continue;
                }
                if (bs > at) {
                    const double take = std::min(left, std::min(bs, j.cancel) - at);
                    j.wire += take;
                    left -= take;
                    at += take;
                    continue;
                }
                if (j.cancel <= be) {
                    at = j.cancel;
                    break;
                }
                at = be;
                ++bi_;
            }
            j.end = std::min(at, j.cancel);
            j.placed = true;
            cursor_ = std::max(cursor_, at);
        }
    }
    double wire_total() const {
        double w = 0;
        for (const Job& j : jobs_) w += j.wire;
        return w;
    }

   private:
    double clock_ = 0, demand_total_ = 0, cursor_ = 0;
    std::vector<std::pair<double, double>> busy_;
    std::vector<Job> jobs_;
    size_t next_ = 0, bi_ = 0;
};

}  // namespace

SimReport simulate(const BatchPlan& plan, const CostModel& cost, TieredCache& cache, SimMode mode) {
    cost.validate();
    const bool managed = cache.capacity() > 0;
    const Trace tr = build_trace(plan, cost, cache);
    SimReport rep;
    Timelines tl;
    std::unordered_map<int, double> ready;
    std::unordered_map<int, size_t> inflight;  // table -> background job
    double cc = 0;  // compute clock

    auto evicted = [&](int victim, double when) {
        if (victim < 0) return;
        ready.erase(victim);
        if (const auto it = inflight.find(victim); it != inflight.end()) {
            Job& j = tl.job(it->second);
            if (!j.placed) j.cancel = std::min(j.cancel, when);
            inflight.erase(it);
        }
    };

    for (size_t wi = 0; wi < plan.windows.size(); ++wi) {
        const auto& w = plan.windows[wi];
        const auto& wt = tr.windows[wi];
        const double boundary = cc;
        for (const LoadRec& r : wt.boundary) {
            if (!r.miss) continue;
            evicted(r.evicted, boundary);
            ready[r.table] = tl.demand(boundary, r.size);
        }
        for (const LoadRec& r : wt.prefetch) {
            evicted(r.evicted, boundary);
            if (mode == SimMode::overlapped)
                inflight[r.table] = tl.add_job(r.size, boundary);
            else
                ready[r.table] = tl.demand(boundary, r.size);
        }
        if (mode == SimMode::serial) cc = std::max(cc, tl.clock());
        for (size_t qi = w.begin; qi < w.end; ++qi) {
            const SimQuery& q = plan.queries[qi];
            for (const LoadRec& r : wt.emergency[qi - w.begin]) {
                const double issue = (mode == SimMode::serial || managed) ? cc : boundary;
                evicted(r.evicted, issue);
                ready[r.table] = tl.demand(issue, r.size);
            }
            double avail = 0;
            for (int t : q.tables) {
                if (const auto it = inflight.find(t); it != inflight.end()) {
                    tl.place_through(it->second);
                    ready[t] = tl.job(it->second).end;
                    inflight.erase(it);
                }
                if (const auto it = ready.find(t); it != ready.end()) avail = std::max(avail, it->second);
            }
            cc = std::max(cc, avail) + tr.compute[qi];
            rep.total_compute += tr.compute[qi];
            rep.query_ids.push_back(q.query_id);
            rep.ttft.push_back(cc);
        }
    }
    if (tl.jobs()) tl.place_through(tl.jobs() - 1);
    for (double t : rep.ttft) rep.total_ttft += t;
    rep.makespan = cc;
    rep.total_transfer = tl.demand_total() + tl.wire_total();
    const CacheCounters& c = cache.counters();
    rep.hits = c.hits;
    rep.misses = c.misses;
    rep.swaps = c.swaps;
    rep.prefetch_loads = c.prefetch_loads;
    return rep;
}

std::vector<size_t> serving_order(const std::vector<QueryRecord>& queries, const RunOptions& opts) {
    if (opts.rerank_on) return rerank(queries, opts.seed, opts.anchor);
    std::vector<size_t> ord(queries.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
    return ord;
}

SimReport run_batch(const std::vector<QueryRecord>& queries, const RunOptions& opts, const CostModel& cost,
                    std::shared_ptr<SlowTier> slow) {
    if (queries.empty()) return SimReport{};
    std::vector<SimQuery> sims;
    sims.reserve(queries.size());
    for (size_t i : serving_order(queries, opts)) sims.push_back({queries[i].query_id, queries[i].tables, queries[i].query_token_count});
    const BatchPlan plan = schedule(std::move(sims), opts.b_c, opts.b_m);
    TieredCache cache(opts.capacity, opts.policy, slow);
    SimReport rep = simulate(plan, cost, cache, opts.pipeline_on ? SimMode::overlapped : SimMode::serial);
    if (opts.pipeline_on) {
        TieredCache fresh(opts.capacity, opts.policy, slow);
        rep.serial_baseline_ttft = simulate(plan, cost, fresh, SimMode::serial).total_ttft;
    } else {
        rep.serial_baseline_ttft = rep.total_ttft;
    }
    return rep;
}

std::string SimReport::to_json() const {
    nlohmann::json j;
    j["format_version"] = 1;
    j["total_ttft"] = total_ttft;
    j["serial_baseline_ttft"] = serial_baseline_ttft;
    j["makespan"] = makespan;
    j["total_compute"] = total_compute;
    j["total_transfer"] = total_transfer;
    j["hits"] = hits;
    j["misses"] = misses;
    j["swaps"] = swaps;
    j["prefetch_loads"] = prefetch_loads;
    nlohmann::json qs = nlohmann::json::array();
    for (size_t i = 0; i < ttft.size(); ++i) qs.push_back({{"query_id", query_ids[i]}, {"ttft", ttft[i]}});
    j["queries"] = std::move(qs);
    return j.dump(2);
}

std::string SimReport::to_csv() const {
    std::string s = "query_id,ttft\n";
    for (size_t i = 0; i < ttft.size(); ++i) s += query_ids[i] + "," + nlohmann::json(ttft[i]).dump() + "\n";
    return s;
}

}  // namespace tablekv
