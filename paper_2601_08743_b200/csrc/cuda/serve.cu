// GPU executor (see serve.cuh). The host computes the canonical trace with the reference's
// exact cache decisions (tablekv::build_trace over a metadata-only slow tier), then replays it:
// every miss / prefetch becomes a page copy from the pinned arena into the HBM pool (demand
// loads on one copy stream, prefetches on another so they overlap the current window's
// compute), evicted tables' pages are recycled only after the compute that may read them.
// Each window of b_c queries is one gather + one batched prefill on the compute stream.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <functional>
#include <memory>
#include <numeric>

#include "common.cuh"
#include "serve.cuh"

namespace tkv {

namespace {

// Slow tier that only knows token counts: the policy trace needs no tensor bytes.
class MetaTier : public tablekv::SlowTier {
   public:
    explicit MetaTier(const Arena& a) : arena_(a) {}
    bool contains(int id) const override { return arena_.find(id) != nullptr; }
    std::shared_ptr<const tablekv::TableKV<float>> load(int id) override {
        auto it = cache_.find(id);
        if (it != cache_.end()) return it->second;
        const TableImage* img = arena_.find(id);
        if (!img) throw tablekv::Error(tablekv::Errc::unknown_table, "table " + std::to_string(id) + " not in the arena");
        auto kv = std::make_shared<tablekv::TableKV<float>>();
        kv->table_id = id;
        kv->token_count = img->tokens;
        cache_.emplace(id, kv);
        return kv;
    }

   private:
    const Arena& arena_;
    std::unordered_map<int, std::shared_ptr<const tablekv::TableKV<float>>> cache_;
};

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct EventPool {
    std::vector<cudaEvent_t> evs;
    size_t used = 0;
    cudaEvent_t get() {
        if (used == evs.size()) {
            cudaEvent_t e;
            TKV_CUDA_CHECK(cudaEventCreate(&e));
            evs.push_back(e);
        }
        return evs[used++];
    }
    ~EventPool() {
        for (auto e : evs) cudaEventDestroy(e);
    }
};

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

}  // namespace

BatchTrace plan_batch(const std::vector<std::vector<int>>& tables, const std::vector<int>& suffix_len,
                      const ServeOptions& opts, const Arena& arena, cudaStream_t stream) {
    BatchTrace bt;
    int n_bits = 0;
    for (const auto& q : tables)
        for (int t : q) n_bits = std::max(n_bits, t + 1);
    std::vector<tablekv::QueryRecord> recs;
    recs.reserve(tables.size());
    for (size_t i = 0; i < tables.size(); ++i) {
        auto r = tablekv::make_query_record("q" + std::to_string(i), {}, tables[i], std::max(1, n_bits), suffix_len[i]);
        r.tables = tables[i];
        recs.push_back(std::move(r));
    }
    if (opts.run.rerank_on && recs.size() >= kDeviceRerankMin) {
        const size_t words = recs.front().inc.words.size();
        std::vector<uint64_t> packed(recs.size() * words, 0);
        for (size_t i = 0; i < recs.size(); ++i)
            if (!recs[i].tables.empty()) std::copy(recs[i].inc.words.begin(), recs[i].inc.words.end(), packed.begin() + long(i * words));
        bt.order = rerank_device(packed.data(), recs.size(), words, opts.run.seed, opts.run.anchor, stream);
    } else {
        bt.order = tablekv::serving_order(recs, opts.run);
    }
    std::vector<tablekv::SimQuery> sims;
    for (size_t i : bt.order) sims.push_back({recs[i].query_id, tables[i], suffix_len[i]});
    bt.plan = tablekv::schedule(std::move(sims), opts.run.b_c, opts.run.b_m);
    auto meta = std::make_shared<MetaTier>(arena);
    tablekv::TieredCache cache(opts.run.capacity, opts.run.policy, meta);
    bt.trace = tablekv::build_trace(bt.plan, opts.cost, cache);
    bt.counters = cache.counters();
    bt.managed = opts.run.capacity > 0;
    return bt;
}

std::unordered_map<int, std::vector<std::pair<int, int>>> residency_intervals(const BatchTrace& bt) {
    // the executor publishes demand loads of window w at compute(w), prefetches of w at
    // compute(w + 1), and revokes a victim after compute(w) (serve() below)
    std::unordered_map<int, std::vector<std::pair<int, int>>> live;
    std::unordered_map<int, int> open;  // table -> publish window
    if (bt.plan.windows.empty() || !bt.managed) return live;
    auto close = [&](int t, int w) {
        auto it = open.find(t);
        if (it == open.end()) return;
        if (it->second <= w) live[t].push_back({it->second, w});
        open.erase(it);
    };
    const int last = int(bt.trace.windows.size()) - 1;
    for (int w = 0; w <= last; ++w) {
        const auto& wt = bt.trace.windows[size_t(w)];
        for (const auto& r : wt.boundary)
            if (r.miss) close(r.evicted, w), open[r.table] = w;
        for (const auto& r : wt.prefetch) close(r.evicted, w), open[r.table] = w + 1;
        for (const auto& q : wt.emergency)
            for (const auto& r : q) close(r.evicted, w), open[r.table] = w;
    }
    for (auto& kv : open)
        if (kv.second <= last) live[kv.first].push_back({kv.second, last});
    return live;
}

Server::Server(Model& model, Arena& arena, PagePool& pool) : model_(model), arena_(arena), pool_(pool) {
    int lo, hi;
    TKV_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    TKV_CUDA_CHECK(cudaStreamCreateWithPriority(&cs_, cudaStreamNonBlocking, hi));
    TKV_CUDA_CHECK(cudaStreamCreateWithPriority(&ds_, cudaStreamNonBlocking, hi));
    TKV_CUDA_CHECK(cudaStreamCreateWithPriority(&ps_, cudaStreamNonBlocking, lo));
    TKV_CUDA_CHECK(cudaStreamCreateWithPriority(&xs_, cudaStreamNonBlocking, hi));
}

void Server::set_peer_plan(int slot, PeerPlan plan) {
    if (plan.tables.size() != plan.suffix_len.size()) throw std::invalid_argument("peer plan: tables/suffix_len size mismatch");
    peer_plans_[slot] = std::move(plan);
}

Server::~Server() {
    cudaDeviceSynchronize();
    cudaFree(ctx_buf_);
    cudaFree(argmax_buf_);
    cudaFree(logits_buf_);
    cudaStreamDestroy(cs_);
    cudaStreamDestroy(ds_);
    cudaStreamDestroy(ps_);
    cudaStreamDestroy(xs_);
}

void Server::set_table_tokens(std::vector<std::vector<int32_t>> tt, std::vector<int> group_of) {
    table_tokens_ = std::move(tt);
    group_of_ = std::move(group_of);
}

void Server::ensure_out(size_t n_argmax, size_t n_logits) {
    // per-batch outputs stay allocated across calls: no allocator traffic (and no implicit
    // synchronisation or pool trimming) inside a serve
    if (n_argmax > argmax_cap_) {
        TKV_CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(argmax_buf_);
        argmax_cap_ = std::max(n_argmax, argmax_cap_ * 2);
        TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&argmax_buf_), argmax_cap_ * sizeof(int32_t)));
    }
    if (n_logits > logits_cap_) {
        TKV_CUDA_CHECK(cudaDeviceSynchronize());
        cudaFree(logits_buf_);
        logits_cap_ = std::max(n_logits, logits_cap_ * 2);
        TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&logits_buf_), logits_cap_ * sizeof(float)));
    }
}

void Server::ensure_ctx(size_t bytes) {
    if (bytes <= ctx_cap_) return;
    TKV_CUDA_CHECK(cudaDeviceSynchronize());
    cudaFree(ctx_buf_);
    ctx_cap_ = std::max(bytes, ctx_cap_ * 2);
    TKV_CUDA_CHECK(cudaMalloc(&ctx_buf_, ctx_cap_));
    TKV_CUDA_CHECK(cudaMemset(ctx_buf_, 0, ctx_cap_));  // rows past a window's prefix stay finite (masked tiles read them)
}

ServeResult Server::serve(const std::vector<ServeQuery>& queries, const ServeOptions& opts) {
    ServeResult R;
    if (queries.empty()) return R;
    const long ring_launches0 = model_.ring().launches();
    const ModelCfg& mc = model_.cfg();
    const int L = mc.num_layers, kvd = mc.kv_dim();
    const DType out_dt = mc.dtype == DType::bf16 ? DType::bf16 : DType::f32;
    const size_t oes = dtype_size(out_dt);
    const size_t P = pool_.page_bytes();
    EventPool evp;
    const double host0 = now_ms();
    cudaEvent_t t0 = evp.get();
    TKV_CUDA_CHECK(cudaEventRecord(t0, cs_));
    TKV_CUDA_CHECK(cudaStreamWaitEvent(ds_, t0));
    TKV_CUDA_CHECK(cudaStreamWaitEvent(ps_, t0));

    // ---- host: records, rerank, schedule, canonical trace (reference decisions)
    std::vector<std::vector<int>> qt;
    std::vector<int> qn;
    for (const auto& q : queries) qt.push_back(q.tables), qn.push_back(int(q.suffix.size()));
    static const bool host_prof = std::getenv("TKV_HOST_PROFILE") != nullptr;  // debug: host-side phase timers
    double hp_plan = 0, hp_copy = 0, hp_fwd = 0, hp_rest = 0, hp_mark = now_ms();
    auto hp_tick = [&](double& acc) {
        const double t = now_ms();
        acc += t - hp_mark;
        hp_mark = t;
    };
    BatchTrace bt = plan_batch(qt, qn, opts, arena_, cs_);
    R.order = std::move(bt.order);
    const tablekv::BatchPlan& plan = bt.plan;
    const tablekv::Trace& tr = bt.trace;
    R.counters = bt.counters;
    // peers' predicted residency (table -> [published window, revoked window] intervals per slot)
    const bool peering = opts.peer_fetch && mesh_ && mesh_->n_peers() > 0;
    std::vector<std::unordered_map<int, std::vector<std::pair<int, int>>>> peer_live;
    if (peering)
        for (int p = 0; p < mesh_->n_peers(); ++p) {
            auto it = peer_plans_.find(p);
            peer_live.push_back(it == peer_plans_.end() ? decltype(peer_live)::value_type{}
                                                        : residency_intervals(plan_batch(it->second.tables, it->second.suffix_len, opts, arena_)));
        }
    // the peers whose pool should hold table t when this GPU fetches for window w: the copy runs
    // during compute(w-1), when a peer in step is between its windows w-1 and w, so a peer whose
    // predicted residency overlaps [w-1, w] is tried first (each copy CTA re-checks the live
    // directory entry and falls back to the host arena if the table is not published yet or any
    // more); -1 terminated
    auto predict = [&](int t, int w) {
        PeerOrder o;
        for (int i = 0; i < kMaxPeers; ++i) o.p[i] = -1;
        int k = 0;
        for (size_t p = 0; p < peer_live.size() && k < kMaxPeers; ++p) {
            auto it = peer_live[p].find(t);
            if (it == peer_live[p].end()) continue;
            for (const auto& iv : it->second)
                if (iv.first <= w && iv.second >= w - 1) {
                    o.p[k++] = int8_t(p);
                    break;
                }
        }
        return o;
    };

    // ---- compute groups: consecutive windows with tiny suffixes (the reference's b_c = 1 demo
    // configuration) share one prefill; a group closes once it holds kGroupRows suffix rows, which a
    // single window of the serving configurations already does (so those run one window at a time).
    // Copies, the cache trace and page lifetimes stay per window; a query's TTFT is its group's end.
    constexpr long kGroupRows = 1024;
    constexpr int kGroupWindows = 64;
    const bool grouping = mesh_ == nullptr && !peering;
    std::vector<char> closes(plan.windows.size(), 1);
    if (grouping) {
        long rows = 0;
        int nw = 0;
        for (size_t wi = 0; wi < plan.windows.size(); ++wi) {
            for (size_t qi = plan.windows[wi].begin; qi < plan.windows[wi].end; ++qi) rows += long(queries[R.order[qi]].suffix.size());
            ++nw;
            closes[wi] = rows >= kGroupRows || nw >= kGroupWindows || wi + 1 == plan.windows.size();
            if (closes[wi]) rows = 0, nw = 0;
        }
    }
    // ---- sizing: context slab for the largest group, rope table for the longest row
    long max_ctx_rows = 0;
    int max_pos = 1;
    size_t max_q = 0;
    {
        long rows = 0;
        size_t nq = 0;
        for (size_t wi = 0; wi < plan.windows.size(); ++wi) {
            const auto& w = plan.windows[wi];
            for (size_t qi = w.begin; qi < w.end; ++qi) {
                long c = 0;
                for (int t : plan.queries[qi].tables) c += arena_.find(t)->tokens;
                rows += c;
                max_pos = std::max<int>(max_pos, int(c + long(queries[R.order[qi]].suffix.size()) + 1));
            }
            nq += w.end - w.begin;
            if (closes[wi]) {
                max_ctx_rows = std::max(max_ctx_rows, rows);
                max_q = std::max(max_q, nq);
                rows = 0, nq = 0;
            }
        }
    }
    model_.rope().ensure(max_pos);
    // bf16 serving streams the prefix one layer at a time (gathered right before that layer's
    // attention), so the slab holds one layer of the window's prefix, not L
    const bool stream_ctx = mc.dtype == DType::bf16;
    const int slab_layers = stream_ctx ? 1 : L;
    ensure_ctx(std::max<size_t>(256, size_t(2) * slab_layers * size_t(max_ctx_rows) * kvd * oes));
    uint8_t* ctx_k = static_cast<uint8_t*>(ctx_buf_);
    uint8_t* ctx_v = ctx_k + size_t(slab_layers) * size_t(max_ctx_rows) * kvd * oes;
    int32_t* d_argmax = nullptr;
    float* d_logits = nullptr;
    const int vp = mc.vocab_padded();
    ensure_out(queries.size(), max_q * size_t(vp));
    d_argmax = argmax_buf_;
    d_logits = logits_buf_;
    std::vector<float> logits_host;
    if (opts.keep_logits) logits_host.resize(queries.size() * size_t(vp));

    // ---- physical replay
    const bool managed = opts.run.capacity > 0;
    std::unordered_map<int, std::vector<int32_t>> resident;
    // Bookkeeping first, bytes second: records only allocate pages and queue the copy; each
    // window's copies are then issued back-to-back per stream so the copy engines stream
    // without host-side gaps between tables.
    struct PendingCopy {
        const TableImage* img;
        std::vector<int32_t> pages;
        cudaStream_t st;
        PeerOrder peers;
    };
    std::vector<PendingCopy> pending;
    size_t cur_window = 0;
    auto load = [&](int t, cudaStream_t st) {
        const TableImage* img = arena_.find(t);
        std::vector<int32_t> pages = pool_.alloc(int((img->bytes + P - 1) / P));
        PeerOrder po{};
        for (int i = 0; i < kMaxPeers; ++i) po.p[i] = -1;
        if (peering && managed && img->bytes % 16 == 0 && int(pages.size()) <= kMaxPagesPerCopy) po = predict(t, int(cur_window));
        if (po.p[0] >= 0) {
            pending.push_back({img, pages, xs_, po});
            R.peer_routed_bytes += img->bytes;
        } else {
            pending.push_back({img, pages, st, po});
            R.h2d_bytes += img->bytes;
            if (st == ds_) R.h2d_demand_bytes += img->bytes;
        }
        return pages;
    };
    auto page_list = [](const std::vector<int32_t>& pages) {
        if (pages.size() > size_t(kMaxPagesPerCopy))
            throw std::invalid_argument("peer page list: " + std::to_string(pages.size()) + " pages exceed " +
                                        std::to_string(kMaxPagesPerCopy));
        PageList pl;
        pl.n = int(pages.size());
        for (size_t i = 0; i < pages.size(); ++i) pl.page[i] = pages[i];
        return pl;
    };
    auto flush_copies = [&](cudaStream_t st) {
        for (const auto& c : pending) {
            if (c.st != st) continue;
            if (st == xs_)
                launch_peer_fetch(mesh_->view(), c.peers, c.img->table_id, c.img->mapped, c.img->bytes, pool_.base(), P,
                                  page_list(c.pages), mesh_->stats(), opts.peer_ctas, xs_);
            else
                copy_table_to_pages(*c.img, pool_, c.pages, opts.engine, opts.sm_copy_ctas, st);
        }
    };
    // tables this GPU has published in its directory for peers (table -> pages), and the loads
    // waiting to be published: demand loads of window w at compute(w), prefetches at compute(w+1)
    std::unordered_map<int, std::vector<int32_t>> published;
    std::vector<std::pair<int, std::vector<int32_t>>> pub_now, pub_next;
    const bool sharing = mesh_ != nullptr && managed;
    // only tables a peer can fetch go into the directory: an id inside it and a page list that
    // fits one DirEntry (larger tables are served from the host arena by every rank)
    auto publishable = [&](int t, const std::vector<int32_t>& pages) {
        return sharing && t >= 0 && t < mesh_->dir_entries() && pages.size() <= size_t(kMaxPagesPerCopy);
    };
    if (peering) {
        TKV_CUDA_CHECK(cudaMemsetAsync(mesh_->stats(), 0, 2 * sizeof(unsigned long long), cs_));
        cudaEvent_t z = evp.get();
        TKV_CUDA_CHECK(cudaEventRecord(z, cs_));
        TKV_CUDA_CHECK(cudaStreamWaitEvent(xs_, z));
    }
    std::vector<cudaEvent_t> win_end(plan.windows.size());
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> dspan, pspan;
    std::vector<cudaEvent_t> cstart(plan.windows.size(), nullptr);
    cudaEvent_t prev_pref = nullptr;
    R.window_of.assign(plan.queries.size(), 0);
    R.argmax.assign(plan.queries.size(), -1);

    // the open compute group's accumulated prefill inputs
    std::vector<GatherSeg> segs;
    std::vector<int32_t> page_ids, tokens, pos, logit_rows;
    std::vector<int64_t> pos64;
    std::vector<AttnSeq> seqs;
    std::vector<size_t> seq_query;
    std::vector<int32_t> seq_seg0;  // per prefilled sequence: its first segment (the attention's page walk)
    int ctx_rows = 0, M = 0;
    size_t group_first = 0;  // first window of the open group
    bool in_dt_set = false;
    DType in_dt_s = DType::bf16;
    std::vector<std::pair<int, std::vector<int32_t>>> dropped;  // evicted in the group: recycle after its compute

    // A throw inside the replay (pool exhausted, CUDA error, bad input) must not leak the batch's
    // pages or leave directory entries published: drain the streams, revoke, return every page.
    struct Unwind {
        std::function<void()> fn;
        bool armed = true;
        ~Unwind() {
            if (!armed) return;
            try {
                fn();
            } catch (...) {
            }
        }
    } unwind{[&] {
        cudaDeviceSynchronize();
        if (mesh_)
            for (auto& kv : published) launch_dir_revoke(*mesh_, kv.first, cs_);
        for (auto& kv : dropped) pool_.release(kv.second, cs_);
        for (auto& kv : resident) pool_.release(kv.second, cs_);
        cudaStreamSynchronize(cs_);
    }};

    // The host runs at most `host_lead` windows ahead of the GPU: without a bound it queues every
    // window's loads at once, and a window's demand copies then wait behind the prefetch backlog
    // of later windows on the copy engines (TKV_HOST_LEAD=0: unbounded)
    static const int host_lead = [] {
        const char* e = std::getenv("TKV_HOST_LEAD");
        return e ? std::atoi(e) : 2;
    }();
    static const bool layered_env = [] {  // TKV_LAYERED_LOADS=1: layer-ordered demand copies (measured slower)
        const char* e = std::getenv("TKV_LAYERED_LOADS");
        return e && std::atoi(e) != 0;
    }();
    constexpr int kLayerChunk = 4;
    const int n_lchunks = (L + kLayerChunk - 1) / kLayerChunk;
    std::vector<std::vector<cudaEvent_t>> lchunk_ev(plan.windows.size(), std::vector<cudaEvent_t>(size_t(n_lchunks), nullptr));
    hp_tick(hp_plan);
    for (size_t wi = 0; wi < plan.windows.size(); ++wi) {
        if (host_lead > 0 && wi >= size_t(host_lead) && win_end[wi - host_lead])
            TKV_CUDA_CHECK(cudaEventSynchronize(win_end[wi - host_lead]));
        const auto& w = plan.windows[wi];
        const auto& wt = tr.windows[wi];
        cur_window = wi;
        pub_now.swap(pub_next);  // prefetches of the previous window
        pub_next.clear();
        // Pages of tables evicted during this window stay readable until compute(wi) is done.
        // The reference trace lets a query's own emergency get evict another of its tables
        // without reloading it (pipeline.cpp:98-107), so snapshots may need them.
        std::unordered_map<int, std::vector<int32_t>> gone;
        auto evict = [&](int victim) {
            if (victim < 0) return;
            auto it = resident.find(victim);
            if (it != resident.end()) {
                gone[victim] = it->second;
                dropped.push_back({victim, std::move(it->second)});
                resident.erase(it);
            }
        };
        pending.clear();
        for (const auto& r : wt.boundary) {
            R.trace.push_back({int(wi), 0, -1, r.table, r.evicted, r.miss, 0});
            if (!r.miss) continue;
            evict(r.evicted);
            resident[r.table] = load(r.table, ds_);
            if (publishable(r.table, resident[r.table])) pub_now.push_back({r.table, resident[r.table]});
            R.trace.back().bytes = arena_.find(r.table)->bytes;
        }
        for (const auto& r : wt.prefetch) {
            R.trace.push_back({int(wi), 1, -1, r.table, r.evicted, true, arena_.find(r.table)->bytes});
            evict(r.evicted);
            resident[r.table] = load(r.table, ps_);
            if (publishable(r.table, resident[r.table])) pub_next.push_back({r.table, resident[r.table]});
        }
        // per query: emergency reloads, then a snapshot of its tables' pages
        struct Seg {
            int table, tokens;
            std::vector<int32_t> pages;
        };
        std::vector<std::vector<Seg>> qsegs(w.end - w.begin);
        for (size_t qi = w.begin; qi < w.end; ++qi) {
            std::unordered_map<int, std::vector<int32_t>> local;  // capacity 0: load-through copies
            for (const auto& r : wt.emergency[qi - w.begin]) {
                R.trace.push_back({int(wi), 2, long(qi), r.table, r.evicted, true, arena_.find(r.table)->bytes});
                evict(r.evicted);
                auto pages = load(r.table, ds_);
                if (managed) {
                    if (publishable(r.table, pages)) pub_now.push_back({r.table, pages});
                    resident[r.table] = std::move(pages);
                }
                else
                    local[r.table] = std::move(pages);
            }
            for (int t : plan.queries[qi].tables) {
                const std::vector<int32_t>* pg = nullptr;
                if (!managed) pg = &local.at(t);
                else if (auto r = resident.find(t); r != resident.end()) pg = &r->second;
                else pg = &gone.at(t);  // evicted earlier in this window, bytes still intact
                qsegs[qi - w.begin].push_back({t, arena_.find(t)->tokens, *pg});
            }
            if (!managed)
                for (auto& kv : local) dropped.push_back({-1, std::move(kv.second)});
        }
        cudaEvent_t d0 = evp.get(), p0 = evp.get(), d1 = evp.get(), p1 = evp.get();
        hp_tick(hp_rest);
        TKV_CUDA_CHECK(cudaEventRecord(d0, ds_));
        // Layer-ordered demand loads: the window's tables are copied kLayerChunk layers at a time
        // (K rows then V rows of those layers, image byte ranges [l0 T, l1 T) rows), an event after
        // each chunk; the prefill starts after the first chunk and each layer's attention waits
        // only for its own chunk — the projections of early layers overlap the later layers' H2D.
        // (Whole tables when a peer may read the published pages, for the SM copy kernel, and for
        // the f32 models whose prefix is gathered for all layers at once.)
        const bool layered = layered_env && stream_ctx && !peering && opts.engine == CopyEngine::dma;
        if (layered) {
            for (int c = 0; c < n_lchunks; ++c) {
                const int l0 = c * kLayerChunk, l1 = std::min(L, l0 + kLayerChunk);
                for (const auto& pc : pending) {
                    if (pc.st != ds_) continue;
                    const size_t blk = pc.img->bytes / size_t(2 * L);  // one layer of K (or V) rows
                    copy_image_range_to_pages(*pc.img, pool_, pc.pages, size_t(l0) * blk, size_t(l1 - l0) * blk, ds_);
                    copy_image_range_to_pages(*pc.img, pool_, pc.pages, size_t(L + l0) * blk, size_t(l1 - l0) * blk, ds_);
                }
                lchunk_ev[wi][size_t(c)] = evp.get();
                TKV_CUDA_CHECK(cudaEventRecord(lchunk_ev[wi][size_t(c)], ds_));
            }
        } else {
            flush_copies(ds_);
        }
        TKV_CUDA_CHECK(cudaEventRecord(d1, ds_));
        TKV_CUDA_CHECK(cudaEventRecord(p0, ps_));
        flush_copies(ps_);
        TKV_CUDA_CHECK(cudaEventRecord(p1, ps_));
        dspan.push_back({d0, d1});
        pspan.push_back({p0, p1});
        hp_tick(hp_copy);
        cudaEvent_t x1 = nullptr;
        if (peering) {
            // peer copies of window w run during compute(w-1): the peers are then around the
            // same window, where the prediction placed the table
            if (wi >= 2) TKV_CUDA_CHECK(cudaStreamWaitEvent(xs_, win_end[wi - 2]));
            flush_copies(xs_);
            x1 = evp.get();
            TKV_CUDA_CHECK(cudaEventRecord(x1, xs_));
        }

        // ---- compute(wi): needs this window's demand loads and every earlier prefetch (a window
        // that opens its own compute group and was loaded layer by layer: only the first chunk here,
        // the rest per layer inside the prefill)
        const bool layer_waits = layered && group_first == wi && closes[wi];
        TKV_CUDA_CHECK(cudaStreamWaitEvent(cs_, layer_waits ? lchunk_ev[wi][0] : d1));
        if (prev_pref) TKV_CUDA_CHECK(cudaStreamWaitEvent(cs_, prev_pref));
        prev_pref = p1;
        if (x1) TKV_CUDA_CHECK(cudaStreamWaitEvent(cs_, x1));
        cstart[wi] = evp.get();  // compute(wi) may start here (its waits are satisfied)
        TKV_CUDA_CHECK(cudaEventRecord(cstart[wi], cs_));
        // publish what landed for this window (still resident with the same pages)
        for (auto& [t, pages] : pub_now) {
            auto it = resident.find(t);
            if (it == resident.end() || it->second != pages) continue;
            launch_dir_publish(*mesh_, t, page_list(pages), cs_);
            published[t] = pages;
        }
        pub_now.clear();

        for (size_t qi = w.begin; qi < w.end; ++qi) {
            const ServeQuery& q = queries[R.order[qi]];
            R.window_of[qi] = int(wi);
            int cursor = 0;
            const int q_ctx0 = ctx_rows;
            const int q_seg0 = int(segs.size());
            for (const Seg& s : qsegs[qi - w.begin]) {
                segs.push_back({int32_t(page_ids.size()), s.tokens, cursor, ctx_rows});
                page_ids.insert(page_ids.end(), s.pages.begin(), s.pages.end());
                cursor += s.tokens;
                ctx_rows += s.tokens;
            }
            R.total_ctx_tokens += cursor;
            if (q.suffix.empty()) continue;  // nothing to prefill, no first token
            seqs.push_back({M, int(q.suffix.size()), q_ctx0, cursor});
            seq_seg0.push_back(q_seg0);
            seq_query.push_back(qi);
            for (size_t i = 0; i < q.suffix.size(); ++i) {
                tokens.push_back(q.suffix[i]);
                pos.push_back(cursor + int(i));
                pos64.push_back(cursor + int64_t(i));
            }
            M += int(q.suffix.size());
            logit_rows.push_back(M - 1);
        }
        for (const auto& qs : qsegs)
            if (!qs.empty() && !in_dt_set) {  // the arena holds one dtype per corpus
                in_dt_s = arena_.find(qs.front().table)->dtype;
                in_dt_set = true;
            }
        if (!closes[wi]) continue;  // the group stays open: this window computes with the next ones
        R.total_suffix_tokens += M;
        StagingRing& ring = model_.ring();
        const GatherSeg* d_segs_s = nullptr;
        const int32_t* d_pages_s = nullptr;
        const int4* d_chunks_s = nullptr;
        int n_chunks_s = 0;
        if (ctx_rows > 0 && stream_ctx && M > 0) {
            d_segs_s = static_cast<GatherSeg*>(ring.upload(segs.data(), segs.size() * sizeof(GatherSeg), cs_));
            d_pages_s = static_cast<int32_t*>(ring.upload(page_ids.data(), page_ids.size() * 4, cs_));
            std::vector<int4> chunks;
            n_chunks_s = gather_chunks(segs.data(), int(segs.size()), chunks);
            d_chunks_s = static_cast<const int4*>(ring.upload(chunks.data(), chunks.size() * sizeof(int4), cs_));
            R.meta_bytes += chunks.size() * sizeof(int4);
            R.meta_bytes += segs.size() * sizeof(GatherSeg) + page_ids.size() * 4;
        } else if (ctx_rows > 0 && !stream_ctx) {
            auto* d_segs = static_cast<GatherSeg*>(ring.upload(segs.data(), segs.size() * sizeof(GatherSeg), cs_));
            auto* d_pages = static_cast<int32_t*>(ring.upload(page_ids.data(), page_ids.size() * 4, cs_));
            R.meta_bytes += segs.size() * sizeof(GatherSeg) + page_ids.size() * 4;
            const DType in_dt = in_dt_set ? in_dt_s : DType::f32;
            cudaEvent_t g0 = nullptr, g1 = nullptr;
            if (opts.time_kernels) {
                g0 = evp.get();
                g1 = evp.get();
                TKV_CUDA_CHECK(cudaEventRecord(g0, cs_));
            }
            ring.flush(cs_);
            launch_gather_rope(pool_.base(), P, d_pages, d_segs, int(segs.size()), ctx_rows, L, kvd, mc.head_dim, in_dt,
                               out_dt, model_.rope().cos_d(), model_.rope().sin_d(), model_.rope().cos_f(),
                               model_.rope().sin_f(), ctx_k, ctx_v, max_ctx_rows, cs_);
            R.launches += 1;
            if (opts.time_kernels) {
                TKV_CUDA_CHECK(cudaEventRecord(g1, cs_));
                model_.add_timed(g0, g1, -double(ctx_rows) * 2 * L * kvd * (dtype_size(in_dt) + oes));  // tagged gather
            }
        }
        if (M > 0) {
            FwdArgs fa;
            fa.M = M;
            fa.tokens = static_cast<const int32_t*>(ring.upload(tokens.data(), tokens.size() * 4, cs_));
            fa.pos = static_cast<const int32_t*>(ring.upload(pos.data(), pos.size() * 4, cs_));
            fa.pos64 = static_cast<const int64_t*>(ring.upload(pos64.data(), pos64.size() * 8, cs_));
            fa.n_seqs = int(seqs.size());
            fa.seqs = static_cast<const AttnSeq*>(ring.upload(seqs.data(), seqs.size() * sizeof(AttnSeq), cs_));
            fa.seqs_host = seqs.data();
            fa.mode = 0;
            fa.ctx_k = ctx_k;
            fa.ctx_v = ctx_v;
            fa.ctx_rows = max_ctx_rows;
            if (d_segs_s) {
                fa.gather_pool = pool_.base();
                fa.gather_page_bytes = P;
                fa.gather_pool_bytes = P * size_t(pool_.n_pages());
                fa.seq_seg0 = static_cast<const int32_t*>(ring.upload(seq_seg0.data(), seq_seg0.size() * 4, cs_));
                fa.gather_pages = d_pages_s;
                fa.gather_segs = d_segs_s;
                fa.gather_n_segs = int(segs.size());
                fa.gather_rows = ctx_rows;
                fa.gather_in = in_dt_s;
                fa.gather_chunks = d_chunks_s;
                fa.gather_n_chunks = n_chunks_s;
                static const bool paged_v = [] {  // TKV_PAGED_V=0 / TKV_PAGED_K=0: gathered slab (A/B)
                    const char* e = std::getenv("TKV_PAGED_V");
                    return !(e && std::string(e) == "0");
                }();
                fa.paged_v = paged_v;
                static const bool paged_k = [] {
                    const char* e = std::getenv("TKV_PAGED_K");
                    return !(e && std::string(e) == "0");
                }();
                fa.paged_k = paged_k;
            }
            std::vector<cudaEvent_t> layer_ready;
            if (layered_env && stream_ctx && !peering && opts.engine == CopyEngine::dma && group_first == wi &&
                !lchunk_ev[wi].empty() && lchunk_ev[wi][0]) {
                layer_ready.resize(size_t(L));
                for (int l = 0; l < L; ++l) layer_ready[size_t(l)] = lchunk_ev[wi][size_t(l / kLayerChunk)];
                fa.layer_ready = layer_ready.data();
            }
            fa.logit_rows = static_cast<const int32_t*>(ring.upload(logit_rows.data(), logit_rows.size() * 4, cs_));
            fa.logit_rows_host = logit_rows.data();
            fa.n_logit_rows = int(logit_rows.size());
            fa.logits_out = d_logits;
            fa.argmax_out = d_argmax + plan.windows[group_first].begin;  // compacted per group; remapped below
            R.meta_bytes += tokens.size() * 16 + seqs.size() * sizeof(AttnSeq) + logit_rows.size() * 4;
            hp_tick(hp_rest);
            model_.set_timing(opts.time_kernels);
            model_.forward(fa, cs_);
            R.launches += model_.launches();
            hp_tick(hp_fwd);
            if (opts.keep_logits) {
                for (size_t k = 0; k < seq_query.size(); ++k)
                    TKV_CUDA_CHECK(cudaMemcpyAsync(logits_host.data() + seq_query[k] * vp, d_logits + k * vp,
                                                   sizeof(float) * vp, cudaMemcpyDeviceToHost, cs_));
                TKV_CUDA_CHECK(cudaStreamSynchronize(cs_));
            }
        }
        cudaEvent_t ge = evp.get();
        TKV_CUDA_CHECK(cudaEventRecord(ge, cs_));
        for (size_t gw = group_first; gw <= wi; ++gw) win_end[gw] = ge;
        for (auto& [t, pg] : dropped) {
            auto it = t >= 0 ? published.find(t) : published.end();
            if (it != published.end() && it->second == pg) {  // peers must drain before the pages recycle
                launch_dir_revoke(*mesh_, t, cs_);
                published.erase(it);
            }
            pool_.release(pg, cs_);
        }
        // the k-th prefilling query of this group writes its argmax to d_argmax[first begin + k]
        for (size_t k = 0; k < seq_query.size(); ++k)
            R.argmax[seq_query[k]] = int32_t(plan.windows[group_first].begin + k);  // slot, resolved below
        dropped.clear();
        segs.clear(), page_ids.clear(), tokens.clear(), pos.clear(), logit_rows.clear(), pos64.clear();
        seqs.clear(), seq_query.clear(), seq_seg0.clear();
        ctx_rows = 0, M = 0;
        group_first = wi + 1;
    }
    // the batch's cache dies with it: every still-resident table's pages go back to the pool
    unwind.armed = false;
    for (auto& kv : published) launch_dir_revoke(*mesh_, kv.first, cs_);
    published.clear();
    for (auto& kv : resident) pool_.release(kv.second, cs_);
    resident.clear();
    R.host_ms = now_ms() - host0;
    hp_tick(hp_rest);
    if (host_prof)
        std::fprintf(stderr, "[tkv host] plan %.1f ms, copies %.1f ms, forward enqueue %.1f ms, rest %.1f ms (windows %zu)\n",
                     hp_plan, hp_copy, hp_fwd, hp_rest, plan.windows.size());
    const double tail0 = now_ms();
    TKV_CUDA_CHECK(cudaStreamSynchronize(ps_));
    TKV_CUDA_CHECK(cudaStreamSynchronize(ds_));
    TKV_CUDA_CHECK(cudaStreamSynchronize(xs_));
    TKV_CUDA_CHECK(cudaStreamSynchronize(cs_));
    const double tail1 = now_ms();
    if (peering) {
        unsigned long long st[2];
        TKV_CUDA_CHECK(cudaMemcpy(st, mesh_->stats(), sizeof(st), cudaMemcpyDeviceToHost));
        R.peer_bytes = st[0];
        R.peer_fallback_bytes = st[1];
    }
    std::vector<int32_t> am(queries.size());
    TKV_CUDA_CHECK(cudaMemcpy(am.data(), d_argmax, sizeof(int32_t) * queries.size(), cudaMemcpyDeviceToHost));
    for (auto& a : R.argmax)
        if (a >= 0) a = am[size_t(a)];
    R.ttft_ms.resize(plan.queries.size());
    R.window_end_ms.resize(plan.windows.size());
    for (size_t wi = 0; wi < plan.windows.size(); ++wi) R.window_end_ms[wi] = elapsed(t0, win_end[wi]);
    for (size_t qi = 0; qi < plan.queries.size(); ++qi) R.ttft_ms[qi] = R.window_end_ms[size_t(R.window_of[qi])];
    R.makespan_ms = R.window_end_ms.back();
    for (size_t i = 0; i < dspan.size(); ++i) {
        const double d = elapsed(dspan[i].first, dspan[i].second);
        R.copy_demand_ms += d;
        R.copy_busy_ms += d + elapsed(pspan[i].first, pspan[i].second);
        // per window: demand copies [start, end), compute(w) ready, window end (ms from submission)
        R.window_timeline.push_back({elapsed(t0, dspan[i].first), elapsed(t0, dspan[i].second),
                                     cstart[i] ? elapsed(t0, cstart[i]) : -1.0, R.window_end_ms[i]});
    }
    if (opts.time_kernels) model_.collect_timing(R.gemm_ms, R.gemm_flops, R.gather_ms, R.attn_ms, R.gather_bytes);
    if (opts.keep_logits) R.logits = std::move(logits_host);
    R.launches += model_.ring().launches() - ring_launches0;  // metadata copy kernels
    R.wall_ms = now_ms() - host0;
    if (host_prof)
        std::fprintf(stderr, "[tkv host] tail: sync %.1f ms, results %.1f ms; makespan %.1f, wall %.1f\n", tail1 - tail0,
                     now_ms() - tail1, R.makespan_ms, R.wall_ms);
    return R;
}

ServeResult Server::serve_nocache(const std::vector<ServeQuery>& queries, const ServeOptions& opts) {
    ServeResult R;
    if (queries.empty()) return R;
    if (table_tokens_.empty()) throw std::invalid_argument("serve_nocache needs set_table_tokens()");
    const ModelCfg& mc = model_.cfg();
    const int vp = mc.vocab_padded();
    EventPool evp;
    const double host0 = now_ms();
    cudaEvent_t t0 = evp.get();
    TKV_CUDA_CHECK(cudaEventRecord(t0, cs_));
    int n_bits = 0;
    for (const auto& q : queries)
        for (int t : q.tables) n_bits = std::max(n_bits, t + 1);
    std::vector<tablekv::QueryRecord> recs;
    for (const auto& q : queries) {
        auto r = tablekv::make_query_record(q.id, {}, q.tables, std::max(1, n_bits), int(q.suffix.size()));
        r.tables = q.tables;
        recs.push_back(std::move(r));
    }
    R.order = tablekv::serving_order(recs, opts.run);
    const size_t n = queries.size(), bc = size_t(opts.run.b_c);
    int max_pos = 1;
    for (const auto& q : queries) {
        long c = long(q.suffix.size()) + 1;
        for (int t : q.tables) c += long(table_tokens_[size_t(t)].size());
        max_pos = std::max<int>(max_pos, int(c));
    }
    model_.rope().ensure(max_pos);
    // Sub-batches in served order: at most kMaxRows prompt rows each (bounded activation workspace),
    // and consecutive tiny windows share one (the same kGroupRows grouping as the cached path); a
    // query's first token is ready when its sub-batch ends.
    constexpr long kMaxRows = 65536, kGroupRows = 1024;
    auto prompt_rows = [&](size_t qi) {
        const ServeQuery& q = queries[R.order[qi]];
        long len = long(q.suffix.size());
        for (int t : q.tables) len += long(table_tokens_[size_t(t)].size());
        return len;
    };
    std::vector<std::pair<size_t, size_t>> subs;  // [first, last) served indices
    {
        size_t a = 0;
        long rows = 0;
        for (size_t qi = 0; qi < n; ++qi) {
            const long len = prompt_rows(qi);
            if (qi > a && rows + len > kMaxRows) subs.push_back({a, qi}), a = qi, rows = 0;
            rows += len;
            const bool window_end = (qi + 1) % bc == 0 || qi + 1 == n;
            if (qi + 1 == n || (window_end && rows >= kGroupRows)) subs.push_back({a, qi + 1}), a = qi + 1, rows = 0;
        }
    }
    size_t max_sub = 1;
    for (const auto& sb : subs) max_sub = std::max(max_sub, sb.second - sb.first);
    int32_t* d_argmax = nullptr;
    float* d_logits = nullptr;
    ensure_out(n, max_sub * size_t(vp));
    d_argmax = argmax_buf_;
    d_logits = logits_buf_;
    std::vector<float> logits_host;
    if (opts.keep_logits) logits_host.resize(n * size_t(vp));
    R.window_of.assign(n, 0);
    R.argmax.assign(n, -1);
    std::vector<cudaEvent_t> win_end((n + bc - 1) / bc, nullptr);
    std::vector<cudaEvent_t> sub_end;
    std::vector<int> sub_of(n, -1);
    for (const auto& [qb, qe] : subs) {
        std::vector<int32_t> tokens, pos, group, logit_rows;
        std::vector<int64_t> pos64;
        std::vector<AttnSeq> seqs;
        std::vector<size_t> seq_query;
        int M = 0;
        for (size_t qi = qb; qi < qe; ++qi) {
            const ServeQuery& q = queries[R.order[qi]];
            R.window_of[qi] = int(qi / bc);
            sub_of[qi] = int(sub_end.size());
            if (q.suffix.empty()) continue;
            const int row0 = M;
            int p = 0;
            for (int t : q.tables) {
                for (int32_t tok : table_tokens_[size_t(t)]) {
                    tokens.push_back(tok);
                    group.push_back(group_of_[size_t(t)]);
                    pos.push_back(p);
                    pos64.push_back(p++);
                }
            }
            R.total_ctx_tokens += p;
            for (int32_t tok : q.suffix) {
                tokens.push_back(tok);
                group.push_back(-1);
                pos.push_back(p);
                pos64.push_back(p++);
            }
            M += p;
            seqs.push_back({row0, p, 0, 0});
            seq_query.push_back(qi);
            logit_rows.push_back(M - 1);
        }
        R.total_suffix_tokens += M;
        if (M > 0) {
            StagingRing& ring = model_.ring();
            FwdArgs fa;
            fa.M = M;
            fa.tokens = static_cast<const int32_t*>(ring.upload(tokens.data(), tokens.size() * 4, cs_));
            fa.pos = static_cast<const int32_t*>(ring.upload(pos.data(), pos.size() * 4, cs_));
            fa.pos64 = static_cast<const int64_t*>(ring.upload(pos64.data(), pos64.size() * 8, cs_));
            fa.group = static_cast<const int32_t*>(ring.upload(group.data(), group.size() * 4, cs_));
            fa.group_host = group.data();
            fa.n_seqs = int(seqs.size());
            fa.seqs = static_cast<const AttnSeq*>(ring.upload(seqs.data(), seqs.size() * sizeof(AttnSeq), cs_));
            fa.seqs_host = seqs.data();
            fa.mode = 1;
            fa.logit_rows = static_cast<const int32_t*>(ring.upload(logit_rows.data(), logit_rows.size() * 4, cs_));
            fa.logit_rows_host = logit_rows.data();
            fa.n_logit_rows = int(logit_rows.size());
            fa.logits_out = d_logits;
            fa.argmax_out = d_argmax + qb;  // the k-th prefilling query of the sub-batch -> slot qb + k
            R.meta_bytes += tokens.size() * 20 + seqs.size() * sizeof(AttnSeq) + logit_rows.size() * 4;
            model_.set_timing(opts.time_kernels);
            model_.forward(fa, cs_);
            R.launches += model_.launches();
            if (opts.keep_logits) {
                for (size_t k = 0; k < seq_query.size(); ++k)
                    TKV_CUDA_CHECK(cudaMemcpyAsync(logits_host.data() + seq_query[k] * vp, d_logits + k * vp,
                                                   sizeof(float) * vp, cudaMemcpyDeviceToHost, cs_));
                TKV_CUDA_CHECK(cudaStreamSynchronize(cs_));
            }
            for (size_t k = 0; k < seq_query.size(); ++k) R.argmax[seq_query[k]] = int32_t(qb + k);
        }
        sub_end.push_back(evp.get());
        TKV_CUDA_CHECK(cudaEventRecord(sub_end.back(), cs_));
        for (size_t qi = qb; qi < qe; ++qi) win_end[qi / bc] = sub_end.back();  // a window ends with its last sub-batch
    }
    R.host_ms = now_ms() - host0;
    TKV_CUDA_CHECK(cudaStreamSynchronize(cs_));
    std::vector<int32_t> am(n);
    TKV_CUDA_CHECK(cudaMemcpy(am.data(), d_argmax, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    for (auto& a : R.argmax)
        if (a >= 0) a = am[size_t(a)];
    R.window_end_ms.resize(win_end.size());
    for (size_t wi = 0; wi < win_end.size(); ++wi) R.window_end_ms[wi] = elapsed(t0, win_end[wi]);
    R.ttft_ms.resize(n);
    for (size_t qi = 0; qi < n; ++qi) R.ttft_ms[qi] = elapsed(t0, sub_end[size_t(sub_of[qi])]);
    R.makespan_ms = R.window_end_ms.back();
    if (opts.time_kernels) model_.collect_timing(R.gemm_ms, R.gemm_flops, R.gather_ms, R.attn_ms, R.gather_bytes);
    if (opts.keep_logits) R.logits = std::move(logits_host);
    return R;
}

}  // namespace tkv
