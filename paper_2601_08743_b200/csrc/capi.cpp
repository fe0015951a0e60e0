// C ABI of libtkv.so (include/tkv.h). Exceptions never cross this boundary: each entry point
// runs inside guard(), which maps tablekv::Error -> 1 + Errc, CUDA failures -> TKV_E_CUDA,
// bad arguments -> TKV_E_INVALID and keeps the message for tkv_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_map>

#include <json.hpp>

#include "cuda/common.cuh"
#include "cuda/gemm_tc.cuh"
#include "cuda/model.cuh"
#include "cuda/runtime.cuh"
#include "cuda/serve.cuh"
#include "tablekv/engine.hpp"
#include "tkv.h"

using nlohmann::json;

struct tkv_engine {
    tablekv::Engine e;
};
struct tkv_trie {
    tablekv::TableTrie t;
};
struct tkv_cache {
    std::unique_ptr<tablekv::TieredCache> c;
};
struct tkv_model {
    int device = 0;
    std::unique_ptr<tkv::Model> m;
    cudaStream_t s = nullptr;
};
struct tkv_store {
    tkv_model* model = nullptr;
    std::unique_ptr<tkv::Arena> arena;
    std::unique_ptr<tkv::PagePool> pool;
    std::unique_ptr<tkv::Server> server;
    std::unique_ptr<tkv::PeerMesh> mesh;
    std::unordered_map<int, std::vector<int32_t>> held;  // peer_publish: table -> pages
    // last precompute: groups, tables, tokens, forwards, device ms, gemm ms, gemm flops, attention ms, launches
    std::array<double, 9> encode_stats{};
    bool encode_timed = false;  // CUDA-event timing of the next precompute's GEMM / attention launches
};

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return TKV_OK;
    } catch (const tablekv::Error& e) {
        g_err = e.what();
        return 1 + int(e.code());
    } catch (const tkv::CudaError& e) {
        g_err = e.what();
        return TKV_E_CUDA;
    } catch (const std::invalid_argument& e) {
        g_err = std::string("invalid argument: ") + e.what();
        return TKV_E_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TKV_E_INTERNAL;
    } catch (...) {
        g_err = "unknown exception";
        return TKV_E_INTERNAL;
    }
}

void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

char* dup_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size() + 1);
    return p;
}

tablekv::EvictionPolicy policy_of(int p) {
    need(p >= 0 && p <= 2, "policy must be 0 (lru), 1 (fifo) or 2 (lfu)");
    return static_cast<tablekv::EvictionPolicy>(p);
}

tkv::DType dtype_of(int d) {
    need(d >= 0 && d <= 2, "dtype must be 0 (f32), 1 (bf16) or 2 (f64)");
    return static_cast<tkv::DType>(d);
}

tablekv::RunOptions run_options_json(const json& r) {
    tablekv::RunOptions o;
    o.rerank_on = r.value("rerank_on", true);
    o.pipeline_on = r.value("pipeline_on", true);
    o.capacity = r.value("capacity", size_t(8));
    o.policy = tablekv::parse_policy(r.value("policy", std::string("lru")));
    o.b_c = r.value("b_c", 100);
    o.b_m = r.value("b_m", 10);
    o.seed = r.value("seed", std::uint64_t(1));
    o.anchor = r.value("anchor", std::string("seeded")) == "fixed_first" ? tablekv::AnchorMode::fixed_first
                                                                         : tablekv::AnchorMode::seeded;
    return o;
}

tablekv::CostModel cost_json(const json& c) {
    tablekv::CostModel m;
    m.compute_per_token = c.value("compute_per_token", 0.01);
    m.load_per_token = c.value("load_per_token", 1.0);
    m.switch_overhead = c.value("switch_overhead", 5.0);
    return m;
}

json recs_json(const std::vector<tablekv::LoadRec>& v) {
    json a = json::array();
    for (const auto& r : v) a.push_back({{"table", r.table}, {"miss", r.miss}, {"evicted", r.evicted}, {"size", r.size}});
    return a;
}

json trace_json(const tablekv::Trace& tr) {
    json w = json::array();
    for (const auto& wt : tr.windows) {
        json e = json::array();
        for (const auto& q : wt.emergency) e.push_back(recs_json(q));
        w.push_back({{"boundary", recs_json(wt.boundary)}, {"prefetch", recs_json(wt.prefetch)}, {"emergency", e}});
    }
    return {{"windows", w}, {"compute", tr.compute}};
}

// metadata-only slow tier over token counts (the cache simulator's fake backend)
std::shared_ptr<tablekv::MemorySlowTier> meta_tier(const std::vector<int>& counts) {
    auto t = std::make_shared<tablekv::MemorySlowTier>();
    for (size_t i = 0; i < counts.size(); ++i) {
        tablekv::TableKV<float> kv;
        kv.table_id = int(i);
        kv.token_count = counts[i];
        t->put(std::move(kv));
    }
    return t;
}

tkv::ServeOptions serve_opts(const tkv_serve_options* o) {
    tkv::ServeOptions so;
    so.run.rerank_on = o->rerank_on != 0;
    so.run.pipeline_on = o->pipeline_on != 0;
    so.run.capacity = o->capacity;
    so.run.policy = policy_of(o->policy);
    so.run.b_c = o->b_c;
    so.run.b_m = o->b_m;
    so.run.seed = o->seed;
    so.run.anchor = o->fixed_anchor ? tablekv::AnchorMode::fixed_first : tablekv::AnchorMode::seeded;
    so.cost.compute_per_token = o->compute_per_token;
    so.cost.load_per_token = o->load_per_token;
    so.cost.switch_overhead = o->switch_overhead;
    so.engine = o->copy_engine ? tkv::CopyEngine::sm : tkv::CopyEngine::dma;
    so.sm_copy_ctas = std::max(1, o->sm_copy_ctas);
    so.time_kernels = o->time_kernels != 0;
    so.peer_fetch = o->peer_fetch != 0;
    so.peer_ctas = std::max(1, o->peer_ctas);
    return so;
}

json serve_result_json(const tkv::ServeResult& R) {
    json tr = json::array();
    for (const auto& t : R.trace) tr.push_back({t.window, t.kind, t.query, t.table, t.evicted, t.miss, t.bytes});
    return {{"order", R.order},
            {"ttft_ms", R.ttft_ms},
            {"argmax", R.argmax},
            {"window_of", R.window_of},
            {"window_end_ms", R.window_end_ms},
            {"window_timeline_ms", R.window_timeline},
            {"trace", tr},
            {"counters", {R.counters.hits, R.counters.misses, R.counters.swaps, R.counters.prefetch_loads}},
            {"h2d_bytes", R.h2d_bytes},
            {"meta_bytes", R.meta_bytes},
            {"copy_busy_ms", R.copy_busy_ms},
            {"h2d_demand_bytes", R.h2d_demand_bytes},
            {"peer_routed_bytes", R.peer_routed_bytes},
            {"peer_bytes", R.peer_bytes},
            {"peer_fallback_bytes", R.peer_fallback_bytes},
            {"copy_demand_ms", R.copy_demand_ms},
            {"makespan_ms", R.makespan_ms},
            {"host_ms", R.host_ms},
            {"wall_ms", R.wall_ms},
            {"launches", R.launches},
            {"gemm_ms", R.gemm_ms},
            {"gemm_flops", R.gemm_flops},
            {"gather_ms", R.gather_ms},
            {"gather_bytes", R.gather_bytes},
            {"attn_ms", R.attn_ms},
            {"ctx_tokens", R.total_ctx_tokens},
            {"suffix_tokens", R.total_suffix_tokens}};
}

void set_device(int d) { TKV_CUDA_CHECK(cudaSetDevice(d)); }

}  // namespace

extern "C" {

int tkv_version(void) { return 1; }

size_t tkv_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        const size_t n = std::min(cap - 1, g_err.size());
        std::memcpy(buf, g_err.data(), n);
        buf[n] = '\0';
    }
    return g_err.size();
}

const char* tkv_status_name(int status) {
    if (status == TKV_OK) return "ok";
    if (status == TKV_E_CUDA) return "CudaError";
    if (status == TKV_E_INVALID) return "InvalidArgument";
    if (status == TKV_E_INTERNAL) return "InternalError";
    if (status >= 1 && status <= 18) return tablekv::errc_name(static_cast<tablekv::Errc>(status - 1));
    return "UnknownStatus";
}

void tkv_free(void* p) { std::free(p); }

// ------------------------------------------------------------------ engine
int tkv_engine_create(const char* schema_path, int break_cycles, tkv_engine** out) {
    return guard([&] {
        need(schema_path && out, "null argument");
        tablekv::EngineOptions o;
        o.schema_path = schema_path;
        o.topo_mode = break_cycles ? tablekv::TopoMode::break_cycles : tablekv::TopoMode::strict;
        *out = new tkv_engine{tablekv::build_engine(o)};
    });
}

int tkv_engine_create_json(const char* corpus_json, int break_cycles, tkv_engine** out) {
    return guard([&] {
        need(corpus_json && out, "null argument");
        tablekv::EngineOptions o;
        o.topo_mode = break_cycles ? tablekv::TopoMode::break_cycles : tablekv::TopoMode::strict;
        *out = new tkv_engine{tablekv::build_engine_from_corpus(tablekv::parse_schema_corpus(corpus_json), o)};
    });
}

void tkv_engine_destroy(tkv_engine* e) { delete e; }

int tkv_engine_info_json(const tkv_engine* h, char** out) {
    return guard([&] {
        need(h && out, "null argument");
        const auto& e = h->e;
        json groups = json::array(), edges = json::array(), removed = json::array();
        for (const auto& g : e.plan.groups) groups.push_back({{"tables", g.tables}, {"offsets", g.offsets}});
        for (int u = 0; u < e.graph.node_count; ++u)
            for (int v : e.graph.out_edges[size_t(u)]) edges.push_back({u, v});
        for (const auto& [u, v] : e.topo.removed_edges) removed.push_back({u, v});
        json j = {{"vocab_size", e.tokenizer.vocab_size()}, {"vocab_hash", e.tokenizer.vocab_hash()},
                  {"topo_order", e.topo.order},           {"removed_edges", removed},
                  {"groups", groups},                     {"group_of", e.plan.group_of},
                  {"local_offset", e.local_offset},       {"table_tokens", e.table_tokens},
                  {"serialized", e.serialized},           {"edges", edges},
                  {"manifest", json::parse(tablekv::manifest_json(e))}};
        *out = dup_string(j.dump());
    });
}

int tkv_analyze_json(const tkv_engine* h, const char* query_id, const char* text, char** out) {
    return guard([&] {
        need(h && text && out, "null argument");
        const auto q = tablekv::analyze_query(h->e, query_id ? query_id : "", text);
        json spans = json::array();
        for (const auto& s : q.spans) spans.push_back({s.table_id, s.start, s.end});
        json j = {{"tokens", q.tokens},
                  {"spans", spans},
                  {"match_order", q.match_order},
                  {"remainder", q.remainder},
                  {"assembly_order", tablekv::assembly_order(h->e, q.match_order)},
                  {"record_tables", q.record.tables},
                  {"query_token_count", q.record.query_token_count}};
        *out = dup_string(j.dump());
    });
}

int tkv_check_manifest(const tkv_engine* h, const char* dir) {
    return guard([&] {
        need(h && dir, "null argument");
        tablekv::check_manifest(h->e, dir);
    });
}

int tkv_run_workload_json(const tkv_engine* h, const char* workload_path, const char* options_json, const char* kv_dir,
                          char** out) {
    return guard([&] {
        need(h && workload_path && out, "null argument");
        const json o = options_json ? json::parse(options_json) : json::object();
        std::shared_ptr<tablekv::SlowTier> slow;
        if (kv_dir && *kv_dir) {
            slow = std::make_shared<tablekv::FileSlowTier>(kv_dir);
        } else {
            std::vector<int> counts;
            for (const auto& t : h->e.table_tokens) counts.push_back(int(t.size()));
            slow = meta_tier(counts);
        }
        const auto rep = tablekv::run_workload(h->e, tablekv::load_workload(workload_path), run_options_json(o),
                                               cost_json(o.value("cost", json::object())), slow);
        *out = dup_string(rep.to_json());
    });
}

// ------------------------------------------------------------------ trie
int tkv_trie_create(tkv_trie** out) {
    return guard([&] {
        need(out, "null argument");
        *out = new tkv_trie{};
    });
}

void tkv_trie_destroy(tkv_trie* t) { delete t; }

int tkv_trie_insert(tkv_trie* t, const int32_t* tokens, size_t n, int table_id, uint64_t handle) {
    return guard([&] {
        need(t && (tokens || n == 0), "null argument");
        t->t.insert(std::span<const tablekv::TokenId>(tokens, n), table_id, handle);
    });
}

int tkv_trie_query(const tkv_trie* t, const int32_t* tokens, size_t n, size_t start, int* found, size_t* next,
                   int* table_id, uint64_t* handle) {
    return guard([&] {
        need(t && (tokens || n == 0), "null argument");
        const auto r = t->t.query(std::span<const tablekv::TokenId>(tokens, n), start);
        if (found) *found = r.found;
        if (next) *next = r.next;
        if (table_id) *table_id = r.table_id;
        if (handle) *handle = r.handle;
    });
}

int tkv_trie_match_all(const tkv_trie* t, const int32_t* tokens, size_t n, int64_t* spans_out, size_t cap, size_t* n_spans,
                       uint64_t* node_visits) {
    return guard([&] {
        need(t && (tokens || n == 0), "null argument");
        tablekv::MatchStats st;
        const auto sp = t->t.match_all(std::span<const tablekv::TokenId>(tokens, n), &st);
        if (n_spans) *n_spans = sp.size();
        if (node_visits) *node_visits = st.node_visits;
        for (size_t i = 0; i < sp.size() && i < cap && spans_out; ++i) {
            spans_out[3 * i] = sp[i].table_id;
            spans_out[3 * i + 1] = int64_t(sp[i].start);
            spans_out[3 * i + 2] = int64_t(sp[i].end);
        }
    });
}

// ------------------------------------------------------------------ rerank
int tkv_rerank(const uint64_t* inc, size_t n, size_t words, uint64_t seed, int fixed_first, int threads, uint64_t* perm) {
    return guard([&] {
        need(inc && perm, "null argument");
        const auto p = tablekv::rerank_packed(inc, n, words, seed,
                                              fixed_first ? tablekv::AnchorMode::fixed_first : tablekv::AnchorMode::seeded,
                                              threads);
        std::copy(p.begin(), p.end(), perm);
    });
}

int tkv_rerank_device(int device, const uint64_t* inc, size_t n, size_t words, uint64_t seed, int fixed_first,
                      uint64_t* perm) {
    return guard([&] {
        need(inc && perm, "null argument");
        set_device(device);
        static thread_local std::unordered_map<int, cudaStream_t> streams;  // one per device, kept
        cudaStream_t& st = streams[device];
        if (!st) TKV_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const std::vector<size_t> p = tkv::rerank_device(
            inc, n, words, seed, fixed_first ? tablekv::AnchorMode::fixed_first : tablekv::AnchorMode::seeded, st);
        std::copy(p.begin(), p.end(), perm);
    });
}

int tkv_rerank_device_stats(double* out, int n) {
    return guard([&] {
        need(out || n == 0, "null argument");
        const tkv::RerankStats st = tkv::last_rerank_stats();
        const double v[5] = {st.classes_ms, st.kernel_ms, st.total_ms, st.n_classes, double(st.cluster)};
        for (int i = 0; i < n && i < 5; ++i) out[i] = v[i];
    });
}

// ------------------------------------------------------------------ cache
int tkv_cache_create(size_t capacity, int policy, const int32_t* counts, size_t n, tkv_cache** out) {
    return guard([&] {
        need(out && (counts || n == 0), "null argument");
        *out = new tkv_cache{std::make_unique<tablekv::TieredCache>(capacity, policy_of(policy),
                                                                    meta_tier(std::vector<int>(counts, counts + n)))};
    });
}

void tkv_cache_destroy(tkv_cache* c) { delete c; }

int tkv_cache_get(tkv_cache* c, int id, int* hit, int* evicted) {
    return guard([&] {
        need(c, "null argument");
        const auto r = c->c->get(id);
        if (hit) *hit = r.hit;
        if (evicted) *evicted = r.evicted_id;
    });
}

int tkv_cache_prefetch(tkv_cache* c, const int32_t* ids, size_t n, int32_t* admitted, size_t* n_admitted) {
    return guard([&] {
        need(c && (ids || n == 0), "null argument");
        const auto a = c->c->prefetch(std::span<const int>(ids, n));
        if (n_admitted) *n_admitted = a.size();
        if (admitted) std::copy(a.begin(), a.end(), admitted);
    });
}

int tkv_cache_evict_candidate(const tkv_cache* c, int* id) {
    return guard([&] {
        need(c && id, "null argument");
        *id = c->c->evict_candidate();
    });
}

int tkv_cache_state(const tkv_cache* c, uint64_t counters[4], int32_t* residents, size_t cap, size_t* n) {
    return guard([&] {
        need(c, "null argument");
        const auto& k = c->c->counters();
        if (counters) counters[0] = k.hits, counters[1] = k.misses, counters[2] = k.swaps, counters[3] = k.prefetch_loads;
        const auto r = c->c->residents();
        if (n) *n = r.size();
        for (size_t i = 0; i < r.size() && i < cap && residents; ++i) residents[i] = r[i];
    });
}

// ------------------------------------------------------------------ pipeline
int tkv_run_batch_json(const char* input_json, char** output_json) {
    return guard([&] {
        need(input_json && output_json, "null argument");
        const json in = json::parse(input_json);
        const std::vector<int> counts = in.at("token_counts");
        auto slow = meta_tier(counts);
        std::vector<tablekv::QueryRecord> recs;
        for (const auto& q : in.at("queries")) {
            std::vector<int> tables = q.at("tables");
            auto r = tablekv::make_query_record(q.at("id"), {}, tables, int(counts.size()), q.at("query_tokens"));
            r.tables = tables;
            recs.push_back(std::move(r));
        }
        json out = json::object();
        for (const auto& r : in.at("runs")) {
            const auto opts = run_options_json(r);
            const auto cost = cost_json(r.value("cost", json::object()));
            json d;
            const auto order = tablekv::serving_order(recs, opts);
            d["order"] = order;
            std::vector<tablekv::SimQuery> sims;
            for (size_t i : order) sims.push_back({recs[i].query_id, recs[i].tables, recs[i].query_token_count});
            const auto plan = tablekv::schedule(sims, opts.b_c, opts.b_m);
            json wins = json::array();
            for (const auto& w : plan.windows)
                wins.push_back({{"begin", w.begin}, {"end", w.end}, {"demand", w.demand}, {"prefetch", w.prefetch}});
            d["plan"] = {{"windows", wins}};
            {
                tablekv::TieredCache c(opts.capacity, opts.policy, slow);
                d["trace"] = trace_json(tablekv::build_trace(plan, cost, c));
                d["final_residents"] = c.residents();
            }
            d["report"] = json::parse(tablekv::run_batch(recs, opts, cost, slow).to_json());
            tablekv::TieredCache c1(opts.capacity, opts.policy, slow), c2(opts.capacity, opts.policy, slow);
            d["report_overlapped"] = json::parse(tablekv::simulate(plan, cost, c1, tablekv::SimMode::overlapped).to_json());
            d["report_serial"] = json::parse(tablekv::simulate(plan, cost, c2, tablekv::SimMode::serial).to_json());
            out[r.at("name").get<std::string>()] = d;
        }
        *output_json = dup_string(out.dump());
    });
}

// ------------------------------------------------------------------ model
int tkv_model_create(int device, const tkv_model_config* c, tkv_model** out) {
    return guard([&] {
        need(c && out, "null argument");
        set_device(device);
        tkv::ModelCfg mc;
        mc.num_layers = c->num_layers;
        mc.num_heads = c->num_heads;
        mc.kv_heads = c->num_kv_heads > 0 ? c->num_kv_heads : c->num_heads;
        mc.head_dim = c->head_dim;
        mc.ffn = c->ffn_dim > 0 ? c->ffn_dim : 4 * c->num_heads * c->head_dim;
        mc.vocab = c->vocab_size;
        mc.rotary_base = c->rotary_base;
        mc.seed = c->weight_seed;
        mc.mlp = c->mlp;
        mc.norm = c->norm;
        mc.dtype = dtype_of(c->dtype);
        need(mc.num_layers > 0 && mc.num_heads > 0 && mc.head_dim > 0, "model dimensions must be positive");
        if (mc.dtype == tkv::DType::bf16) {
            need(mc.hidden() % 64 == 0 || mc.hidden() % 32 == 0, "bf16 models need hidden % 32 == 0");
            need(mc.kv_dim() % 32 == 0, "bf16 models need kv_heads*head_dim % 32 == 0");
            need(mc.ffn % 32 == 0, "bf16 models need ffn % 32 == 0");
        }
        auto h = std::make_unique<tkv_model>();
        h->device = device;
        TKV_CUDA_CHECK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
        h->m = std::make_unique<tkv::Model>(mc, h->s);
        *out = h.release();
    });
}

void tkv_model_destroy(tkv_model* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    m->m.reset();
    cudaStreamDestroy(m->s);
    delete m;
}

int tkv_model_set_attention(tkv_model* m, int impl) {
    return guard([&] {
        need(m && (impl == 0 || impl == 1), "impl must be 0 (tcgen05) or 1 (mma.sync)");
        m->m->set_attention_impl(impl);
    });
}

int tkv_model_weights(tkv_model* m, int which, void* host_out, size_t bytes) {
    return guard([&] {
        need(m && host_out, "null argument");
        set_device(m->device);
        const auto& c = m->m->cfg();
        const size_t es = tkv::dtype_size(c.dtype);
        const size_t rows = which == 0 ? size_t(c.vocab) : size_t(c.dtype == tkv::DType::bf16 ? c.vocab_padded() : c.vocab);
        need(bytes == rows * size_t(c.hidden()) * es, "byte count does not match the weight tensor");
        TKV_CUDA_CHECK(cudaMemcpy(host_out, which == 0 ? m->m->embedding() : m->m->head(), bytes, cudaMemcpyDeviceToHost));
    });
}

int tkv_model_forward(tkv_model* m, const int32_t* tokens, const int32_t* positions, const int32_t* groups, int n, int mode,
                      const void* ctx_k, const void* ctx_v, int n_ctx, void* hidden_out, void* kraw_out, void* v_out,
                      float* logits_out, int32_t* argmax_out) {
    return guard([&] {
        need(m && tokens && n > 0, "need a model and at least one token");
        need(mode == 0 || mode == 1, "mode must be 0 or 1");
        need(mode == 1 || n_ctx == 0 || (ctx_k && ctx_v), "mode 0 with n_ctx > 0 needs ctx_k / ctx_v");
        need(mode == 0 || groups, "mode 1 needs group ids");
        set_device(m->device);
        const auto& c = m->m->cfg();
        for (int i = 0; i < n; ++i)
            if (tokens[i] < 0 || tokens[i] >= c.vocab)
                throw tablekv::Error(tablekv::Errc::bad_config, "token id " + std::to_string(tokens[i]) + " outside vocabulary");
        std::vector<int64_t> pos;
        if (positions) pos.assign(positions, positions + n);
        tkv::HostFwd h;
        h.tokens = tokens;
        h.positions = positions ? pos.data() : nullptr;
        h.groups = groups;
        h.n = n;
        h.mode = mode;
        h.n_ctx = mode == 0 ? n_ctx : 0;
        h.ctx_k = ctx_k;
        h.ctx_v = ctx_v;
        h.hidden = hidden_out;
        h.kraw = kraw_out;
        h.v = v_out;
        h.logits = logits_out;
        h.argmax = argmax_out;
        tkv::forward_host(*m->m, m->s, h);
    });
}

// ------------------------------------------------------------------ store
int tkv_store_create(tkv_model* m, size_t page_bytes, int n_pages, tkv_store** out) {
    return guard([&] {
        need(m && out && page_bytes > 0 && n_pages > 0, "need a model, page size and page count");
        set_device(m->device);
        auto s = std::make_unique<tkv_store>();
        s->model = m;
        s->arena = std::make_unique<tkv::Arena>();
        s->pool = std::make_unique<tkv::PagePool>(page_bytes, n_pages);
        s->server = std::make_unique<tkv::Server>(*m->m, *s->arena, *s->pool);
        *out = s.release();
    });
}

void tkv_store_destroy(tkv_store* s) {
    if (!s) return;
    cudaSetDevice(s->model->device);
    s->server.reset();
    for (auto& kv : s->held) {
        if (s->mesh) tkv::launch_dir_revoke(*s->mesh, kv.first, s->model->s);
        s->pool->release(kv.second, s->model->s);
    }
    cudaStreamSynchronize(s->model->s);
    s->mesh.reset();
    s->pool.reset();
    s->arena.reset();
    delete s;
}

int tkv_store_put(tkv_store* s, int table_id, int tokens, int local_offset, int dtype, const void* payload) {
    return guard([&] {
        need(s && payload && tokens > 0, "need a store, payload and tokens > 0");
        const auto& c = s->model->m->cfg();
        const auto dt = dtype_of(dtype);
        need(dt != tkv::DType::f64, "arena images are f32 or bf16");
        s->arena->put(table_id, tokens, c.num_layers, c.kv_dim(), local_offset, dt, payload);
    });
}

int tkv_store_load_kv_file(tkv_store* s, const char* path, int* table_id) {
    return guard([&] {
        need(s && path, "null argument");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw tablekv::Error(tablekv::Errc::io_error, std::string("cannot open KV file: ") + path);
        const std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        if (bytes.size() < 24) throw tablekv::Error(tablekv::Errc::io_error, std::string("truncated KV file: ") + path);
        const auto* p = reinterpret_cast<const unsigned char*>(bytes.data());
        int f[6];
        for (int i = 0; i < 6; ++i) f[i] = int(tablekv::kvfile::rd32(p + 4 * i));
        const auto& c = s->model->m->cfg();
        const size_t per_layer = size_t(f[1]) * size_t(f[3]) * size_t(f[4]);
        if (bytes.size() != 24 + 8 * per_layer * size_t(f[2]))
            throw tablekv::Error(tablekv::Errc::io_error, std::string("KV file size mismatch: ") + path);
        if (f[2] != c.num_layers || f[3] * f[4] != c.kv_dim())
            throw tablekv::Error(tablekv::Errc::dimension_mismatch, "KV block shape does not match the model");
        s->arena->put(f[0], f[1], f[2], f[3] * f[4], f[5], tkv::DType::f32, bytes.data() + 24);
        if (table_id) *table_id = f[0];
    });
}

int tkv_store_load_dir(tkv_store* s, const char* dir, const tkv_engine* e, int threads, int* n_loaded) {
    return guard([&] {
        need(s && dir, "null argument");
        namespace fs = std::filesystem;
        if (e) tablekv::check_manifest(e->e, dir);  // engine.cpp:114-131: model/tokenizer must match
        const auto& c = s->model->m->cfg();
        struct Job {
            fs::path path;
            const tkv::TableImage* img;
        };
        std::vector<Job> jobs;
        std::error_code ec;
        for (const auto& ent : fs::directory_iterator(dir, ec)) {
            const auto ext = ent.path().extension().string();
            if (ext != ".kv" && ext != ".kvb") continue;
            const tkv::DType dt = ext == ".kv" ? tkv::DType::f32 : tkv::DType::bf16;
            std::ifstream in(ent.path(), std::ios::binary);
            unsigned char h[24];
            if (!in.read(reinterpret_cast<char*>(h), 24))
                throw tablekv::Error(tablekv::Errc::io_error, "truncated KV file: " + ent.path().string());
            int f[6];
            for (int i = 0; i < 6; ++i) f[i] = int(tablekv::kvfile::rd32(h + 4 * i));
            const size_t payload = size_t(2) * f[2] * f[1] * f[3] * f[4] * tkv::dtype_size(dt);
            if (fs::file_size(ent.path()) != 24 + payload)
                throw tablekv::Error(tablekv::Errc::io_error, "KV file size mismatch: " + ent.path().string());
            if (f[2] != c.num_layers || f[3] * f[4] != c.kv_dim())
                throw tablekv::Error(tablekv::Errc::dimension_mismatch, "KV block shape does not match the model");
            if (s->arena->find(f[0])) continue;  // already resident in the arena
            // reserve pinned space now (the arena is single-writer), fill it from the file below
            jobs.push_back({ent.path(), &s->arena->put(f[0], f[1], f[2], f[3] * f[4], f[5], dt, nullptr)});
        }
        if (ec) throw tablekv::Error(tablekv::Errc::io_error, "cannot list " + std::string(dir));
        // file bytes go straight into pinned memory (no staging copy), files spread over threads
        const size_t n_thr = std::max<size_t>(1, std::min<size_t>(jobs.size(), threads > 0 ? size_t(threads) : 8));
        std::vector<std::exception_ptr> errs(n_thr);
        auto work = [&](size_t w) {
            try {
                for (size_t i = w; i < jobs.size(); i += n_thr) {
                    std::ifstream in(jobs[i].path, std::ios::binary);
                    in.seekg(24);
                    if (!in.read(reinterpret_cast<char*>(jobs[i].img->host), std::streamsize(jobs[i].img->bytes)))
                        throw tablekv::Error(tablekv::Errc::io_error, "short read on " + jobs[i].path.string());
                }
            } catch (...) {
                errs[w] = std::current_exception();
            }
        };
        std::vector<std::thread> pool;
        for (size_t w = 1; w < n_thr; ++w) pool.emplace_back(work, w);
        work(0);
        for (auto& t : pool) t.join();
        for (auto& ep : errs)
            if (ep) std::rethrow_exception(ep);
        if (n_loaded) *n_loaded = int(jobs.size());
    });
}

int tkv_store_bind_engine(tkv_store* s, const tkv_engine* e) {
    return guard([&] {
        need(s && e, "null argument");
        std::vector<std::vector<int32_t>> tt(e->e.table_tokens.begin(), e->e.table_tokens.end());
        s->server->set_table_tokens(std::move(tt), e->e.plan.group_of);
    });
}

// Offline encode (precompute_corpus, engine.cpp:83-112; encode_group, attention.hpp:254-294) on
// the GPU. Groups are packed into block-causal mode-1 forwards: one sequence per group at its
// local positions 0..n-1 (encode_group's single causal block), up to TKV_ENCODE_ROWS (16384)
// tokens per forward, groups taken largest first so each forward's attention items are alike.
// Every row's result is independent of what else shares its forward (row-wise GEMM tiles,
// per-sequence attention), so the images equal one forward per group. Each table's raw K and V
// go from the forward's [L][M][kv_dim] outputs straight into its pinned arena image by one 2-D
// copy each (no host staging); .kv / .kvb files are written from the images afterwards.
int tkv_store_precompute(tkv_store* s, const tkv_engine* eh, const char* out_dir) {
    return guard([&] {
        need(s && eh, "null argument");
        namespace fs = std::filesystem;
        const auto& e = eh->e;
        tkv_model* m = s->model;
        set_device(m->device);
        tkv::Model& model = *m->m;
        const auto& c = model.cfg();
        const int L = c.num_layers, kvd = c.kv_dim();
        const size_t es = tkv::dtype_size(c.dtype);
        const size_t row = size_t(kvd) * es;
        need(c.dtype != tkv::DType::f64, "precompute stores f32 or bf16 images");
        const tkv::DType img_dt = c.dtype;
        fs::path tmp;
        if (out_dir) {
            tmp = fs::path(std::string(out_dir) + ".tmp");
            std::error_code ec;
            fs::remove_all(tmp, ec);
            if (!fs::create_directories(tmp)) throw tablekv::Error(tablekv::Errc::io_error, "cannot create " + tmp.string());
        }
        std::vector<int> gsz(e.plan.groups.size(), 0), gorder(e.plan.groups.size());
        for (size_t gi = 0; gi < e.plan.groups.size(); ++gi) {
            for (int t : e.plan.groups[gi].tables) {
                if (e.table_tokens[size_t(t)].empty())
                    throw tablekv::Error(tablekv::Errc::empty_group, "table " + std::to_string(t) + " has no tokens");
                gsz[gi] += int(e.table_tokens[size_t(t)].size());
            }
        }
        std::iota(gorder.begin(), gorder.end(), 0);
        std::stable_sort(gorder.begin(), gorder.end(), [&](int x, int y) { return gsz[size_t(x)] > gsz[size_t(y)]; });
        static const int kRows = [] {
            const char* v = std::getenv("TKV_ENCODE_ROWS");
            return v ? std::max(1, std::atoi(v)) : 16384;
        }();
        std::vector<std::vector<int>> batches;
        for (size_t i = 0, rows = 0; i < gorder.size(); ++i) {
            const int gs = gsz[size_t(gorder[i])];
            if (batches.empty() || rows + size_t(gs) > size_t(kRows)) batches.emplace_back(), rows = 0;
            batches.back().push_back(gorder[i]);
            rows += size_t(gs);
        }
        int max_rows = 1;
        for (const auto& bt : batches) {
            int r = 0;
            for (int gi : bt) r += gsz[size_t(gi)];
            max_rows = std::max(max_rows, r);
        }
        cudaStream_t st = m->s;
        void *dk = nullptr, *dv = nullptr;
        TKV_CUDA_CHECK(cudaMalloc(&dk, size_t(L) * max_rows * row));
        struct Free {
            void*& a;
            void*& b;
            ~Free() {
                if (a) cudaFree(a);
                if (b) cudaFree(b);
            }
        } freer{dk, dv};
        TKV_CUDA_CHECK(cudaMalloc(&dv, size_t(L) * max_rows * row));
        cudaEvent_t e0, e1;
        TKV_CUDA_CHECK(cudaEventCreate(&e0));
        TKV_CUDA_CHECK(cudaEventCreate(&e1));
        double gemm_ms = 0, gemm_fl = 0, gath_ms = 0, attn_ms = 0, gath_b = 0;
        model.set_timing(s->encode_timed);
        long launches = 0, tokens_total = 0, tables_total = 0;
        TKV_CUDA_CHECK(cudaEventRecord(e0, st));
        tkv::StagingRing& ring = model.ring();
        for (const auto& bt : batches) {
            std::vector<int32_t> toks, pos, grp;
            std::vector<tkv::AttnSeq> seqs;
            for (int gi : bt) {
                const int row0 = int(toks.size());
                for (int t : e.plan.groups[size_t(gi)].tables)
                    toks.insert(toks.end(), e.table_tokens[size_t(t)].begin(), e.table_tokens[size_t(t)].end());
                const int n = int(toks.size()) - row0;
                for (int i = 0; i < n; ++i) pos.push_back(i), grp.push_back(0);
                seqs.push_back({row0, n, 0, 0});
            }
            const int M = int(toks.size());
            std::vector<int64_t> pos64(pos.begin(), pos.end());
            int max_pos = 0;
            for (int gi : bt) max_pos = std::max(max_pos, gsz[size_t(gi)]);
            model.rope().ensure(max_pos + 2);
            tkv::FwdArgs fa;
            fa.M = M;
            fa.tokens = static_cast<const int32_t*>(ring.upload(toks.data(), toks.size() * 4, st));
            fa.pos = static_cast<const int32_t*>(ring.upload(pos.data(), pos.size() * 4, st));
            fa.pos64 = static_cast<const int64_t*>(ring.upload(pos64.data(), pos64.size() * 8, st));
            fa.group = static_cast<const int32_t*>(ring.upload(grp.data(), grp.size() * 4, st));
            fa.group_host = grp.data();
            fa.n_seqs = int(seqs.size());
            fa.seqs = static_cast<const tkv::AttnSeq*>(ring.upload(seqs.data(), seqs.size() * sizeof(tkv::AttnSeq), st));
            fa.seqs_host = seqs.data();
            fa.mode = 1;
            fa.kraw_out = dk;
            fa.v_out = dv;
            model.forward(fa, st);
            launches += model.launches();
            tokens_total += M;
            // each table's rows [row0 + off, +T) of every layer -> its image ([K: L][T] then [V: L][T])
            for (size_t si = 0; si < bt.size(); ++si) {
                const auto& g = e.plan.groups[size_t(bt[si])];
                for (size_t i = 0; i < g.tables.size(); ++i) {
                    const int t = g.tables[i], off = g.offsets[i], T = int(e.table_tokens[size_t(t)].size());
                    const tkv::TableImage* img = s->arena->find(t);
                    if (img && (img->dtype != img_dt || img->tokens != T || img->layers != L || img->kv_dim != kvd))
                        continue;  // a loaded image of another format stays as it is
                    if (!img) img = &s->arena->put(t, T, L, kvd, off, img_dt, nullptr);
                    const size_t src0 = (size_t(seqs[si].q_row0) + size_t(off)) * row;
                    for (int kvi = 0; kvi < 2; ++kvi)
                        TKV_CUDA_CHECK(cudaMemcpy2DAsync(img->host + size_t(kvi) * L * T * row, size_t(T) * row,
                                                         static_cast<const uint8_t*>(kvi ? dv : dk) + src0, size_t(M) * row,
                                                         size_t(T) * row, size_t(L), cudaMemcpyDeviceToHost, st));
                    ++tables_total;
                }
            }
            // the host vectors above back the staging uploads and group_host: drain before reuse
            TKV_CUDA_CHECK(cudaStreamSynchronize(st));
        }
        TKV_CUDA_CHECK(cudaEventRecord(e1, st));
        TKV_CUDA_CHECK(cudaEventSynchronize(e1));
        float ms = 0;
        TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (s->encode_timed) model.collect_timing(gemm_ms, gemm_fl, gath_ms, attn_ms, gath_b);
        model.set_timing(false);
        s->encode_stats = {double(e.plan.groups.size()), double(tables_total), double(tokens_total), double(batches.size()),
                           double(ms), gemm_ms, gemm_fl, attn_ms, double(launches)};
        if (out_dir) {
            for (const auto& g : e.plan.groups)
                for (int t : g.tables) {
                    const tkv::TableImage* img = s->arena->find(t);
                    if (!img || img->dtype != img_dt) continue;
                    std::string file;
                    for (int fld : {t, img->tokens, L, c.kv_heads, c.head_dim, img->local_offset})
                        tablekv::kvfile::le32(file, std::uint32_t(fld));
                    file.append(reinterpret_cast<const char*>(img->host), img->bytes);
                    const auto name = std::to_string(t) + (img_dt == tkv::DType::f32 ? ".kv" : ".kvb");
                    std::ofstream of(tmp / name, std::ios::binary);
                    of.write(file.data(), std::streamsize(file.size()));
                    if (!of) throw tablekv::Error(tablekv::Errc::io_error, "short write on " + (tmp / name).string());
                }
            std::ofstream mf(tmp / "manifest.json", std::ios::binary);
            mf << tablekv::manifest_json(e);
            mf.close();
            std::error_code ec;
            fs::remove_all(out_dir, ec);
            fs::rename(tmp, out_dir);
        }
    });
}

int tkv_store_precompute_stats(const tkv_store* s, int timed_next, double* out, int n) {
    return guard([&] {
        need(s != nullptr, "null argument");
        const_cast<tkv_store*>(s)->encode_timed = timed_next != 0;
        for (int i = 0; out && i < n && i < int(s->encode_stats.size()); ++i) out[i] = s->encode_stats[size_t(i)];
    });
}

int tkv_store_fetch(tkv_store* s, int table_id, int copy_engine, void* host_out, size_t bytes) {
    return guard([&] {
        need(s && host_out, "null argument");
        set_device(s->model->device);
        const tkv::TableImage* img = s->arena->find(table_id);
        if (!img) throw tablekv::Error(tablekv::Errc::unknown_table, "table " + std::to_string(table_id) + " not in the arena");
        need(bytes == img->bytes, "byte count does not match the table image");
        const size_t P = s->pool->page_bytes();
        cudaStream_t st = s->model->s;
        auto pages = s->pool->alloc(int((img->bytes + P - 1) / P));
        tkv::copy_table_to_pages(*img, *s->pool, pages, copy_engine ? tkv::CopyEngine::sm : tkv::CopyEngine::dma, 16, st);
        for (size_t i = 0; i * P < img->bytes; ++i)
            TKV_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + i * P, s->pool->base() + size_t(pages[i]) * P,
                                           std::min(P, img->bytes - i * P), cudaMemcpyDeviceToHost, st));
        TKV_CUDA_CHECK(cudaStreamSynchronize(st));
        s->pool->release(pages, st);
    });
}

int tkv_store_assemble(tkv_store* s, const int32_t* tables, int n_tables, size_t cap_tokens, void* k_out, void* v_out,
                       int* total_tokens) {
    return guard([&] {
        need(s && (tables || n_tables == 0), "null argument");
        long need_tokens = 0;
        for (int i = 0; i < n_tables; ++i)
            if (const tkv::TableImage* img = s->arena->find(tables[i])) need_tokens += img->tokens;
        if (total_tokens) *total_tokens = int(need_tokens);
        need(!(k_out || v_out) || size_t(need_tokens) <= cap_tokens, "output buffers hold fewer tokens than the prefix");
        if (!k_out && !v_out) return;
        set_device(s->model->device);
        tkv::Model& model = *s->model->m;
        const auto& c = model.cfg();
        const int L = c.num_layers, kvd = c.kv_dim();
        const tkv::DType out_dt = c.dtype == tkv::DType::bf16 ? tkv::DType::bf16 : tkv::DType::f32;
        const size_t P = s->pool->page_bytes();
        cudaStream_t st = s->model->s;
        std::vector<tkv::GatherSeg> segs;
        std::vector<int32_t> page_ids;
        std::vector<std::vector<int32_t>> held;
        int total = 0;
        tkv::DType in_dt = tkv::DType::f32;
        for (int i = 0; i < n_tables; ++i) {
            const tkv::TableImage* img = s->arena->find(tables[i]);
            if (!img)
                throw tablekv::Error(tablekv::Errc::missing_table_kv, "no precomputed KV for table " + std::to_string(tables[i]));
            in_dt = img->dtype;
            auto pages = s->pool->alloc(int((img->bytes + P - 1) / P));
            tkv::copy_table_to_pages(*img, *s->pool, pages, tkv::CopyEngine::dma, 16, st);
            segs.push_back({int32_t(page_ids.size()), img->tokens, total, total});
            page_ids.insert(page_ids.end(), pages.begin(), pages.end());
            total += img->tokens;
            held.push_back(std::move(pages));
        }
        if (total_tokens) *total_tokens = total;
        if (total > 0) {
            model.rope().ensure(total + 1);
            const size_t ob = size_t(L) * total * kvd * tkv::dtype_size(out_dt);
            void *dk = nullptr, *dv = nullptr, *dseg = nullptr, *dpg = nullptr;
            TKV_CUDA_CHECK(cudaMalloc(&dk, ob));
            TKV_CUDA_CHECK(cudaMalloc(&dv, ob));
            TKV_CUDA_CHECK(cudaMalloc(&dseg, segs.size() * sizeof(tkv::GatherSeg)));
            TKV_CUDA_CHECK(cudaMalloc(&dpg, page_ids.size() * 4));
            TKV_CUDA_CHECK(cudaMemcpyAsync(dseg, segs.data(), segs.size() * sizeof(tkv::GatherSeg), cudaMemcpyHostToDevice, st));
            TKV_CUDA_CHECK(cudaMemcpyAsync(dpg, page_ids.data(), page_ids.size() * 4, cudaMemcpyHostToDevice, st));
            tkv::launch_gather_rope(s->pool->base(), P, static_cast<int32_t*>(dpg), static_cast<tkv::GatherSeg*>(dseg),
                                    int(segs.size()), total, L, kvd, c.head_dim, in_dt, out_dt, model.rope().cos_d(),
                                    model.rope().sin_d(), model.rope().cos_f(), model.rope().sin_f(), dk, dv, total, st);
            if (k_out) TKV_CUDA_CHECK(cudaMemcpyAsync(k_out, dk, ob, cudaMemcpyDeviceToHost, st));
            if (v_out) TKV_CUDA_CHECK(cudaMemcpyAsync(v_out, dv, ob, cudaMemcpyDeviceToHost, st));
            TKV_CUDA_CHECK(cudaStreamSynchronize(st));
            cudaFree(dk);
            cudaFree(dv);
            cudaFree(dseg);
            cudaFree(dpg);
        }
        for (auto& p : held) s->pool->release(p, st);
    });
}

namespace {
tkv::PageList page_list(const std::vector<int32_t>& pages) {
    if (pages.size() > size_t(tkv::kMaxPagesPerCopy)) throw std::invalid_argument("table spans too many pages for one copy");
    tkv::PageList pl;
    pl.n = int(pages.size());
    for (size_t i = 0; i < pages.size(); ++i) pl.page[i] = pages[i];
    return pl;
}
tkv::PeerMesh& mesh_of(tkv_store* s) {
    if (!s->mesh) throw std::invalid_argument("no peer mesh: call tkv_store_peer_export first");
    return *s->mesh;
}
}  // namespace

int tkv_store_peer_export(tkv_store* s, int dir_entries, void* blob_out, size_t cap, size_t* n) {
    return guard([&] {
        need(s && n, "null argument");
        set_device(s->model->device);
        if (!s->mesh) {
            const int entries = dir_entries > 0 ? dir_entries : s->arena->max_table_id() + 1;
            need(entries > 0, "peer directory needs at least one table (load the arena first)");
            s->mesh = std::make_unique<tkv::PeerMesh>(s->pool->base(), s->pool->page_bytes(), s->pool->n_pages(), entries);
            s->server->set_mesh(s->mesh.get());
        }
        *n = sizeof(tkv::PeerBlob);
        if (blob_out) {
            need(cap >= sizeof(tkv::PeerBlob), "blob buffer too small");
            const tkv::PeerBlob b = s->mesh->blob();
            std::memcpy(blob_out, &b, sizeof(b));
        }
    });
}

int tkv_store_peer_attach(tkv_store* s, int n, const void* const* blobs, const size_t* sizes) {
    return guard([&] {
        need(s && (blobs || n == 0), "null argument");
        set_device(s->model->device);
        std::vector<tkv::PeerBlob> v(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            need(blobs[i] && (!sizes || sizes[i] == sizeof(tkv::PeerBlob)), "bad peer blob");
            std::memcpy(&v[size_t(i)], blobs[i], sizeof(tkv::PeerBlob));
        }
        mesh_of(s).attach(v);
    });
}

int tkv_store_peer_plan(tkv_store* s, int slot, size_t n, const int64_t* table_off, const int32_t* tables,
                        const int32_t* suffix_len) {
    return guard([&] {
        need(s && table_off && (suffix_len || n == 0), "null argument");
        need(slot >= 0 && slot < tkv::kMaxPeers, "peer slot out of range");
        tkv::PeerPlan p;
        for (size_t i = 0; i < n; ++i) {
            p.tables.emplace_back(tables + table_off[i], tables + table_off[i + 1]);
            p.suffix_len.push_back(suffix_len[i]);
        }
        s->server->set_peer_plan(slot, std::move(p));
    });
}

int tkv_store_peer_publish(tkv_store* s, int table_id) {
    return guard([&] {
        need(s, "null argument");
        set_device(s->model->device);
        tkv::PeerMesh& m = mesh_of(s);
        need(table_id >= 0 && table_id < m.dir_entries(), "table id outside the peer directory");
        need(!s->held.count(table_id), "table already published");
        const tkv::TableImage* img = s->arena->find(table_id);
        if (!img) throw tablekv::Error(tablekv::Errc::unknown_table, "table " + std::to_string(table_id) + " not in the arena");
        const size_t P = s->pool->page_bytes();
        auto pages = s->pool->alloc(int((img->bytes + P - 1) / P));
        tkv::copy_table_to_pages(*img, *s->pool, pages, tkv::CopyEngine::dma, 16, s->model->s);
        tkv::launch_dir_publish(m, table_id, page_list(pages), s->model->s);
        TKV_CUDA_CHECK(cudaStreamSynchronize(s->model->s));
        s->held[table_id] = std::move(pages);
    });
}

int tkv_store_peer_unpublish(tkv_store* s, int table_id) {
    return guard([&] {
        need(s, "null argument");
        set_device(s->model->device);
        auto it = s->held.find(table_id);
        need(it != s->held.end(), "table not published");
        tkv::launch_dir_revoke(mesh_of(s), table_id, s->model->s);
        s->pool->release(it->second, s->model->s);
        TKV_CUDA_CHECK(cudaStreamSynchronize(s->model->s));
        s->held.erase(it);
    });
}

int tkv_store_peer_fetch(tkv_store* s, int table_id, void* host_out, size_t bytes, uint64_t* peer_bytes) {
    return guard([&] {
        need(s && host_out, "null argument");
        set_device(s->model->device);
        tkv::PeerMesh& m = mesh_of(s);
        const tkv::TableImage* img = s->arena->find(table_id);
        if (!img) throw tablekv::Error(tablekv::Errc::unknown_table, "table " + std::to_string(table_id) + " not in the arena");
        need(bytes == img->bytes, "byte count does not match the table image");
        const size_t P = s->pool->page_bytes();
        cudaStream_t st = s->model->s;
        auto pages = s->pool->alloc(int((img->bytes + P - 1) / P));
        tkv::PeerOrder po;
        for (int i = 0; i < tkv::kMaxPeers; ++i) po.p[i] = int8_t(i < m.n_peers() ? i : -1);
        TKV_CUDA_CHECK(cudaMemsetAsync(m.stats(), 0, 2 * sizeof(unsigned long long), st));
        tkv::launch_peer_fetch(m.view(), po, table_id, img->mapped, img->bytes, s->pool->base(), P, page_list(pages),
                               m.stats(), 64, st);
        for (size_t i = 0; i * P < img->bytes; ++i)
            TKV_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(host_out) + i * P, s->pool->base() + size_t(pages[i]) * P,
                                           std::min(P, img->bytes - i * P), cudaMemcpyDeviceToHost, st));
        unsigned long long stv[2];
        TKV_CUDA_CHECK(cudaMemcpyAsync(stv, m.stats(), sizeof(stv), cudaMemcpyDeviceToHost, st));
        TKV_CUDA_CHECK(cudaStreamSynchronize(st));
        s->pool->release(pages, st);
        if (peer_bytes) *peer_bytes = stv[0];
    });
}

int tkv_store_info(const tkv_store* s, size_t* tables, size_t* arena_bytes, size_t* free_pages) {
    return guard([&] {
        need(s, "null argument");
        s->pool->reclaim();  // fold completed deferred frees back into the free list
        if (tables) *tables = s->arena->size();
        if (arena_bytes) *arena_bytes = s->arena->total_bytes();
        if (free_pages) *free_pages = size_t(s->pool->free_pages());
    });
}

void tkv_serve_options_default(tkv_serve_options* o) {
    if (!o) return;
    *o = tkv_serve_options{};
    o->rerank_on = 1;
    o->pipeline_on = 1;
    o->capacity = 8;
    o->policy = 0;
    o->b_c = 100;
    o->b_m = 10;
    o->seed = 1;
    o->compute_per_token = 0.01;
    o->load_per_token = 1.0;
    o->switch_overhead = 5.0;
    o->copy_engine = 0;
    o->sm_copy_ctas = 16;
    o->peer_fetch = 0;
    o->peer_ctas = 64;
}

namespace {
int serve_impl(tkv_store* s, std::vector<tkv::ServeQuery>& qs, const tkv_serve_options* o, float* logits_out, char** result_json,
               double analyze_ms = 0) {
    return guard([&] {
        need(s && o, "null argument");
        set_device(s->model->device);
        tkv::ServeOptions so = serve_opts(o);
        so.keep_logits = logits_out != nullptr;
        tkv::ServeResult R = o->nocache ? s->server->serve_nocache(qs, so) : s->server->serve(qs, so);
        if (logits_out && !R.logits.empty()) std::memcpy(logits_out, R.logits.data(), R.logits.size() * 4);
        if (result_json) {
            json j = serve_result_json(R);
            j["analyze_ms"] = analyze_ms;  // prompt text -> tables + suffix on the host (tkv_serve_text)
            *result_json = dup_string(j.dump());
        }
    });
}
}  // namespace

int tkv_serve(tkv_store* s, size_t n, const int64_t* table_off, const int32_t* tables, const int64_t* suffix_off,
              const int32_t* suffix, const tkv_serve_options* o, float* logits_out, char** result_json) {
    std::vector<tkv::ServeQuery> qs(n);
    const int rc = guard([&] {
        need(table_off && suffix_off, "null offsets");
        for (size_t i = 0; i < n; ++i) {
            qs[i].id = "q" + std::to_string(i);
            qs[i].tables.assign(tables + table_off[i], tables + table_off[i + 1]);
            qs[i].suffix.assign(suffix + suffix_off[i], suffix + suffix_off[i + 1]);
        }
    });
    if (rc != TKV_OK) return rc;
    return serve_impl(s, qs, o, logits_out, result_json);
}

int tkv_serve_text(tkv_store* s, const tkv_engine* e, size_t n, const char* const* ids, const char* const* texts,
                   const tkv_serve_options* o, float* logits_out, char** result_json) {
    std::vector<tkv::ServeQuery> qs(n);
    const auto t_an = std::chrono::steady_clock::now();
    const int rc = guard([&] {
        need(e && texts, "null argument");
        // prompt analysis (tokenize -> Table Trie -> assembly order) is pure per prompt and the trie
        // is immutable after construction (trie.hpp:31-33), so prompts fan out over host threads;
        // results land by index, identical to the sequential loop
        const size_t n_thr = std::max<size_t>(1, std::min<size_t>({n / 32 + 1, 16, std::thread::hardware_concurrency()}));
        std::vector<std::exception_ptr> errs(n_thr);
        auto work = [&](size_t w) {
            try {
                for (size_t i = w; i < n; i += n_thr) {
                    auto a = tablekv::analyze_query(e->e, ids ? ids[i] : std::to_string(i), texts[i]);
                    qs[i].id = a.record.query_id;
                    qs[i].tables = tablekv::assembly_order(e->e, a.match_order);
                    qs[i].suffix.assign(a.remainder.begin(), a.remainder.end());
                }
            } catch (...) {
                errs[w] = std::current_exception();
            }
        };
        std::vector<std::thread> pool;
        for (size_t w = 1; w < n_thr; ++w) pool.emplace_back(work, w);
        work(0);
        for (auto& t : pool) t.join();
        for (auto& ep : errs)
            if (ep) std::rethrow_exception(ep);
    });
    if (rc != TKV_OK) return rc;
    const double an_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_an).count();
    return serve_impl(s, qs, o, logits_out, result_json, an_ms);
}

// ------------------------------------------------------------------ measurement
int tkv_measure_h2d(int device, size_t bytes, int reps, double* gbs) {
    return guard([&] {
        need(gbs && bytes > 0, "null argument");
        set_device(device);
        void *h = nullptr, *d = nullptr;
        TKV_CUDA_CHECK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
        TKV_CUDA_CHECK(cudaMalloc(&d, bytes));
        std::memset(h, 1, bytes);
        cudaStream_t st;
        cudaEvent_t a, b;
        TKV_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        TKV_CUDA_CHECK(cudaEventCreate(&a));
        TKV_CUDA_CHECK(cudaEventCreate(&b));
        double best = 0;
        for (int r = 0; r < std::max(1, reps); ++r) {
            TKV_CUDA_CHECK(cudaEventRecord(a, st));
            TKV_CUDA_CHECK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
            TKV_CUDA_CHECK(cudaEventRecord(b, st));
            TKV_CUDA_CHECK(cudaEventSynchronize(b));
            float ms = 0;
            TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
            best = std::max(best, double(bytes) / (ms * 1e6));
        }
        *gbs = best;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(st);
        cudaFree(d);
        cudaFreeHost(h);
    });
}

int tkv_debug_gemm(int M, int N, int K, const uint16_t* A, const uint16_t* B, int epilogue, int simt, void* C, double* ms_out) {
    return guard([&] {
        need(A && B && C && M > 0 && N > 0 && K > 0, "bad gemm arguments");
        void *dA, *dB, *dC;
        const size_t cb = size_t(M) * N * (epilogue == 1 ? 4 : 2);
        TKV_CUDA_CHECK(cudaMalloc(&dA, size_t(M) * K * 2));
        TKV_CUDA_CHECK(cudaMalloc(&dB, size_t(N) * K * 2));
        TKV_CUDA_CHECK(cudaMalloc(&dC, cb));
        TKV_CUDA_CHECK(cudaMemcpy(dA, A, size_t(M) * K * 2, cudaMemcpyHostToDevice));
        TKV_CUDA_CHECK(cudaMemcpy(dB, B, size_t(N) * K * 2, cudaMemcpyHostToDevice));
        tkv::EpiParams ep;
        ep.kind = epilogue == 1 ? tkv::Epi::store_f32 : tkv::Epi::store_bf16;
        ep.out = dC;
        ep.ldo = N;
        cudaEvent_t a, b;
        TKV_CUDA_CHECK(cudaEventCreate(&a));
        TKV_CUDA_CHECK(cudaEventCreate(&b));
        // simt: 0 = product kernel (persistent tcgen05), 1 = SIMT reference, 2 = one-tile-per-CTA tcgen05
        auto run = [&] {
            if (simt == 1) tkv::gemm_bf16_simt(dA, dB, M, N, K, ep, nullptr);
            else if (simt == 2) tkv::gemm_bf16_classic(dA, dB, M, N, K, ep, nullptr);
            else tkv::gemm_bf16(dA, dB, M, N, K, ep, nullptr);
        };
        run();  // warm-up (tensor maps, smem attributes)
        const int reps = simt == 1 ? 1 : 5;
        TKV_CUDA_CHECK(cudaEventRecord(a, nullptr));
        for (int r = 0; r < reps; ++r) run();
        TKV_CUDA_CHECK(cudaEventRecord(b, nullptr));
        TKV_CUDA_CHECK(cudaEventSynchronize(b));
        float ms = 0;
        TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
        if (ms_out) *ms_out = ms / reps;
        TKV_CUDA_CHECK(cudaMemcpy(C, dC, cb, cudaMemcpyDeviceToHost));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dC);
    });
}

}  // extern "C"
