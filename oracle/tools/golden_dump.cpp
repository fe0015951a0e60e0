// Golden-vector generator (TEST INFRASTRUCTURE, never shipped).
//
// Drives the UNCHANGED reference library (compiled from /root/reference/proj by
// oracle/Makefile, namespace renamed to tablekv_ref) on JSON-described inputs and writes
// JSON (+ a raw little-endian tensor blob) that tests/golden/ commits. The repo's own
// oracle restatement (oracle/tkv_oracle.py) and the CUDA product are both checked
// against these files. Usage:
//     golden_dump <command> <in.json> <out.json> [<out.bin>]
// Commands: engine | run_batch | cache_ops | rerank | trie | attention | rng | rotary
//
// The reference's pipeline.cpp is #included textually (REF_PIPELINE_SRC) because its
// canonical cache trajectory `build_trace` (proj/src/pipeline.cpp:44-116) is file-local;
// dumping it lets the GPU executor prove its hit/miss/evict sequence is identical.

#include REF_PIPELINE_SRC

#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

#include "corpus_gen.hpp"
#include "tablekv/attention.hpp"
#include "tablekv/engine.hpp"
#include "tablekv/rng.hpp"
#include "tablekv/rotary.hpp"
#include "tablekv/table_kv.hpp"

using nlohmann::json;
using namespace tablekv;  // renamed to tablekv_ref by -D
namespace fs = std::filesystem;

namespace {

// ---- tensor blob -------------------------------------------------------------------
struct Blob {
    std::string bytes;
    json index = json::object();
    template <typename T>
    void put(const std::string& name, const std::vector<T>& v, std::vector<size_t> shape) {
        static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>);
        // 16-byte align every tensor
        while (bytes.size() % 16) bytes.push_back('\0');
        index[name] = {{"offset", bytes.size()},
                       {"count", v.size()},
                       {"dtype", std::is_same_v<T, float> ? "f32" : "f64"},
                       {"shape", shape}};
        bytes.append(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
    }
};

json read_json(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    json j;
    in >> j;
    return j;
}

void write_text(const std::string& path, const std::string& body) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    out << body;
}

json span_json(const std::vector<MatchSpan>& spans) {
    json a = json::array();
    for (const auto& s : spans) a.push_back({s.table_id, s.start, s.end});
    return a;
}

json load_rec_json(const std::vector<LoadRec>& v) {
    json a = json::array();
    for (const auto& r : v) a.push_back({{"table", r.table}, {"miss", r.miss}, {"evicted", r.evicted}, {"size", r.size}});
    return a;
}

json trace_json(const Trace& tr) {
    json w = json::array();
    for (const auto& wt : tr.windows) {
        json e = json::array();
        for (const auto& q : wt.emergency) e.push_back(load_rec_json(q));
        w.push_back({{"boundary", load_rec_json(wt.boundary)}, {"prefetch", load_rec_json(wt.prefetch)}, {"emergency", e}});
    }
    return {{"windows", w}, {"compute", tr.compute}};
}

json plan_json(const BatchPlan& plan) {
    json w = json::array();
    for (const auto& win : plan.windows)
        w.push_back({{"begin", win.begin}, {"end", win.end}, {"demand", win.demand}, {"prefetch", win.prefetch}});
    json lu = json::object();
    for (const auto& [t, i] : plan.last_use) lu[std::to_string(t)] = i;
    return {{"b_c", plan.b_c}, {"b_m", plan.b_m}, {"windows", w}, {"last_use", lu}};
}

RunOptions run_options(const json& r) {
    RunOptions o;
    o.rerank_on = r.value("rerank_on", true);
    o.pipeline_on = r.value("pipeline_on", true);
    o.capacity = r.value("capacity", size_t(8));
    o.policy = parse_policy(r.value("policy", std::string("lru")));
    o.b_c = r.value("b_c", 100);
    o.b_m = r.value("b_m", 10);
    o.seed = r.value("seed", uint64_t(1));
    o.anchor = r.value("anchor", std::string("seeded")) == "fixed_first" ? AnchorMode::fixed_first : AnchorMode::seeded;
    return o;
}

CostModel cost_model(const json& c) {
    CostModel m;
    m.compute_per_token = c.value("compute_per_token", 0.01);
    m.load_per_token = c.value("load_per_token", 1.0);
    m.switch_overhead = c.value("switch_overhead", 5.0);
    return m;
}

json report_json(const SimReport& r) { return json::parse(r.to_json()); }

// The full run_batch pipeline with every intermediate exposed: rerank permutation,
// schedule windows, the canonical trace, and both simulated reports.
json run_batch_detailed(const std::vector<QueryRecord>& recs, const RunOptions& opts, const CostModel& cost,
                        std::shared_ptr<SlowTier> slow) {
    json out;
    std::vector<size_t> order;
    if (opts.rerank_on) {
        order = rerank(recs, opts.seed, opts.anchor);
    } else {
        order.resize(recs.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    }
    out["order"] = order;
    std::vector<SimQuery> sims;
    for (size_t i : order) sims.push_back({recs[i].query_id, recs[i].tables, recs[i].query_token_count});
    BatchPlan plan = schedule(sims, opts.b_c, opts.b_m);
    out["plan"] = plan_json(plan);
    {
        TieredCache cache(opts.capacity, opts.policy, slow);
        out["trace"] = trace_json(build_trace(plan, cost, cache));
        const auto& c = cache.counters();
        out["trace_counters"] = {{"hits", c.hits}, {"misses", c.misses}, {"swaps", c.swaps}, {"prefetch_loads", c.prefetch_loads}};
        out["final_residents"] = cache.residents();
    }
    SimReport via = run_batch(recs, opts, cost, slow);
    out["report"] = report_json(via);
    {
        TieredCache c1(opts.capacity, opts.policy, slow);
        out["report_overlapped"] = report_json(simulate(plan, cost, c1, SimMode::overlapped));
        TieredCache c2(opts.capacity, opts.policy, slow);
        out["report_serial"] = report_json(simulate(plan, cost, c2, SimMode::serial));
    }
    return out;
}

// Documented extension G1 (the reference has no LM head): final LayerNorm (no affine,
// eps 1e-5) of the last hidden row, then an untied head W_head[vocab][hidden] with
// W[i] = float(u64_to_signed_unit(mix3(seed, 8*131, i)) / sqrt(hidden)) (cast like every
// reference weight, model.hpp:85), logits accumulated in double.
// The same definition lives in oracle/tkv_oracle.py and in the CUDA model.
std::vector<double> head_logits(const ModelConfig& cfg, const std::vector<float>& last_row) {
    const int h = cfg.hidden_dim();
    double mean = 0, var = 0;
    for (int i = 0; i < h; ++i) mean += last_row[i];
    mean /= h;
    for (int i = 0; i < h; ++i) var += (last_row[i] - mean) * (last_row[i] - mean);
    var /= h;
    const double inv = 1.0 / std::sqrt(var + 1e-5);
    std::vector<double> xn(h);
    for (int i = 0; i < h; ++i) xn[i] = (last_row[i] - mean) * inv;
    const double scale = 1.0 / std::sqrt(double(h));
    std::vector<double> logits(cfg.vocab_size);
    for (int v = 0; v < cfg.vocab_size; ++v) {
        double acc = 0;
        for (int i = 0; i < h; ++i) {
            const double w = static_cast<float>(u64_to_signed_unit(mix3(cfg.weight_seed, 8 * 131ull, uint64_t(v) * h + i)) * scale);
            acc += w * xn[i];
        }
        logits[v] = acc;
    }
    return logits;
}

// ---- commands -----------------------------------------------------------------------

json cmd_engine(const json& in, Blob& blob) {
    EngineOptions eo;
    eo.schema_path = in.at("schema_path");
    const json mo = in.value("model", json::object());
    eo.num_layers = mo.value("num_layers", 2);
    eo.num_heads = mo.value("num_heads", 4);
    eo.head_dim = mo.value("head_dim", 16);
    eo.rotary_base = mo.value("rotary_base", 10000.0);
    eo.weight_seed = mo.value("weight_seed", uint64_t(1));
    if (in.value("break_cycles", false)) eo.topo_mode = TopoMode::break_cycles;
    Engine e = build_engine(eo);

    json out;
    out["vocab_size"] = e.tokenizer.vocab_size();
    out["vocab_hash"] = e.tokenizer.vocab_hash();
    out["topo_order"] = e.topo.order;
    json groups = json::array();
    for (const auto& g : e.plan.groups) groups.push_back({{"tables", g.tables}, {"offsets", g.offsets}});
    out["groups"] = groups;
    out["group_of"] = e.plan.group_of;
    out["local_offset"] = e.local_offset;
    out["serialized"] = e.serialized;
    out["table_tokens"] = e.table_tokens;
    {
        json es = json::array();
        for (int u = 0; u < e.graph.node_count; ++u)
            for (int v : e.graph.out_edges[u]) es.push_back({u, v});
        out["edges"] = es;
    }
    // weight samples (first 8 entries of each tensor of layer 0 + embedding)
    {
        auto head = [](const std::vector<float>& v) { return std::vector<float>(v.begin(), v.begin() + std::min<size_t>(8, v.size())); };
        const auto& L0 = e.weights.layers.at(0);
        out["weight_samples"] = {{"embedding", head(e.weights.embedding)}, {"wq", head(L0.wq)}, {"wk", head(L0.wk)},
                                 {"wv", head(L0.wv)}, {"wo", head(L0.wo)}, {"ffn_in", head(L0.ffn_in)}, {"ffn_out", head(L0.ffn_out)}};
        double s = 0;
        for (float x : e.weights.embedding) s += x;
        for (const auto& L : e.weights.layers)
            for (const auto* v : {&L.wq, &L.wk, &L.wv, &L.wo, &L.ffn_in, &L.ffn_out})
                for (float x : *v) s += x;
        out["weight_sum"] = s;
    }

    // precompute .kv files (the loaded-bytes ground truth)
    const std::string kv_dir = in.value("kv_dir", std::string());
    std::shared_ptr<SlowTier> slow;
    auto mem = std::make_shared<MemorySlowTier>();
    {
        for (const auto& g : e.plan.groups) {
            std::vector<GroupTableRef<float>> refs;
            for (int id : g.tables) refs.push_back({id, std::span<const TokenId>(e.table_tokens[id])});
            for (auto& kv : encode_group<float>(e.config, e.weights, refs)) mem->put(std::move(kv));
        }
        slow = mem;
        if (!kv_dir.empty()) {
            precompute_corpus(e, kv_dir);
            slow = std::make_shared<FileSlowTier>(kv_dir);
        }
    }

    // workload analysis
    auto workload = load_workload(in.at("workload_path"));
    const size_t nq = std::min<size_t>(workload.size(), in.value("n_queries", workload.size()));
    workload.resize(nq);
    json qs = json::array();
    std::vector<AnalyzedQuery> analyzed;
    std::vector<QueryRecord> recs;
    for (const auto& w : workload) {
        AnalyzedQuery q = analyze_query(e, w.query_id, w.text);
        const auto order = assembly_order(e, q.match_order);
        qs.push_back({{"query_id", w.query_id}, {"tokens", q.tokens}, {"spans", span_json(q.spans)},
                      {"match_order", q.match_order}, {"remainder", q.remainder}, {"assembly_order", order},
                      {"record_tables_sorted", q.record.tables}, {"query_token_count", q.record.query_token_count}});
        QueryRecord rec = q.record;
        rec.tables = order;
        recs.push_back(std::move(rec));
        analyzed.push_back(std::move(q));
    }
    out["queries"] = qs;

    // serving runs
    json runs = json::object();
    for (const auto& r : in.value("runs", json::array())) {
        const RunOptions opts = run_options(r);
        const CostModel cost = cost_model(r.value("cost", json::object()));
        json d = run_batch_detailed(recs, opts, cost, slow);
        d["run_workload"] = report_json(run_workload(e, workload, opts, cost, slow));
        runs[r.at("name").get<std::string>()] = d;
    }
    out["runs"] = runs;

    // numerics: assembled context for a few queries, query_attend hidden, block-masked oracle
    const json tq = in.value("tensors", json::object());
    const size_t n_asm = tq.value("assemble_queries", 0);
    const size_t n_hidden = tq.value("hidden_queries", 0);
    const int hdim = e.config.hidden_dim();
    json numerics = json::array();
    for (size_t qi = 0; qi < std::min(n_hidden, analyzed.size()); ++qi) {
        const auto& q = analyzed[qi];
        const auto order = assembly_order(e, q.match_order);
        std::vector<TableKV<float>> kvs;
        for (int id : order) kvs.push_back(*slow->load(id));
        const auto ctx = assemble<float>(e.config, e.plan, kvs, order);
        const auto served = query_attend<float>(e.config, e.weights, ctx, q.remainder);
        const double vd = verify_query(e, *slow, q);
        const std::string p = "q" + std::to_string(qi) + ".";
        blob.put(p + "hidden", served, {q.remainder.size(), size_t(hdim)});
        // block-masked oracle rows for the remainder
        std::vector<TokenId> concat;
        BlockMask mask;
        for (int id : order) {
            concat.insert(concat.end(), e.table_tokens[id].begin(), e.table_tokens[id].end());
            mask.append_block(e.plan.group_of[id], int(e.table_tokens[id].size()));
        }
        concat.insert(concat.end(), q.remainder.begin(), q.remainder.end());
        mask.append_block(kQueryGroup, int(q.remainder.size()));
        const auto oracle = prefill<float>(e.config, e.weights, concat, mask);
        const size_t ctx_tok = concat.size() - q.remainder.size();
        std::vector<float> orows(oracle.hidden.begin() + ctx_tok * hdim, oracle.hidden.end());
        blob.put(p + "oracle_hidden", orows, {q.remainder.size(), size_t(hdim)});
        json info = {{"query", qi}, {"nctx", ctx.total_tokens}, {"n_rem", q.remainder.size()}, {"verify_max_diff", vd}};
        if (!q.remainder.empty()) {
            std::vector<float> last(served.end() - hdim, served.end());
            const auto logits = head_logits(e.config, last);
            blob.put(p + "logits", logits, {logits.size()});
            info["argmax"] = std::max_element(logits.begin(), logits.end()) - logits.begin();
        }
        if (qi < n_asm) {
            for (int l = 0; l < e.config.num_layers; ++l) {
                blob.put(p + "ctx_k" + std::to_string(l), ctx.k[l], {size_t(ctx.total_tokens), size_t(hdim)});
                blob.put(p + "ctx_v" + std::to_string(l), ctx.v[l], {size_t(ctx.total_tokens), size_t(hdim)});
            }
            json sp = json::array();
            for (const auto& s : ctx.span_index) sp.push_back({s.table_id, s.start, s.end});
            info["span_index"] = sp;
        }
        numerics.push_back(info);
    }
    out["numerics"] = numerics;
    return out;
}

std::shared_ptr<MemorySlowTier> metadata_tier(const std::vector<int>& token_counts) {
    auto slow = std::make_shared<MemorySlowTier>();
    for (size_t id = 0; id < token_counts.size(); ++id) {
        TableKV<float> kv;
        kv.table_id = int(id);
        kv.token_count = token_counts[id];
        kv.num_heads = 4;
        kv.head_dim = 16;
        slow->put(std::move(kv));
    }
    return slow;
}

// Records with tables in serving (assembly) order; incidence from the same set.
json cmd_run_batch(const json& in) {
    const std::vector<int> counts = in.at("token_counts");
    auto slow = metadata_tier(counts);
    std::vector<QueryRecord> recs;
    for (const auto& q : in.at("queries")) {
        std::vector<int> tables = q.at("tables");
        QueryRecord rec = make_query_record(q.at("id"), {}, tables, int(counts.size()), q.at("query_tokens"));
        rec.tables = tables;
        recs.push_back(std::move(rec));
    }
    json out = json::object();
    for (const auto& r : in.at("runs")) {
        out[r.at("name").get<std::string>()] =
            run_batch_detailed(recs, run_options(r), cost_model(r.value("cost", json::object())), slow);
    }
    return out;
}

json cmd_cache_ops(const json& in) {
    auto slow = metadata_tier(in.at("token_counts").get<std::vector<int>>());
    json out = json::array();
    for (const auto& c : in.at("cases")) {
        TieredCache cache(c.at("capacity"), parse_policy(c.at("policy")), slow);
        json steps = json::array();
        for (const auto& op : c.at("ops")) {
            json s;
            if (cache.capacity() > 0 && cache.size() == cache.capacity()) s["candidate"] = cache.evict_candidate();
            if (op.contains("get")) {
                auto r = cache.get(op.at("get").get<int>());
                s["hit"] = r.hit;
                s["evicted"] = r.evicted_id;
            } else {
                std::vector<int> ids = op.at("prefetch");
                s["admitted"] = cache.prefetch(ids);
            }
            s["residents"] = cache.residents();
            const auto& k = cache.counters();
            s["counters"] = {k.hits, k.misses, k.swaps, k.prefetch_loads};
            steps.push_back(s);
        }
        out.push_back({{"capacity", c.at("capacity")}, {"policy", c.at("policy")}, {"steps", steps}});
    }
    return out;
}

json cmd_rerank(const json& in) {
    json out = json::array();
    for (const auto& b : in.at("batches")) {
        const int n_bits = b.at("n_bits");
        std::vector<QueryRecord> qs;
        int i = 0;
        for (const auto& t : b.at("queries"))
            qs.push_back(make_query_record("q" + std::to_string(i++), {}, t.get<std::vector<int>>(), n_bits, 5));
        const auto mode = b.value("mode", std::string("seeded")) == "fixed_first" ? AnchorMode::fixed_first : AnchorMode::seeded;
        json ham = json::array();
        for (size_t a = 0; a < std::min<size_t>(qs.size(), 6); ++a)
            for (size_t c = 0; c < std::min<size_t>(qs.size(), 6); ++c) ham.push_back(hamming(qs[a].inc, qs[c].inc));
        out.push_back({{"order", rerank(qs, b.at("seed").get<uint64_t>(), mode)}, {"hamming6x6", ham}});
    }
    return out;
}

json cmd_trie(const json& in) {
    TableTrie trie;
    int id = 0;
    for (const auto& p : in.at("patterns")) {
        std::vector<TokenId> t = p;
        trie.insert(t, id, CacheHandle(id));
        ++id;
    }
    json out = json::array();
    for (const auto& x : in.at("inputs")) {
        std::vector<TokenId> t = x;
        MatchStats st;
        auto spans = trie.match_all(t, &st);
        json q = json::array();
        for (size_t s = 0; s < std::min<size_t>(t.size(), 32); ++s) {
            auto r = trie.query(t, s);
            q.push_back({r.found, r.next, r.table_id});
        }
        out.push_back({{"spans", span_json(spans)}, {"node_visits", st.node_visits}, {"query_first32", q}});
    }
    return out;
}

template <typename Real>
void attention_case(const json& c, Blob& blob, const std::string& tag, json& info) {
    using namespace testsupport;
    const auto corp = random_token_corpus(c.at("corpus_seed"), c.at("n_tables"), c.at("max_group"), c.at("min_tokens"),
                                          c.at("max_tokens"), c.at("vocab"));
    ModelConfig cfg;
    cfg.vocab_size = c.at("vocab");
    cfg.num_layers = c.value("num_layers", 2);
    cfg.num_heads = c.value("num_heads", 4);
    cfg.head_dim = c.value("head_dim", 16);
    cfg.weight_seed = c.at("weight_seed");
    const auto w = ModelWeights<Real>::create(cfg);
    const auto kvs = encode_corpus<Real>(cfg, w, corp);
    const size_t hd = size_t(cfg.hidden_dim());
    for (size_t t = 0; t < kvs.size(); ++t)
        for (int l = 0; l < cfg.num_layers; ++l) {
            blob.put(tag + "kv" + std::to_string(t) + ".k" + std::to_string(l), kvs[t].k[l], {size_t(kvs[t].token_count), hd});
            blob.put(tag + "kv" + std::to_string(t) + ".v" + std::to_string(l), kvs[t].v[l], {size_t(kvs[t].token_count), hd});
        }
    const auto order = shuffled_group_order(corp, c.at("order_seed"));
    const auto ctx = assemble<Real>(cfg, corp.plan, kvs, order);
    const auto tokens = concat_tokens(corp, order);
    const auto mask = mask_for_order(corp, order);
    const auto pre = prefill<Real>(cfg, w, tokens, mask);
    for (int l = 0; l < cfg.num_layers; ++l) {
        blob.put(tag + "ctx_k" + std::to_string(l), ctx.k[l], {size_t(ctx.total_tokens), hd});
        blob.put(tag + "ctx_v" + std::to_string(l), ctx.v[l], {size_t(ctx.total_tokens), hd});
        blob.put(tag + "pre_krot" + std::to_string(l), pre.k_rot[l], {tokens.size(), hd});
        blob.put(tag + "pre_kraw" + std::to_string(l), pre.k_raw[l], {tokens.size(), hd});
    }
    blob.put(tag + "pre_hidden", pre.hidden, {tokens.size(), hd});
    std::vector<TokenId> qt = c.at("query_tokens");
    const auto served = query_attend<Real>(cfg, w, ctx, qt);
    blob.put(tag + "served", served, {qt.size(), hd});
    // block-masked oracle for served rows
    auto full = tokens;
    full.insert(full.end(), qt.begin(), qt.end());
    auto m2 = mask;
    m2.append_block(kQueryGroup, int(qt.size()));
    const auto pre2 = prefill<Real>(cfg, w, full, m2);
    std::vector<Real> rows(pre2.hidden.begin() + tokens.size() * hd, pre2.hidden.end());
    blob.put(tag + "served_oracle", rows, {qt.size(), hd});
    info["order"] = order;
    info["table_tokens"] = corp.table_tokens;
    json groups = json::array();
    for (const auto& g : corp.plan.groups) groups.push_back({{"tables", g.tables}, {"offsets", g.offsets}});
    info["groups"] = groups;
    info["group_of"] = corp.plan.group_of;
}

json cmd_attention(const json& in, Blob& blob) {
    json out = json::array();
    int k = 0;
    for (const auto& c : in.at("cases")) {
        json info;
        const std::string tag = "c" + std::to_string(k++) + ".";
        if (c.value("double", false))
            attention_case<double>(c, blob, tag, info);
        else
            attention_case<float>(c, blob, tag, info);
        info["tag"] = tag;
        out.push_back(info);
    }
    return out;
}

json cmd_rng(const json& in) {
    json out;
    json m = json::array();
    for (const auto& t : in.at("mix3")) m.push_back(std::to_string(mix3(t[0].get<uint64_t>(), t[1].get<uint64_t>(), t[2].get<uint64_t>())));
    out["mix3"] = m;
    json s = json::array();
    for (const auto& seed : in.at("seeded")) {
        SeededRng r(seed.get<uint64_t>());
        json seq = json::array();
        for (int i = 0; i < 8; ++i) seq.push_back(std::to_string(r.next_u64()));
        s.push_back(seq);
    }
    out["seeded"] = s;
    json u = json::array();
    for (const auto& t : in.at("mix3")) u.push_back(u64_to_signed_unit(mix3(t[0].get<uint64_t>(), t[1].get<uint64_t>(), t[2].get<uint64_t>())));
    out["signed_unit"] = u;
    return out;
}

json cmd_rotary(const json& in, Blob& blob) {
    json out = json::array();
    int k = 0;
    for (const auto& c : in.at("cases")) {
        const int H = c.at("heads"), D = c.at("head_dim");
        std::vector<int64_t> pos = c.at("positions");
        std::vector<float> data(pos.size() * H * D);
        SeededRng r(c.at("seed"));
        for (auto& x : data) x = float(r.next_unit() * 2 - 1);
        const std::string tag = "r" + std::to_string(k++) + ".";
        blob.put(tag + "in", data, {pos.size(), size_t(H * D)});
        apply_rotation<float>(data, pos, H, D, c.value("base", 10000.0));
        blob.put(tag + "out", data, {pos.size(), size_t(H * D)});
        out.push_back(tag);
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::cerr << "usage: golden_dump <command> <in.json> <out.json> [<out.bin>]\n";
        return 2;
    }
    try {
        const std::string cmd = argv[1];
        const json in = read_json(argv[2]);
        Blob blob;
        json out;
        if (cmd == "engine") out = cmd_engine(in, blob);
        else if (cmd == "run_batch") out = cmd_run_batch(in);
        else if (cmd == "cache_ops") out = cmd_cache_ops(in);
        else if (cmd == "rerank") out = cmd_rerank(in);
        else if (cmd == "trie") out = cmd_trie(in);
        else if (cmd == "attention") out = cmd_attention(in, blob);
        else if (cmd == "rng") out = cmd_rng(in);
        else if (cmd == "rotary") out = cmd_rotary(in, blob);
        else throw std::runtime_error("unknown command " + cmd);
        if (argc >= 5) {
            write_text(argv[4], blob.bytes);
            out = {{"result", out}, {"tensors", blob.index}};
        } else {
            out = {{"result", out}};
        }
        write_text(argv[3], out.dump(1) + "\n");
    } catch (const std::exception& e) {
        std::cerr << "golden_dump: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
