// CPU baseline timer (TEST/BENCH INFRASTRUCTURE, never shipped).
//
// Times the UNCHANGED reference library's own CPU implementation of the online path
// on this host's cores, for bench.py's `cpu_baseline` object and its `--impl reference`
// arm. Output: one JSON object on stdout.
//
//   ref_bench demo <schema.json> <workload.jsonl> <n_queries> <threads>
//       reference default model (2 layers, 4x16 heads): per query, the cached path
//       (FileSlowTier-equivalent loads from memory -> assemble -> query_attend,
//       proj/src/engine.cpp:174-205 minus the oracle) and the no-cache block-masked
//       prefill over the same layout. Queries are sharded over <threads> threads
//       (the attention functions are pure).
//   ref_bench wide <heads> <head_dim> <threads> [--cached-only] <nctx:nq>...
//       ONE layer of the reference architecture at the given width (MHA, LN, SiLU 4h),
//       per sample: query_attend of nq tokens over an nctx-token assembled context,
//       and the no-cache prefill of nctx+nq tokens. The caller scales by layer count.
//   ref_bench serve <schema.json> <workload.jsonl> <threads> <heads> <head_dim> <n_queries>
//       the reference's cached serving path on the bench workload itself: per query, the
//       reference's own prompt analysis (analyze_query + assembly_order, engine.cpp:133-172),
//       MemorySlowTier loads of the matched tables' KV, assemble (attention.hpp:300-362) and
//       query_attend (:368-414) -- ONE layer of the reference architecture at the given width
//       (MHA, LayerNorm, SiLU 4h; the reference cannot express GQA/SwiGLU/RMSNorm). The first
//       <n_queries> prompts (arrival order) run as one wave over <threads> cores (queries are
//       independent, the functions are pure), after an untimed warm wave of analysis + loads +
//       assemble (a CPU path has nothing to JIT; it pages the tables in). The caller
//       extrapolates the per-layer part by the served model's layer count and says so.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <iostream>
#include <thread>

#include <json.hpp>

#include "tablekv/attention.hpp"
#include "tablekv/engine.hpp"

using nlohmann::json;
using namespace tablekv;

namespace {

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

double pct(std::vector<double> v, double p) {
    if (v.empty()) return 0;
    std::sort(v.begin(), v.end());
    const double idx = p * (v.size() - 1);
    const size_t lo = size_t(idx);
    const size_t hi = std::min(lo + 1, v.size() - 1);
    return v[lo] + (v[hi] - v[lo]) * (idx - lo);
}

template <typename Fn>
double run_sharded(int n, int threads, Fn fn) {
    std::atomic<int> next{0};
    const double t0 = now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&] {
            for (int i = next++; i < n; i = next++) fn(i);
        });
    for (auto& th : pool) th.join();
    return now() - t0;
}

int cmd_demo(int argc, char** argv) {
    EngineOptions eo;
    eo.schema_path = argv[2];
    Engine e = build_engine(eo);
    auto workload = load_workload(argv[3]);
    const int nq = std::min<int>(std::stoi(argv[4]), int(workload.size()));
    const int threads = std::stoi(argv[5]);
    auto mem = std::make_shared<MemorySlowTier>();
    for (const auto& g : e.plan.groups) {
        std::vector<GroupTableRef<float>> refs;
        for (int id : g.tables) refs.push_back({id, std::span<const TokenId>(e.table_tokens[id])});
        for (auto& kv : encode_group<float>(e.config, e.weights, refs)) mem->put(std::move(kv));
    }
    std::vector<AnalyzedQuery> qs;
    for (int i = 0; i < nq; ++i) qs.push_back(analyze_query(e, workload[i].query_id, workload[i].text));

    std::vector<double> cached(nq), nocache(nq);
    const double wall_cached = run_sharded(nq, threads, [&](int i) {
        const double t0 = now();
        const auto order = assembly_order(e, qs[i].match_order);
        std::vector<TableKV<float>> kvs;
        for (int id : order) kvs.push_back(*mem->load(id));
        const auto ctx = assemble<float>(e.config, e.plan, kvs, order);
        const auto h = query_attend<float>(e.config, e.weights, ctx, qs[i].remainder);
        cached[i] = now() - t0;
        (void)h;
    });
    const double wall_nocache = run_sharded(nq, threads, [&](int i) {
        const double t0 = now();
        const auto order = assembly_order(e, qs[i].match_order);
        std::vector<TokenId> concat;
        BlockMask mask;
        for (int id : order) {
            concat.insert(concat.end(), e.table_tokens[id].begin(), e.table_tokens[id].end());
            mask.append_block(e.plan.group_of[id], int(e.table_tokens[id].size()));
        }
        concat.insert(concat.end(), qs[i].remainder.begin(), qs[i].remainder.end());
        mask.append_block(kQueryGroup, int(qs[i].remainder.size()));
        const auto r = prefill<float>(e.config, e.weights, concat, mask);
        nocache[i] = now() - t0;
        (void)r;
    });
    json out = {{"mode", "demo"}, {"queries", nq}, {"threads", threads},
                {"cached_p50_ms", pct(cached, 0.5) * 1e3}, {"cached_p99_ms", pct(cached, 0.99) * 1e3},
                {"nocache_p50_ms", pct(nocache, 0.5) * 1e3}, {"nocache_p99_ms", pct(nocache, 0.99) * 1e3},
                {"cached_wall_s", wall_cached}, {"nocache_wall_s", wall_nocache},
                {"cached_qps", nq / wall_cached}, {"nocache_qps", nq / wall_nocache}};
    std::cout << out.dump() << "\n";
    return 0;
}

int cmd_wide(int argc, char** argv) {
    ModelConfig cfg;
    cfg.num_layers = 1;
    cfg.num_heads = std::stoi(argv[2]);
    cfg.head_dim = std::stoi(argv[3]);
    cfg.vocab_size = 1024;  // embedding lookups are free; a small vocab keeps init cheap
    cfg.weight_seed = 1;
    const int threads = std::stoi(argv[4]);
    struct Sample { int nctx, nq; };
    std::vector<Sample> samples;
    bool cached_only = false;  // --cached-only: skip the no-cache prefill (the reference arm's metric is the cached path)
    for (int a = 5; a < argc; ++a) {
        std::string s = argv[a];
        if (s == "--cached-only") {
            cached_only = true;
            continue;
        }
        const auto c = s.find(':');
        samples.push_back({std::stoi(s.substr(0, c)), std::stoi(s.substr(c + 1))});
    }
    const double ti = now();
    const auto w = ModelWeights<float>::create(cfg);
    const double init_s = now() - ti;
    const int n = int(samples.size());
    std::vector<double> cached(n), nocache(n);
    const size_t per_tok = size_t(cfg.hidden_dim());
    SeededRng rng(7);
    std::vector<std::vector<TokenId>> toks(n);
    for (int i = 0; i < n; ++i) {
        toks[i].resize(samples[i].nctx + samples[i].nq);
        for (auto& t : toks[i]) t = TokenId(rng.next_below(cfg.vocab_size));
    }
    const double wall_cached = run_sharded(n, threads, [&](int i) {
        AssembledContext<float> ctx;
        ctx.total_tokens = samples[i].nctx;
        ctx.k.assign(1, std::vector<float>(size_t(samples[i].nctx) * per_tok, 0.01f));
        ctx.v.assign(1, std::vector<float>(size_t(samples[i].nctx) * per_tok, 0.02f));
        std::span<const TokenId> q(toks[i].data() + samples[i].nctx, samples[i].nq);
        const double t0 = now();
        const auto h = query_attend<float>(cfg, w, ctx, q);
        cached[i] = now() - t0;
        (void)h;
    });
    const double wall_nocache = cached_only ? 0.0 : run_sharded(n, threads, [&](int i) {
        BlockMask mask;
        mask.append_block(0, samples[i].nctx);
        mask.append_block(kQueryGroup, samples[i].nq);
        const double t0 = now();
        const auto r = prefill<float>(cfg, w, toks[i], mask);
        nocache[i] = now() - t0;
        (void)r;
    });
    json out = {{"mode", "wide"}, {"layers_timed", 1}, {"heads", cfg.num_heads}, {"head_dim", cfg.head_dim},
                {"threads", threads}, {"init_s", init_s}, {"cached_s", cached}, {"nocache_s", nocache},
                {"cached_wall_s", wall_cached}, {"nocache_wall_s", wall_nocache}};
    std::cout << out.dump() << "\n";
    return 0;
}

int cmd_serve(int argc, char** argv) {
    EngineOptions eo;
    eo.schema_path = argv[2];
    const double tb = now();
    Engine e = build_engine(eo);  // tokenizer, trie, plan (the default tiny model is unused here)
    auto workload = load_workload(argv[3]);
    const int threads = std::stoi(argv[4]);
    ModelConfig cfg;
    cfg.num_layers = 1;
    cfg.num_heads = std::stoi(argv[5]);
    cfg.head_dim = std::stoi(argv[6]);
    cfg.vocab_size = e.tokenizer.vocab_size();
    cfg.weight_seed = 1;
    const int nq = std::min<int>(std::stoi(argv[7]), int(workload.size()));
    if (nq <= 0 || threads <= 0) throw std::runtime_error("empty sample or no threads");
    const auto w = ModelWeights<float>::create(cfg);
    // the slow tier: one-layer KV blocks at the wide shape for every table the sample touches
    // (contents are irrelevant to the timing; shapes, ids and local offsets are the engine's)
    std::vector<char> need(e.table_count(), 0);
    for (int i = 0; i < nq; ++i)
        for (int id : analyze_query(e, workload[i].query_id, workload[i].text).match_order) need[id] = 1;
    auto mem = std::make_shared<MemorySlowTier>();
    const size_t per_tok = size_t(cfg.hidden_dim());
    for (int id = 0; id < e.table_count(); ++id) {
        if (!need[id]) continue;
        TableKV<float> kv;
        kv.table_id = id;
        kv.token_count = int(e.table_tokens[id].size());
        kv.num_layers = 1;
        kv.num_heads = cfg.num_heads;
        kv.head_dim = cfg.head_dim;
        kv.local_offset = e.local_offset[id];
        kv.k.assign(1, std::vector<float>(size_t(kv.token_count) * per_tok, 0.01f));
        kv.v.assign(1, std::vector<float>(size_t(kv.token_count) * per_tok, 0.02f));
        mem->put(std::move(kv));
    }
    const double setup_s = now() - tb;
    std::vector<double> analysis(nq), layer(nq), ctx(nq), qlen(nq);
    auto wave = [&](bool attend) {
        return run_sharded(nq, threads, [&](int i) {
            const double t0 = now();
            const auto q = analyze_query(e, workload[i].query_id, workload[i].text);
            const auto order = assembly_order(e, q.match_order);
            const double t1 = now();
            std::vector<TableKV<float>> kvs;
            for (int id : order) kvs.push_back(*mem->load(id));
            const auto c = assemble<float>(cfg, e.plan, kvs, order);
            if (attend) {
                const auto h = query_attend<float>(cfg, w, c, q.remainder);
                (void)h;
            }
            analysis[i] = t1 - t0;
            layer[i] = now() - t1;
            ctx[i] = c.total_tokens;
            qlen[i] = double(q.remainder.size());
        });
    };
    const double warm_s = wave(false);  // page-in: analysis + loads + assemble, no attention
    const double wall = wave(true);
    json out = {{"mode", "serve"}, {"layers_timed", 1}, {"heads", cfg.num_heads}, {"head_dim", cfg.head_dim},
                {"threads", threads}, {"queries", nq}, {"setup_s", setup_s}, {"warm_s", warm_s},
                {"wall_s", wall}, {"analysis_s", analysis}, {"layer_s", layer}, {"nctx", ctx}, {"nq", qlen}};
    std::cout << out.dump() << "\n";
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc >= 6 && std::string(argv[1]) == "demo") return cmd_demo(argc, argv);
        if (argc >= 6 && std::string(argv[1]) == "wide") return cmd_wide(argc, argv);
        if (argc >= 8 && std::string(argv[1]) == "serve") return cmd_serve(argc, argv);
        std::cerr << "usage: ref_bench demo <schema> <workload> <n> <threads> | wide <heads> <dim> <threads> <nctx:nq>...\n";
        return 2;
    } catch (const std::exception& ex) {
        std::cerr << "ref_bench: " << ex.what() << "\n";
        return 1;
    }
}
