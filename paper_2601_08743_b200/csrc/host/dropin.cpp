// Device bridge of the C++ drop-in API (include/tablekv/device.hpp) and the engine calls that
// need the model: precompute_corpus (engine.cpp:83-112) and verify_query (engine.cpp:174-205).
#include <cuda_runtime.h>

#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "cuda/common.cuh"
#include "cuda/kernels.cuh"
#include "cuda/model.cuh"
#include "cuda/runtime.cuh"
#include "tablekv/engine.hpp"

namespace tablekv::device {

namespace {

struct Slot {
    std::unique_ptr<tkv::Model> model;
    cudaStream_t stream = nullptr;
    std::mutex mu;  // held for a whole call: reseed + compute (the API's functions are callable from any thread)
};

std::mutex g_mu;
std::map<std::tuple<int, int, int, int, int, int, int, double, std::uint64_t, int, int, int, int>, std::unique_ptr<Slot>> g_models;

Slot& model_for(const ModelConfig& cfg, int precision) {
    int dev = 0;
    TKV_CUDA_CHECK(cudaGetDevice(&dev));
    // one device model per shape; a different weight seed regenerates the weights in place
    const auto key = std::make_tuple(dev, precision, cfg.num_layers, cfg.num_heads, cfg.kv_heads(), cfg.head_dim,
                                     cfg.vocab_size, cfg.rotary_base, std::uint64_t(0), cfg.ffn_dim(), cfg.mlp, cfg.norm, 0);
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_models[key];
    if (!slot) {
        slot = std::make_unique<Slot>();
        tkv::ModelCfg mc;
        mc.num_layers = cfg.num_layers;
        mc.num_heads = cfg.num_heads;
        mc.kv_heads = cfg.kv_heads();
        mc.head_dim = cfg.head_dim;
        mc.ffn = cfg.ffn_dim();
        mc.vocab = cfg.vocab_size;
        mc.rotary_base = cfg.rotary_base;
        mc.seed = cfg.weight_seed;
        mc.mlp = cfg.mlp;
        mc.norm = cfg.norm;
        mc.dtype = precision == 2 ? tkv::DType::f64 : tkv::DType::f32;
        TKV_CUDA_CHECK(cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking));
        slot->model = std::make_unique<tkv::Model>(mc, slot->stream);
    }
    return *slot;
}

}  // namespace

void forward(const Forward& f) {
    Slot& s = model_for(*f.cfg, f.precision);
    std::lock_guard<std::mutex> use(s.mu);
    s.model->reseed(f.cfg->weight_seed, s.stream);
    std::vector<int32_t> groups;
    if (f.groups) groups.assign(f.groups, f.groups + f.n);
    tkv::HostFwd h;
    h.tokens = f.tokens;
    h.positions = f.positions;
    h.groups = f.groups ? groups.data() : nullptr;
    h.n = f.n;
    h.mode = f.mode;
    h.n_ctx = f.n_ctx;
    h.ctx_k = f.ctx_k;
    h.ctx_v = f.ctx_v;
    h.hidden = f.hidden;
    h.kraw = f.kraw;
    h.krot = f.krot;
    h.v = f.v;
    try {
        tkv::forward_host(*s.model, s.stream, h);
    } catch (const std::invalid_argument& e) {
        throw Error(Errc::bad_config, e.what());
    }
}

void gather_f32(const ModelConfig& cfg, const std::vector<const TableKV<float>*>& tables, std::vector<std::vector<float>>& k,
                std::vector<std::vector<float>>& v) {
    const int L = cfg.num_layers;
    const int kvd = cfg.kv_heads() * cfg.head_dim;
    k.assign(size_t(L), {});
    v.assign(size_t(L), {});
    int total = 0;
    size_t pages = 0;
    constexpr size_t P = 4096;
    for (const auto* t : tables) {
        total += t->token_count;
        pages += (size_t(2) * L * t->token_count * kvd * 4 + P - 1) / P;
    }
    if (total == 0) return;
    Slot& s = model_for(cfg, 0);
    std::lock_guard<std::mutex> use(s.mu);  // the gather only uses the model's rope tables (seed-free)
    // Table images live in pageable host buffers for the length of this call (copy-engine DMA from
    // pageable memory): a pinned Arena here would pin a 256 MiB chunk per assemble() call, which
    // dominated the reference acceptance gate's 100-corpus criterion.
    tkv::PagePool pool(P, int(pages));
    std::vector<tkv::GatherSeg> segs;
    std::vector<int32_t> page_ids;
    std::vector<std::vector<float>> images(tables.size());
    int cursor = 0;
    for (size_t i = 0; i < tables.size(); ++i) {
        const auto* t = tables[i];
        if (t->token_count == 0) continue;
        auto& image = images[i];  // the .kv payload layout: K layers then V layers
        for (const auto& l : t->k) image.insert(image.end(), l.begin(), l.end());
        for (const auto& l : t->v) image.insert(image.end(), l.begin(), l.end());
        tkv::TableImage img;
        img.table_id = int(i);
        img.tokens = t->token_count;
        img.layers = L;
        img.kv_dim = kvd;
        img.local_offset = t->local_offset;
        img.dtype = tkv::DType::f32;
        img.bytes = image.size() * sizeof(float);
        img.host = reinterpret_cast<uint8_t*>(image.data());
        if (img.bytes != size_t(2) * L * t->token_count * kvd * sizeof(float))
            throw Error(Errc::dimension_mismatch, "KV block shape does not match model config");
        auto pg = pool.alloc(int((img.bytes + P - 1) / P));
        tkv::copy_table_to_pages(img, pool, pg, tkv::CopyEngine::dma, 16, s.stream);
        segs.push_back({int32_t(page_ids.size()), t->token_count, cursor, cursor});
        page_ids.insert(page_ids.end(), pg.begin(), pg.end());
        cursor += t->token_count;
    }
    tkv::Model& m = *s.model;
    m.rope().ensure(total + 1);
    const size_t ob = size_t(L) * total * kvd * 4;
    void *dk, *dv, *dseg, *dpg;
    TKV_CUDA_CHECK(cudaMalloc(&dk, ob));
    TKV_CUDA_CHECK(cudaMalloc(&dv, ob));
    TKV_CUDA_CHECK(cudaMalloc(&dseg, segs.size() * sizeof(tkv::GatherSeg)));
    TKV_CUDA_CHECK(cudaMalloc(&dpg, page_ids.size() * 4));
    TKV_CUDA_CHECK(cudaMemcpyAsync(dseg, segs.data(), segs.size() * sizeof(tkv::GatherSeg), cudaMemcpyHostToDevice, s.stream));
    TKV_CUDA_CHECK(cudaMemcpyAsync(dpg, page_ids.data(), page_ids.size() * 4, cudaMemcpyHostToDevice, s.stream));
    tkv::launch_gather_rope(pool.base(), P, static_cast<int32_t*>(dpg), static_cast<tkv::GatherSeg*>(dseg), int(segs.size()),
                            total, L, kvd, cfg.head_dim, tkv::DType::f32, tkv::DType::f32, m.rope().cos_d(), m.rope().sin_d(),
                            m.rope().cos_f(), m.rope().sin_f(), dk, dv, total, s.stream);
    std::vector<float> hk(size_t(L) * total * kvd), hv(hk.size());
    TKV_CUDA_CHECK(cudaMemcpyAsync(hk.data(), dk, ob, cudaMemcpyDeviceToHost, s.stream));
    TKV_CUDA_CHECK(cudaMemcpyAsync(hv.data(), dv, ob, cudaMemcpyDeviceToHost, s.stream));
    TKV_CUDA_CHECK(cudaStreamSynchronize(s.stream));
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dseg);
    cudaFree(dpg);
    const size_t per = size_t(total) * kvd;
    for (int l = 0; l < L; ++l) {
        k[size_t(l)].assign(hk.begin() + long(l * per), hk.begin() + long((l + 1) * per));
        v[size_t(l)].assign(hv.begin() + long(l * per), hv.begin() + long((l + 1) * per));
    }
}

void check_weights(const ModelConfig& cfg, const double* e, const double* q, int n) {
    const double sh = 1.0 / std::sqrt(double(cfg.hidden_dim()));
    for (int i = 0; i < n; ++i) {
        const double ue = u64_to_signed_unit(mix3(cfg.weight_seed, weight_tag::embedding * 131, std::uint64_t(i))) * 0.5;
        const double uq = u64_to_signed_unit(mix3(cfg.weight_seed, weight_tag::wq * 131, std::uint64_t(i))) * sh;
        const bool ok_e = e[i] == ue || e[i] == double(float(ue));
        const bool ok_q = q[i] == uq || q[i] == double(float(uq));
        if (!ok_e || !ok_q)
            throw Error(Errc::bad_config,
                        "device weights are generated from cfg.weight_seed; pass ModelWeights<Real>::create(cfg)");
    }
}

}  // namespace tablekv::device

namespace tablekv {

void precompute_corpus(const Engine& engine, const std::string& cache_dir) {
    namespace fs = std::filesystem;
    const fs::path final_dir(cache_dir), tmp(cache_dir + ".tmp");
    std::error_code ec;
    fs::remove_all(tmp, ec);
    if (!fs::create_directories(tmp)) throw Error(Errc::io_error, "cannot create directory " + tmp.string());
    try {
        const auto weights = ModelWeights<float>::create(engine.config);
        for (const auto& g : engine.plan.groups) {
            std::vector<GroupTableRef<float>> refs;
            for (int id : g.tables) refs.push_back({id, std::span<const TokenId>(engine.table_tokens[size_t(id)])});
            for (const auto& kv : encode_group<float>(engine.config, weights, refs))
                save_table_kv((tmp / (std::to_string(kv.table_id) + ".kv")).string(), kv);
        }
        std::ofstream mf(tmp / "manifest.json", std::ios::binary);
        if (!mf) throw Error(Errc::io_error, "cannot write manifest");
        mf << manifest_json(engine);
        mf.close();
        fs::remove_all(final_dir, ec);
        fs::rename(tmp, final_dir);
    } catch (...) {
        fs::remove_all(tmp, ec);
        throw;
    }
}

double verify_query(const Engine& engine, SlowTier& slow, const AnalyzedQuery& q) {
    const auto order = assembly_order(engine, q.match_order);
    std::vector<TableKV<float>> kvs;
    for (int id : order) kvs.push_back(*slow.load(id));
    const auto weights = ModelWeights<float>::create(engine.config);
    const auto ctx = assemble<float>(engine.config, engine.plan, kvs, order);
    const auto served = query_attend<float>(engine.config, weights, ctx, q.remainder);
    std::vector<TokenId> concat;
    BlockMask mask;
    for (int id : order) {
        const auto& tt = engine.table_tokens[size_t(id)];
        concat.insert(concat.end(), tt.begin(), tt.end());
        mask.append_block(engine.plan.group_of[size_t(id)], int(tt.size()));
    }
    concat.insert(concat.end(), q.remainder.begin(), q.remainder.end());
    mask.append_block(kQueryGroup, int(q.remainder.size()));
    const auto oracle = prefill<float>(engine.config, weights, concat, mask);
    const size_t h = size_t(engine.config.hidden_dim()), ctx_tokens = concat.size() - q.remainder.size();
    double worst = 0.0;
    for (size_t i = 0; i < q.remainder.size() * h; ++i)
        worst = std::max(worst, std::abs(double(served[i]) - double(oracle.hidden[ctx_tokens * h + i])));
    return worst;
}

}  // namespace tablekv
