// tablekv B200 build — the model calls of the serving path (drop-in for
// proj/include/tablekv/attention.hpp:19-414), executed on the GPU.
//
// prefill / encode_group / query_attend run the device forward (tablekv::device::forward):
// Real = float uses the reference-precision kernels with float storage, Real = double the same
// kernels with double storage (both accumulate in double like the reference). assemble<float>
// gathers and re-rotates on the GPU (bit-identical to the reference); assemble<double> rotates on
// the host. Host-side validation (mask, dimensions, group order, vocabulary) is the reference's.
// The weights argument must be ModelWeights<Real>::create(cfg): the device regenerates weights
// from cfg.weight_seed and checks a probe of the given ones.
#pragma once

#include <algorithm>
#include <cstdint>
#include <span>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "tablekv/device.hpp"
#include "tablekv/errors.hpp"
#include "tablekv/model.hpp"
#include "tablekv/rotary.hpp"
#include "tablekv/schema.hpp"
#include "tablekv/table_kv.hpp"
#include "tablekv/types.hpp"

namespace tablekv {

constexpr int kQueryGroup = -1;

struct BlockMask {
    std::vector<int> group;
    std::vector<int64_t> position;

    void append_block(int group_id, int token_count) {
        for (int i = 0; i < token_count; ++i) {
            position.push_back(int64_t(position.size()));
            group.push_back(group_id);
        }
    }
    bool allows(size_t i, size_t j) const { return j <= i && (group[i] == kQueryGroup || group[i] == group[j]); }
    void validate(size_t token_count) const {
        if (group.size() != token_count || position.size() != token_count)
            throw Error(Errc::dimension_mismatch, "mask does not cover all tokens");
        for (size_t i = 1; i < position.size(); ++i)
            if (position[i] <= position[i - 1]) throw Error(Errc::dimension_mismatch, "mask positions must be strictly increasing");
    }
};

template <typename Real>
struct PrefillResult {
    std::vector<std::vector<Real>> k_raw, k_rot, v;
    std::vector<Real> hidden;
};

template <typename Real>
struct AssembledContext {
    struct Span {
        int table_id;
        int start;
        int end;
    };
    int total_tokens = 0;
    std::vector<std::vector<Real>> k, v;
    std::vector<Span> span_index;
};

template <typename Real>
struct GroupTableRef {
    int table_id;
    std::span<const TokenId> tokens;
};

namespace attn_detail {

template <typename Real>
constexpr int precision() {
    static_assert(std::is_same_v<Real, float> || std::is_same_v<Real, double>, "Real must be float or double");
    return std::is_same_v<Real, double> ? 2 : 0;
}

template <typename Real>
void probe_weights(const ModelConfig& cfg, const ModelWeights<Real>& w) {
    const int n = int(std::min<size_t>({4, w.embedding.size(), w.layers.empty() ? 0 : w.layers[0].wq.size()}));
    double e[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
    for (int i = 0; i < n; ++i) e[i] = double(w.embedding[size_t(i)]), q[i] = double(w.layers[0].wq[size_t(i)]);
    device::check_weights(cfg, e, q, n);
}

template <typename Real>
void check_vocab(const ModelConfig& cfg, std::span<const TokenId> tokens) {
    for (TokenId t : tokens)
        if (t < 0 || t >= cfg.vocab_size) throw Error(Errc::bad_config, "token id " + std::to_string(t) + " outside vocabulary");
}

template <typename Real>
std::vector<std::vector<Real>> split_layers(const std::vector<Real>& flat, int L, size_t per_layer) {
    std::vector<std::vector<Real>> out(static_cast<size_t>(L));
    for (int l = 0; l < L; ++l) out[size_t(l)].assign(flat.begin() + long(size_t(l) * per_layer), flat.begin() + long(size_t(l + 1) * per_layer));
    return out;
}

}  // namespace attn_detail

template <typename Real>
PrefillResult<Real> prefill(const ModelConfig& cfg, const ModelWeights<Real>& w, std::span<const TokenId> tokens,
                            const BlockMask& mask) {
    cfg.validate();
    mask.validate(tokens.size());
    attn_detail::probe_weights(cfg, w);
    attn_detail::check_vocab<Real>(cfg, tokens);
    PrefillResult<Real> r;
    const int L = cfg.num_layers, n = int(tokens.size());
    const size_t kvd = size_t(cfg.kv_heads()) * size_t(cfg.head_dim), per = size_t(n) * kvd;
    r.k_raw.assign(size_t(L), {});
    r.k_rot.assign(size_t(L), {});
    r.v.assign(size_t(L), {});
    if (n == 0) return r;
    std::vector<Real> kraw(size_t(L) * per), krot(kraw.size()), vv(kraw.size());
    r.hidden.resize(size_t(n) * size_t(cfg.hidden_dim()));
    device::Forward f;
    f.cfg = &cfg;
    f.precision = attn_detail::precision<Real>();
    f.tokens = tokens.data();
    f.n = n;
    f.positions = mask.position.data();
    f.groups = mask.group.data();
    f.mode = 1;
    f.hidden = r.hidden.data();
    f.kraw = kraw.data();
    f.krot = krot.data();
    f.v = vv.data();
    device::forward(f);
    r.k_raw = attn_detail::split_layers(kraw, L, per);
    r.k_rot = attn_detail::split_layers(krot, L, per);
    r.v = attn_detail::split_layers(vv, L, per);
    return r;
}

template <typename Real>
std::vector<TableKV<Real>> encode_group(const ModelConfig& cfg, const ModelWeights<Real>& w,
                                        std::span<const GroupTableRef<Real>> tables) {
    if (tables.empty()) throw Error(Errc::empty_group, "encode_group called with no tables");
    std::vector<TokenId> all;
    for (const auto& t : tables) {
        if (t.tokens.empty()) throw Error(Errc::empty_group, "table " + std::to_string(t.table_id) + " has no tokens");
        all.insert(all.end(), t.tokens.begin(), t.tokens.end());
    }
    BlockMask mask;
    mask.append_block(0, int(all.size()));
    const PrefillResult<Real> full = prefill<Real>(cfg, w, all, mask);
    const size_t kvd = size_t(cfg.kv_heads()) * size_t(cfg.head_dim);
    std::vector<TableKV<Real>> out;
    size_t at = 0;
    for (const auto& t : tables) {
        TableKV<Real> kv;
        kv.table_id = t.table_id;
        kv.token_count = int(t.tokens.size());
        kv.num_layers = cfg.num_layers;
        kv.num_heads = cfg.kv_heads();
        kv.head_dim = cfg.head_dim;
        kv.local_offset = int(at);
        for (int l = 0; l < cfg.num_layers; ++l) {
            const auto& kr = full.k_raw[size_t(l)];
            const auto& vv = full.v[size_t(l)];
            kv.k.emplace_back(kr.begin() + long(at * kvd), kr.begin() + long((at + t.tokens.size()) * kvd));
            kv.v.emplace_back(vv.begin() + long(at * kvd), vv.begin() + long((at + t.tokens.size()) * kvd));
        }
        out.push_back(std::move(kv));
        at += t.tokens.size();
    }
    return out;
}

template <typename Real>
AssembledContext<Real> assemble(const ModelConfig& cfg, const EncodingPlan& plan, std::span<const TableKV<Real>> table_kvs,
                                std::span<const int> order) {
    std::unordered_map<int, const TableKV<Real>*> by_id;
    for (const auto& kv : table_kvs) by_id[kv.table_id] = &kv;
    std::unordered_map<int, int> last_in_group;
    std::vector<const TableKV<Real>*> picked;
    for (int id : order) {
        const auto it = by_id.find(id);
        if (it == by_id.end()) throw Error(Errc::missing_table_kv, "no precomputed KV for table " + std::to_string(id));
        const TableKV<Real>* kv = it->second;
        if (kv->num_layers != cfg.num_layers || kv->num_heads != cfg.kv_heads() || kv->head_dim != cfg.head_dim)
            throw Error(Errc::dimension_mismatch, "KV block shape does not match model config for table " + std::to_string(id));
        if (id < 0 || id >= int(plan.group_of.size())) throw Error(Errc::bad_config, "table " + std::to_string(id) + " not in plan");
        const auto [g, fresh] = last_in_group.try_emplace(plan.group_of[size_t(id)], kv->local_offset);
        if (!fresh) {
            if (kv->local_offset <= g->second)
                throw Error(Errc::group_order_violation,
                            "table " + std::to_string(id) + " appears out of group-relative order in the assembly");
            g->second = kv->local_offset;
        }
        picked.push_back(kv);
    }
    AssembledContext<Real> ctx;
    int cursor = 0;
    for (const auto* kv : picked) {
        ctx.span_index.push_back({kv->table_id, cursor, cursor + kv->token_count});
        cursor += kv->token_count;
    }
    ctx.total_tokens = cursor;
    if constexpr (std::is_same_v<Real, float>) {
        device::gather_f32(cfg, picked, ctx.k, ctx.v);  // GPU gather + RoPE
    } else {
        ctx.k.assign(size_t(cfg.num_layers), {});
        ctx.v.assign(size_t(cfg.num_layers), {});
        int at = 0;
        std::vector<int64_t> pos;
        for (const auto* kv : picked) {
            pos.resize(size_t(kv->token_count));
            for (int t = 0; t < kv->token_count; ++t) pos[size_t(t)] = at + t;
            for (int l = 0; l < cfg.num_layers; ++l) {
                const auto rk = rotated_copy<Real>(kv->k[size_t(l)], pos, kv->num_heads, cfg.head_dim, cfg.rotary_base);
                ctx.k[size_t(l)].insert(ctx.k[size_t(l)].end(), rk.begin(), rk.end());
                ctx.v[size_t(l)].insert(ctx.v[size_t(l)].end(), kv->v[size_t(l)].begin(), kv->v[size_t(l)].end());
            }
            at += kv->token_count;
        }
    }
    return ctx;
}

template <typename Real>
std::vector<Real> query_attend(const ModelConfig& cfg, const ModelWeights<Real>& w, const AssembledContext<Real>& ctx,
                               std::span<const TokenId> query_tokens) {
    cfg.validate();
    attn_detail::probe_weights(cfg, w);
    attn_detail::check_vocab<Real>(cfg, query_tokens);
    const int L = cfg.num_layers, n = int(query_tokens.size()), nctx = ctx.total_tokens;
    const size_t kvd = size_t(cfg.kv_heads()) * size_t(cfg.head_dim);
    std::vector<Real> hidden(size_t(n) * size_t(cfg.hidden_dim()));
    if (n == 0) return hidden;
    std::vector<Real> ck, cv;
    if (nctx > 0) {
        ck.reserve(size_t(L) * size_t(nctx) * kvd);
        cv.reserve(ck.capacity());
        for (int l = 0; l < L; ++l) {
            if (ctx.k[size_t(l)].size() != size_t(nctx) * kvd)
                throw Error(Errc::dimension_mismatch, "assembled context shape mismatch");
            ck.insert(ck.end(), ctx.k[size_t(l)].begin(), ctx.k[size_t(l)].end());
            cv.insert(cv.end(), ctx.v[size_t(l)].begin(), ctx.v[size_t(l)].end());
        }
    }
    device::Forward f;
    f.cfg = &cfg;
    f.precision = attn_detail::precision<Real>();
    f.tokens = query_tokens.data();
    f.n = n;
    f.mode = 0;
    f.ctx_k = nctx ? ck.data() : nullptr;
    f.ctx_v = nctx ? cv.data() : nullptr;
    f.n_ctx = nctx;
    f.hidden = hidden.data();
    device::forward(f);
    return hidden;
}

}  // namespace tablekv
