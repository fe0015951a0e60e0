// Device model: weight init + the prefill forward in two precisions.
//   bf16 (performance path): tcgen05 GEMMs with fused RoPE / SiLU|SwiGLU / residual epilogues,
//     tensor-core attention over [cached prefix ; own rows], f32 residual stream.
//   f32 / f64 (reference-precision path): the SIMT kernels of simt.cu, operation-for-operation
//     the reference's arithmetic (attention.hpp:210-247 and :368-414).
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "model.cuh"
#include "norm.cuh"

namespace tkv {

// ------------------------------------------------------------------ StagingRing
// Per-window metadata (tokens, positions, sequences, segments, page ids, tiles) reaches the device
// through a pinned, device-mapped ring copied by a small SM kernel on the compute stream — NOT by
// cudaMemcpyAsync: the copy engines are busy with the next window's multi-GB KV page copies, and a
// DMA upload queued behind them stalled the window's whole prefill until those copies finished
// (~100 ms per batch at C4: profiles/r2/executor_window_timeline_*).
namespace {
__global__ void stage_copy_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t n) {
    const size_t n16 = n / 16;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    if (blockIdx.x == 0 && threadIdx.x < n % 16) dst[n16 * 16 + threadIdx.x] = src[n16 * 16 + threadIdx.x];
}
}  // namespace

StagingRing::StagingRing(size_t bytes) : cap_(bytes) {
    TKV_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&host_), bytes, cudaHostAllocMapped));
    TKV_CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped_), host_, 0));
    TKV_CUDA_CHECK(cudaMalloc(reinterpret_cast<void**>(&dev_), bytes));
}

StagingRing::~StagingRing() {
    cudaFreeHost(host_);
    cudaFree(dev_);
}

// Uploads are lazy: the bytes land in the pinned ring now and the device pointer is returned at once;
// flush() copies everything uploaded since the last flush with ONE kernel (the uploads of a window
// are contiguous in the ring), right before the first kernel that reads them.
void* StagingRing::upload(const void* src, size_t bytes, cudaStream_t s) {
    const size_t n = (bytes + 255) & ~size_t(255);  // keep every chunk 256-byte aligned
    if (off_ + n > cap_) flush(s);  // (reserve may wrap: nothing may stay pending across it)
    reserve(n);
    if (bytes) {
        std::memcpy(host_ + off_, src, bytes);
        if (pend_end_ == pend_begin_) pend_begin_ = off_;
        pend_end_ = off_ + bytes;
    }
    void* d = dev_ + off_;
    off_ += n;
    return d;
}

void StagingRing::flush(cudaStream_t s) {
    if (pend_end_ == pend_begin_) return;
    const size_t bytes = pend_end_ - pend_begin_;
    const int blocks = int(std::min<size_t>(148, (bytes / 16 + 255) / 256 + 1));
    stage_copy_kernel<<<blocks, 256, 0, s>>>(dev_ + pend_begin_, mapped_ + pend_begin_, bytes);
    TKV_CUDA_CHECK(cudaGetLastError());
    ++launches_;
    pend_begin_ = pend_end_ = 0;
}

void StagingRing::reserve(size_t n) {
    if (n > cap_) throw std::runtime_error("staging ring too small for one upload");
    if (off_ + n > cap_) {
        // wrap: every earlier chunk may still be read by queued work
        TKV_CUDA_CHECK(cudaDeviceSynchronize());
        off_ = 0;
    }
}

// ------------------------------------------------------------------ RopeTables
RopeTables::RopeTables(int head_dim, double base) : d_(head_dim), base_(base) {}

RopeTables::~RopeTables() {
    cudaFree(cos_d_);
    cudaFree(sin_d_);
    cudaFree(cos_f_);
    cudaFree(sin_f_);
}

void RopeTables::ensure(int max_pos) {
    if (max_pos <= max_pos_) return;
    int cap = std::max(4096, max_pos_);
    while (cap < max_pos) cap *= 2;
    TKV_CUDA_CHECK(cudaDeviceSynchronize());
    cudaFree(cos_d_);
    cudaFree(sin_d_);
    cudaFree(cos_f_);
    cudaFree(sin_f_);
    const int half = d_ / 2;
    std::vector<double> inv(half), cd(size_t(cap) * half), sd(size_t(cap) * half);
    std::vector<float> cf(cd.size()), sf(cd.size());
    for (int k = 0; k < half; ++k) inv[k] = std::pow(base_, -2.0 * k / d_);
    for (long p = 0; p < cap; ++p)
        for (int k = 0; k < half; ++k) {
            const double angle = double(p) * inv[k];
            cd[p * half + k] = std::cos(angle);
            sd[p * half + k] = std::sin(angle);
            cf[p * half + k] = float(cd[p * half + k]);
            sf[p * half + k] = float(sd[p * half + k]);
        }
    TKV_CUDA_CHECK(cudaMalloc(&cos_d_, cd.size() * 8));
    TKV_CUDA_CHECK(cudaMalloc(&sin_d_, cd.size() * 8));
    TKV_CUDA_CHECK(cudaMalloc(&cos_f_, cd.size() * 4));
    TKV_CUDA_CHECK(cudaMalloc(&sin_f_, cd.size() * 4));
    TKV_CUDA_CHECK(cudaMemcpy(cos_d_, cd.data(), cd.size() * 8, cudaMemcpyHostToDevice));
    TKV_CUDA_CHECK(cudaMemcpy(sin_d_, sd.data(), sd.size() * 8, cudaMemcpyHostToDevice));
    TKV_CUDA_CHECK(cudaMemcpy(cos_f_, cf.data(), cf.size() * 4, cudaMemcpyHostToDevice));
    TKV_CUDA_CHECK(cudaMemcpy(sin_f_, sf.data(), sf.size() * 4, cudaMemcpyHostToDevice));
    max_pos_ = cap;
}

// ------------------------------------------------------------------ Model
namespace {
// weight tags (model.hpp:36-44) + extensions: 8 = untied LM head, 9 = SwiGLU gate
constexpr uint64_t kEmb = 1, kWq = 2, kWk = 3, kWv = 4, kWo = 5, kIn = 6, kOut = 7, kHead = 8, kGate = 9;
}  // namespace

Model::Model(const ModelCfg& cfg, cudaStream_t s) : cfg_(cfg), rope_(cfg.head_dim, cfg.rotary_base), ring_(64u << 20) {
    if (cfg.num_heads % cfg.kv_heads) throw std::invalid_argument("num_heads must be a multiple of kv_heads");
    if (cfg.head_dim % 2) throw std::invalid_argument("head_dim must be even for rotary pairs");
    if (cfg.vocab <= 0) throw std::invalid_argument("vocab must be positive");
    alloc_weights(s);
    rope_.ensure(8192);
    // TKV_ATTN=mma forces the mma.sync attention kernel everywhere (A/B measurements)
    if (const char* e = std::getenv("TKV_ATTN"); e && std::string(e) == "mma") attn_impl_ = 1;
}

Model::~Model() {
    cudaDeviceSynchronize();
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
    for (void* p : allocs_) cudaFree(p);
    cudaFree(ws_);
}

void Model::alloc_weights(cudaStream_t s) {
    const ModelCfg& c = cfg_;
    const long h = c.hidden(), kvd = c.kv_dim(), f = c.ffn, qd = long(c.num_heads) * c.head_dim;
    const size_t es = dtype_size(c.dtype);
    size_t next = 0;
    const bool refill = !allocs_.empty();  // reseed(): same buffers, new counter-hash values
    auto alloc = [&](long elems) {
        if (refill) return allocs_[next++];
        void* p = nullptr;
        TKV_CUDA_CHECK(cudaMalloc(&p, size_t(elems) * es));
        allocs_.push_back(p);
        weight_bytes_ += size_t(elems) * es;
        return p;
    };
    const double sh = 1.0 / std::sqrt(double(h)), sf = 1.0 / std::sqrt(double(f));
    emb_ = alloc(long(c.vocab) * h);
    launch_fill_matrix(emb_, c.dtype, c.vocab, h, 0, c.seed, kEmb * 131, 0.5, 0, 0, s);
    layers_.resize(c.num_layers);
    for (int l = 0; l < c.num_layers; ++l) {
        Layer& L = layers_[l];
        if (c.dtype == DType::bf16) {
            L.wqkv = alloc((qd + 2 * kvd) * h);
            launch_fill_matrix(L.wqkv, c.dtype, qd, h, 0, c.seed, kWq * 131 + l, sh, 0, 0, s);
            launch_fill_matrix(L.wqkv, c.dtype, kvd, h, qd, c.seed, kWk * 131 + l, sh, 0, 0, s);
            launch_fill_matrix(L.wqkv, c.dtype, kvd, h, qd + kvd, c.seed, kWv * 131 + l, sh, 0, 0, s);
            if (c.mlp == 1) {  // [gate 16 | up 16] row blocks for the fused SwiGLU epilogue
                L.w_in = alloc(2 * f * h);
                launch_fill_matrix(L.w_in, c.dtype, f, h, 0, c.seed, kGate * 131 + l, sh, 16, 0, s);
                launch_fill_matrix(L.w_in, c.dtype, f, h, 0, c.seed, kIn * 131 + l, sh, 16, 1, s);
            } else {
                L.w_in = alloc(f * h);
                launch_fill_matrix(L.w_in, c.dtype, f, h, 0, c.seed, kIn * 131 + l, sh, 0, 0, s);
            }
        } else {
            L.wq = alloc(qd * h);
            L.wk = alloc(kvd * h);
            L.wv = alloc(kvd * h);
            launch_fill_matrix(L.wq, c.dtype, qd, h, 0, c.seed, kWq * 131 + l, sh, 0, 0, s);
            launch_fill_matrix(L.wk, c.dtype, kvd, h, 0, c.seed, kWk * 131 + l, sh, 0, 0, s);
            launch_fill_matrix(L.wv, c.dtype, kvd, h, 0, c.seed, kWv * 131 + l, sh, 0, 0, s);
            L.w_in = alloc(f * h);
            launch_fill_matrix(L.w_in, c.dtype, f, h, 0, c.seed, kIn * 131 + l, sh, 0, 0, s);
            if (c.mlp == 1) {
                L.w_gate = alloc(f * h);
                launch_fill_matrix(L.w_gate, c.dtype, f, h, 0, c.seed, kGate * 131 + l, sh, 0, 0, s);
            }
        }
        L.wo = alloc(h * qd);
        launch_fill_matrix(L.wo, c.dtype, h, qd, 0, c.seed, kWo * 131 + l, sh, 0, 0, s);
        L.w_out = alloc(h * f);
        launch_fill_matrix(L.w_out, c.dtype, h, f, 0, c.seed, kOut * 131 + l, sf, 0, 0, s);
    }
    const long vp = c.dtype == DType::bf16 ? c.vocab_padded() : c.vocab;
    head_ = alloc(vp * h);
    TKV_CUDA_CHECK(cudaMemsetAsync(head_, 0, size_t(vp * h) * es, s));
    launch_fill_matrix(head_, c.dtype, c.vocab, h, 0, c.seed, kHead * 131, sh, 0, 0, s);
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
}

void Model::reseed(uint64_t seed, cudaStream_t s) {
    if (seed == cfg_.seed) return;
    cfg_.seed = seed;
    alloc_weights(s);
}

void Model::ensure_ws(int M, cudaStream_t s) {
    if (M <= ws_rows_) return;
    int cap = std::max(256, ws_rows_);
    while (cap < M) cap *= 2;
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFree(ws_);
    const ModelCfg& c = cfg_;
    const size_t es = dtype_size(c.dtype);
    const long h = c.hidden(), qd = long(c.num_heads) * c.head_dim, kvd = c.kv_dim(), f = c.ffn;
    // x (f32 or T), xn, q, k, v, attn, proj (T), mid (f), gate (f)
    // + the folded norm's sum-of-squares partials (h / 128 floats)
    const size_t per_row = size_t(h) * std::max<size_t>(4, es) + (h + qd + 2 * kvd + qd + h) * es + 2 * size_t(f) * es + 64 +
                           size_t(h / 128 + 4) * 4;
    TKV_CUDA_CHECK(cudaMalloc(&ws_, per_row * cap + 4096));
    TKV_CUDA_CHECK(cudaMemsetAsync(ws_, 0, per_row * cap + 4096, s));  // finite padding rows for masked tiles
    ws_rows_ = cap;
}

void Model::forward(const FwdArgs& a, cudaStream_t s) {
    if (a.M == 0) return;
    ensure_ws(a.M, s);
    if (cfg_.dtype == DType::bf16) {
        forward_bf16(a, s);  // flushes the staging ring after its own uploads
    } else {
        ring_.flush(s);
        forward_ref(a, s);
    }
}

cudaEvent_t Model::timing_event() {
    if (ev_used_ == ev_pool_.size()) {
        cudaEvent_t e;
        TKV_CUDA_CHECK(cudaEventCreate(&e));
        ev_pool_.push_back(e);
    }
    return ev_pool_[ev_used_++];
}

void Model::add_timed(cudaEvent_t a, cudaEvent_t b, double flops) {
    timed_.push_back({a, b, flops < 0 ? -flops : flops, flops < 0 ? 2 : (flops == 0 ? 1 : 0)});
}

void Model::collect_timing(double& gemm_ms, double& gemm_flops, double& gather_ms, double& attn_ms, double& gather_bytes) {
    gemm_ms = gemm_flops = gather_ms = attn_ms = gather_bytes = 0;
    static const char* dump = std::getenv("TKV_DUMP_TIMING");  // debug: every timed launch (kind, start, end ms)
    if (dump && !timed_.empty())
        if (FILE* f = std::fopen(dump, "a")) {
            for (const TimedRec& r : timed_) {
                float a0 = 0, a1 = 0;
                cudaEventElapsedTime(&a0, timed_.front().a, r.a);
                cudaEventElapsedTime(&a1, timed_.front().a, r.b);
                std::fprintf(f, "%d %.4f %.4f %.0f\n", r.kind, a0, a1, r.flops);
            }
            std::fprintf(f, "--\n");
            std::fclose(f);
        }
    for (const TimedRec& r : timed_) {
        float ms = 0;
        TKV_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
        if (r.kind == 0) gemm_ms += ms, gemm_flops += r.flops;
        else if (r.kind == 1) attn_ms += ms;
        else gather_ms += ms, gather_bytes += r.flops;
    }
    timed_.clear();
    ev_used_ = 0;
}

void Model::forward_bf16(const FwdArgs& a, cudaStream_t s) {
    const ModelCfg& c = cfg_;
    const int M = a.M, h = c.hidden(), qd = c.num_heads * c.head_dim, kvd = c.kv_dim(), f = c.ffn;
    const int rms = c.norm == 1;
    const float eps = float(c.eps);
    uint8_t* p = static_cast<uint8_t*>(ws_);
    auto take = [&](size_t bytes) {
        void* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    const long R = ws_rows_;
    float* x = static_cast<float*>(take(size_t(R) * h * 4));
    void* xn = take(size_t(R) * h * 2);
    void* q = take(size_t(R) * qd * 2);
    void* k = take(size_t(R) * kvd * 2);
    void* v = take(size_t(R) * kvd * 2);
    void* att = take(size_t(R) * qd * 2);
    void* mid = take(size_t(R) * f * 2);
    float* ssq = static_cast<float*>(take(size_t(R) * (h / 128 + 4) * 4));
    // RMSNorm folded into the GEMMs (gemm_tc.cuh EpiParams): the O / down projections' epilogues
    // write bf16(x) into xn plus per-128-column sums of squares, the next projection scales its
    // accumulator rows; no norm kernel inside the layer stack. TKV_NORM_FOLD=0: separate norms.
    static const bool fold_env = [] {
        const char* e = std::getenv("TKV_NORM_FOLD");
        return !(e && std::atoi(e) == 0);
    }();
    const bool fold = fold_env && rms && h % 512 == 0;
    auto fold_in = [&](EpiParams& e, bool on) {
        if (!on) return;
        e.ss_in = ssq;
        e.ss_chunks = h / 128;
        e.ss_n = float(h);
        e.eps = eps;
    };
    auto fold_out = [&](EpiParams& e, bool on) {
        if (!on) return;
        e.xb_out = xn;
        e.ss_out = ssq;
    };

    // attention work list: (seq, first token, kv head)
    // tcgen05 attention over cached prefixes at head_dim 128 (the Llama-shaped serving path); the
    // mma.sync kernel for other head dims and for block-mask prefill (mode 1: its per-key group
    // test runs cheaper there)
    const int G = c.num_heads / c.kv_heads;
    // block-causal prefill (mode 1) runs on the tcgen05 kernel when every sequence's group ids form
    // contiguous blocks (the prompt layout of prefill / encode_group): row i then sees own keys
    // [start of its block, i], or [0, i] for query rows (group -1)
    const int32_t* d_row_lo = nullptr;
    if (a.mode == 1 && a.group_host && attn_impl_ == 0 && c.head_dim == 128 && 128 % G == 0) {
        std::vector<int32_t> lo(static_cast<size_t>(M), 0);
        bool contiguous = true;
        for (int si = 0; si < a.n_seqs && contiguous; ++si) {
            const AttnSeq& q = a.seqs_host[si];
            std::vector<int32_t> seen;
            int start = 0;
            for (int i = 0; i < q.n_own; ++i) {
                const int32_t g = a.group_host[q.q_row0 + i];
                if (i == 0 || g != a.group_host[q.q_row0 + i - 1]) {
                    start = i;
                    if (g != -1) {
                        if (std::find(seen.begin(), seen.end(), g) != seen.end()) contiguous = false;
                        seen.push_back(g);
                    }
                }
                lo[size_t(q.q_row0 + i)] = g == -1 ? 0 : start;
            }
        }
        if (contiguous) d_row_lo = static_cast<const int32_t*>(ring_.upload(lo.data(), lo.size() * 4, s));
    }
    const bool use_tc5 = attn_impl_ == 0 && c.head_dim == 128 && 128 % G == 0 && (a.mode == 0 || d_row_lo != nullptr);
    // paged prefix (the serving default): the tcgen05 attention reads cached K and V straight from
    // the pool pages by TMA and rotates K in shared memory — no gather, no prefix slab. Needs bf16
    // images and power-of-two pages holding whole token rows; else (or TKV_PAGED_K / TKV_PAGED_V =
    // 0) the gather writes rotated K and V into the one-layer slab first.
    const size_t kv_row_bytes = size_t(kvd) * 2;
    auto pow2 = [](size_t v) { return v && !(v & (v - 1)); };
    const bool paged = a.paged_v && a.paged_k && use_tc5 && a.mode == 0 && a.gather_segs && a.gather_in == DType::bf16 &&
                       a.gather_pool_bytes > 0 && pow2(a.gather_page_bytes) && pow2(kv_row_bytes) &&
                       a.gather_page_bytes % kv_row_bytes == 0;
    const int tq = use_tc5 ? attn_tc5_rows_per_tile(c.num_heads, c.kv_heads) : attn_rows_per_tile(c.num_heads, c.kv_heads);
    std::vector<int4> tiles;
    for (int si = 0; si < a.n_seqs; ++si)
        for (int t0 = 0; t0 < a.seqs_host[si].n_own; t0 += tq)
            for (int kh = 0; kh < c.kv_heads; ++kh) tiles.push_back(make_int4(si, t0, kh, 0));
    if (use_tc5)  // persistent kernel walks the list round-robin: heaviest items first balances the SMs
        std::stable_sort(tiles.begin(), tiles.end(), [&](const int4& x, const int4& y) {
            auto cost = [&](const int4& w) {
                const AttnSeq& q = a.seqs_host[w.x];
                return (q.n_ctx + 63) / 64 + (std::min(q.n_own, w.y + tq) + 63) / 64;
            };
            return cost(x) > cost(y);
        });
    const int4* d_tiles = tiles.empty() ? nullptr
                                        : static_cast<const int4*>(ring_.upload(tiles.data(), tiles.size() * sizeof(int4), s));
    long nl = 0;
    auto run_gemm = [&](const void* A, const void* B, int m, int n, int k, const EpiParams& e) {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing_) {
            e0 = timing_event();
            e1 = timing_event();
            TKV_CUDA_CHECK(cudaEventRecord(e0, s));
        }
        gemm_bf16(A, B, m, n, k, e, s);
        if (timing_) {
            TKV_CUDA_CHECK(cudaEventRecord(e1, s));
            add_timed(e0, e1, 2.0 * m * n * double(k));
        }
    };

    ring_.flush(s);  // every metadata upload of this forward (and the caller's) reaches HBM here
    embed_norm_bf16(emb_, a.tokens, M, h, x, xn, rms, eps, s);
    ++nl;
    for (int l = 0; l < c.num_layers; ++l) {
        const Layer& L = layers_[l];
        void* v_l = a.v_out ? static_cast<uint8_t*>(a.v_out) + size_t(l) * M * kvd * 2 : v;
        EpiParams e;
        e.kind = Epi::qkv_rope;
        e.q_out = q;
        e.k_out = k;
        e.v_out = v_l;
        e.k_raw_out = a.kraw_out ? static_cast<uint8_t*>(a.kraw_out) + size_t(l) * M * kvd * 2 : nullptr;
        e.q_cols = qd;
        e.kv_cols = kvd;
        e.head_dim = c.head_dim;
        e.pos = a.pos;
        e.cos_f = rope_.cos_f();
        e.sin_f = rope_.sin_f();
        fold_in(e, fold && l > 0);  // layer 0 reads the embedding's normalised rows
        run_gemm(xn, L.wqkv, M, qd + 2 * kvd, h, e);

        AttnArgs aa;
        aa.q = static_cast<const __nv_bfloat16*>(q);
        aa.k_own = static_cast<const __nv_bfloat16*>(k);
        aa.v_own = static_cast<const __nv_bfloat16*>(v_l);
        const bool streamed = a.gather_segs != nullptr;
        if (a.layer_ready && a.layer_ready[l]) TKV_CUDA_CHECK(cudaStreamWaitEvent(s, a.layer_ready[l]));
        if (streamed && !paged) {
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (timing_) {
                e0 = timing_event();
                e1 = timing_event();
                TKV_CUDA_CHECK(cudaEventRecord(e0, s));
            }
            if (a.gather_chunks && a.gather_in == DType::bf16 && !(a.gather_page_bytes & (a.gather_page_bytes - 1)))
                launch_gather_rope_bf16(a.gather_pool, a.gather_page_bytes, a.gather_pages, a.gather_segs, a.gather_chunks,
                                        a.gather_n_chunks, c.num_layers, l, kvd, c.head_dim, rope_.cos_f(), rope_.sin_f(),
                                        const_cast<void*>(a.ctx_k), const_cast<void*>(a.ctx_v), a.ctx_rows, s);
            else
                launch_gather_rope(a.gather_pool, a.gather_page_bytes, a.gather_pages, a.gather_segs, a.gather_n_segs,
                                   a.gather_rows, c.num_layers, kvd, c.head_dim, a.gather_in, DType::bf16, rope_.cos_d(),
                                   rope_.sin_d(), rope_.cos_f(), rope_.sin_f(), const_cast<void*>(a.ctx_k),
                                   const_cast<void*>(a.ctx_v), a.ctx_rows, s, l, 1);
            ++nl;
            if (timing_) {
                TKV_CUDA_CHECK(cudaEventRecord(e1, s));
                // algorithmic bytes: each prefix row's K and V read from the pages + written
                const double in_b = a.gather_in == DType::bf16 ? 2.0 : 4.0;
                add_timed(e0, e1, -double(a.ctx_rows) * kvd * 2 * (in_b + 2.0));
            }
        }
        const size_t ctx_off = streamed ? 0 : size_t(l) * a.ctx_rows * kvd * 2;
        aa.k_ctx = a.ctx_k ? reinterpret_cast<const __nv_bfloat16*>(static_cast<const uint8_t*>(a.ctx_k) + ctx_off) : aa.k_own;
        aa.v_ctx = a.ctx_v ? reinterpret_cast<const __nv_bfloat16*>(static_cast<const uint8_t*>(a.ctx_v) + ctx_off) : aa.v_own;
        aa.group = a.group;
        aa.seqs = a.seqs;
        aa.tiles = d_tiles;
        aa.out = static_cast<__nv_bfloat16*>(att);
        aa.num_heads = c.num_heads;
        aa.kv_heads = c.kv_heads;
        aa.head_dim = c.head_dim;
        aa.mode = a.mode;
        aa.scale = float(1.0 / std::sqrt(double(c.head_dim)));
        aa.row_lo = d_row_lo;
        static const int attn_prefetch = [] {  // L2 prefetch distance of the tcgen05 attention's K/V tiles
            const char* e = std::getenv("TKV_ATTN_PREFETCH");
            return e ? std::atoi(e) : 0;
        }();
        aa.prefetch = attn_prefetch;
        if (paged) {
            aa.vpool = a.gather_pool;
            aa.pool_rows = long(a.gather_pool_bytes / kv_row_bytes);
            int sh = 0;
            while ((kv_row_bytes << sh) < a.gather_page_bytes) ++sh;
            aa.rows_shift = sh;
            aa.page_ids = a.gather_pages;
            aa.segs = a.gather_segs;
            aa.n_segs = a.gather_n_segs;
            aa.layer = l;
            aa.layers = c.num_layers;
            aa.kpaged = true;
            aa.seq_seg0 = a.seq_seg0;
            aa.cos_f = rope_.cos_f();
            aa.sin_f = rope_.sin_f();
        }
        {
            cudaEvent_t e0 = nullptr, e1 = nullptr;
            if (timing_) {
                e0 = timing_event();
                e1 = timing_event();
                TKV_CUDA_CHECK(cudaEventRecord(e0, s));
            }
            if (use_tc5)
                attention_tc5(aa, d_tiles, int(tiles.size()), a.ctx_k ? a.ctx_rows : 0, M, s);
            else
                attention_bf16(aa, int(tiles.size()), s);
            if (timing_) {
                TKV_CUDA_CHECK(cudaEventRecord(e1, s));
                add_timed(e0, e1, 0.0);
            }
        }
        if (a.krot_out)
            TKV_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(a.krot_out) + size_t(l) * M * kvd * 2, k,
                                           size_t(M) * kvd * 2, cudaMemcpyDeviceToDevice, s));

        EpiParams eo;
        eo.kind = Epi::resid_f32;
        eo.out = x;
        eo.ldo = h;
        fold_out(eo, fold);
        run_gemm(att, L.wo, M, h, qd, eo);
        if (!fold) {
            norm_bf16(x, nullptr, M, h, xn, rms, eps, s);
            ++nl;
        }

        EpiParams em;
        em.out = mid;
        em.ldo = f;
        fold_in(em, fold);
        if (c.mlp == 1) {
            em.kind = Epi::swiglu_bf16;
            run_gemm(xn, L.w_in, M, 2 * f, h, em);
        } else {
            em.kind = Epi::silu_bf16;
            run_gemm(xn, L.w_in, M, f, h, em);
        }
        EpiParams ed;
        ed.kind = Epi::resid_f32;
        ed.out = x;
        ed.ldo = h;
        fold_out(ed, fold && l + 1 < c.num_layers);
        run_gemm(mid, L.w_out, M, h, f, ed);
        nl += 5;
        if (l + 1 < c.num_layers && !fold) {
            norm_bf16(x, nullptr, M, h, xn, rms, eps, s);
            ++nl;
        }
    }
    if (a.hidden_out) TKV_CUDA_CHECK(cudaMemcpyAsync(a.hidden_out, x, size_t(M) * h * 4, cudaMemcpyDeviceToDevice, s));
    if (a.n_logit_rows > 0 && a.logits_out) {
        norm_bf16(x, a.logit_rows, a.n_logit_rows, h, xn, rms, eps, s);
        EpiParams eh;
        eh.kind = Epi::store_f32;
        eh.out = a.logits_out;
        eh.ldo = c.vocab_padded();
        run_gemm(xn, head_, a.n_logit_rows, c.vocab_padded(), h, eh);
        nl += 2;
        if (a.argmax_out) {
            argmax_rows(a.logits_out, a.n_logit_rows, c.vocab, c.vocab_padded(), a.argmax_out, nullptr, s);
            ++nl;
        }
    }
    launches_ = nl;
}

void Model::forward_ref(const FwdArgs& a, cudaStream_t s) {
    const ModelCfg& c = cfg_;
    const DType dt = c.dtype;
    const size_t es = dtype_size(dt);
    const int M = a.M, h = c.hidden(), qd = c.num_heads * c.head_dim, kvd = c.kv_dim(), f = c.ffn;
    uint8_t* p = static_cast<uint8_t*>(ws_);
    auto take = [&](size_t elems) {
        void* r = p;
        p += (elems * es + 255) & ~size_t(255);
        return r;
    };
    const long R = ws_rows_;
    void* x = take(size_t(R) * h);
    void* xn = take(size_t(R) * h);
    void* q = take(size_t(R) * qd);
    void* k = take(size_t(R) * kvd);
    void* v = take(size_t(R) * kvd);
    void* att = take(size_t(R) * qd);
    void* proj = take(size_t(R) * h);
    void* mid = take(size_t(R) * f);
    void* gate = take(size_t(R) * f);
    const int rms = c.norm == 1;
    long nl = 0;

    launch_embed(emb_, dt, a.tokens, M, h, x, s);
    for (int l = 0; l < c.num_layers; ++l) {
        const Layer& L = layers_[l];
        void* v_l = a.v_out ? static_cast<uint8_t*>(a.v_out) + size_t(l) * M * kvd * es : v;
        launch_layer_norm_ref(x, xn, dt, M, h, rms, c.eps, s);
        launch_matmul_ref(L.wq, xn, q, dt, qd, h, M, 0, s);
        launch_matmul_ref(L.wk, xn, k, dt, kvd, h, M, 0, s);
        launch_matmul_ref(L.wv, xn, v_l, dt, kvd, h, M, 0, s);
        if (a.kraw_out)
            TKV_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(a.kraw_out) + size_t(l) * M * kvd * es, k,
                                           size_t(M) * kvd * es, cudaMemcpyDeviceToDevice, s));
        launch_rope_ref(q, dt, a.pos64, M, c.num_heads, c.head_dim, rope_.cos_d(), rope_.sin_d(), rope_.max_pos(), s);
        launch_rope_ref(k, dt, a.pos64, M, c.kv_heads, c.head_dim, rope_.cos_d(), rope_.sin_d(), rope_.max_pos(), s);
        if (a.krot_out)
            TKV_CUDA_CHECK(cudaMemcpyAsync(static_cast<uint8_t*>(a.krot_out) + size_t(l) * M * kvd * es, k,
                                           size_t(M) * kvd * es, cudaMemcpyDeviceToDevice, s));
        const size_t ctx_off = size_t(l) * a.ctx_rows * kvd * es;
        const void* kc = a.ctx_k ? static_cast<const uint8_t*>(a.ctx_k) + ctx_off : k;
        const void* vc = a.ctx_v ? static_cast<const uint8_t*>(a.ctx_v) + ctx_off : v_l;
        launch_attend_ref(q, k, v_l, kc, vc, a.group, a.seqs, a.n_seqs, M, att, dt, c.num_heads, c.kv_heads, c.head_dim,
                          a.mode, s, a.seqs_host);
        launch_matmul_ref(L.wo, att, proj, dt, h, qd, M, 0, s);
        launch_add_ref(x, proj, dt, long(M) * h, s);
        launch_layer_norm_ref(x, xn, dt, M, h, rms, c.eps, s);
        launch_matmul_ref(L.w_in, xn, mid, dt, f, h, M, c.mlp == 0, s);
        if (c.mlp == 1) {
            launch_matmul_ref(L.w_gate, xn, gate, dt, f, h, M, 1, s);
            launch_mul_ref(mid, gate, dt, long(M) * f, s);
        }
        launch_matmul_ref(L.w_out, mid, proj, dt, h, f, M, 0, s);
        launch_add_ref(x, proj, dt, long(M) * h, s);
        nl += 15;
    }
    if (a.hidden_out) TKV_CUDA_CHECK(cudaMemcpyAsync(a.hidden_out, x, size_t(M) * h * es, cudaMemcpyDeviceToDevice, s));
    if (a.n_logit_rows > 0 && a.logits_out && dt == DType::f32) {
        // documented head: final norm of the row, untied head, f32 logits
        for (int r = 0; r < a.n_logit_rows; ++r) {
            const int row = a.logit_rows_host ? a.logit_rows_host[r] : M - 1;
            launch_layer_norm_ref(static_cast<const uint8_t*>(x) + size_t(row) * h * es, xn, dt, 1, h, rms, c.eps, s);
            launch_matmul_ref(head_, xn, a.logits_out + size_t(r) * c.vocab_padded(), dt, c.vocab, h, 1, 0, s);
            nl += 2;
        }
        if (a.argmax_out) {
            argmax_rows(a.logits_out, a.n_logit_rows, c.vocab, c.vocab_padded(), a.argmax_out, nullptr, s);
            ++nl;
        }
    }
    launches_ = nl;
}

}  // namespace tkv
