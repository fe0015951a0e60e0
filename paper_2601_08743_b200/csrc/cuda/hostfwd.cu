// Host-buffer wrapper around Model::forward for single sequences (parity entry points).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "model.cuh"

namespace tkv {

void forward_host(Model& model, cudaStream_t s, const HostFwd& h) {
    const ModelCfg& c = model.cfg();
    if (h.n <= 0) return;
    for (int i = 0; i < h.n; ++i)
        if (h.tokens[i] < 0 || h.tokens[i] >= c.vocab) throw std::invalid_argument("token id outside vocabulary");
    const size_t es = dtype_size(c.dtype);
    const int L = c.num_layers, kvd = c.kv_dim(), hd = c.hidden();
    std::vector<int32_t> pos(static_cast<size_t>(h.n));
    std::vector<int64_t> pos64(static_cast<size_t>(h.n));
    for (int i = 0; i < h.n; ++i) {
        pos64[size_t(i)] = h.positions ? h.positions[i] : int64_t(h.n_ctx) + i;
        pos[size_t(i)] = int32_t(pos64[size_t(i)]);
    }
    model.rope().ensure(int(*std::max_element(pos64.begin(), pos64.end())) + 2);
    std::vector<void*> bufs;
    struct Free {
        std::vector<void*>& b;
        ~Free() {
            for (void* p : b) cudaFree(p);
        }
    } freer{bufs};
    auto dmalloc = [&](size_t bytes) {
        void* p = nullptr;
        TKV_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        bufs.push_back(p);
        return p;
    };
    auto up = [&](const void* src, size_t bytes) {
        void* d = dmalloc(bytes);
        TKV_CUDA_CHECK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
        return d;
    };
    FwdArgs a;
    a.M = h.n;
    a.tokens = static_cast<const int32_t*>(up(h.tokens, size_t(h.n) * 4));
    a.pos = static_cast<const int32_t*>(up(pos.data(), size_t(h.n) * 4));
    a.pos64 = static_cast<const int64_t*>(up(pos64.data(), size_t(h.n) * 8));
    if (h.groups) a.group = static_cast<const int32_t*>(up(h.groups, size_t(h.n) * 4));
    a.group_host = h.groups;
    const AttnSeq seq{0, h.n, 0, h.mode == 0 ? h.n_ctx : 0};
    a.n_seqs = 1;
    a.seqs = static_cast<const AttnSeq*>(up(&seq, sizeof(seq)));
    a.seqs_host = &seq;
    a.mode = h.mode;
    if (h.mode == 0 && h.n_ctx > 0) {
        const size_t cb = size_t(L) * size_t(h.n_ctx) * kvd * es;
        a.ctx_k = up(h.ctx_k, cb);
        a.ctx_v = up(h.ctx_v, cb);
        a.ctx_rows = h.n_ctx;
    }
    const size_t hbytes = size_t(h.n) * hd * (c.dtype == DType::bf16 ? 4 : es);
    const size_t kvb = size_t(L) * h.n * kvd * es;
    if (h.hidden) a.hidden_out = dmalloc(hbytes);
    if (h.kraw) a.kraw_out = dmalloc(kvb);
    if (h.krot) a.krot_out = dmalloc(kvb);
    if (h.v) a.v_out = dmalloc(kvb);
    const int32_t last = h.n - 1;
    if (h.logits || h.argmax) {
        if (c.dtype == DType::f64) throw std::invalid_argument("logits are produced by f32 / bf16 models");
        a.logit_rows = static_cast<const int32_t*>(up(&last, 4));
        a.logit_rows_host = &last;
        a.n_logit_rows = 1;
        a.logits_out = static_cast<float*>(dmalloc(size_t(c.vocab_padded()) * 4));
        a.argmax_out = static_cast<int32_t*>(dmalloc(4));
    }
    model.forward(a, s);
    if (h.hidden) TKV_CUDA_CHECK(cudaMemcpyAsync(h.hidden, a.hidden_out, hbytes, cudaMemcpyDeviceToHost, s));
    if (h.kraw) TKV_CUDA_CHECK(cudaMemcpyAsync(h.kraw, a.kraw_out, kvb, cudaMemcpyDeviceToHost, s));
    if (h.krot) TKV_CUDA_CHECK(cudaMemcpyAsync(h.krot, a.krot_out, kvb, cudaMemcpyDeviceToHost, s));
    if (h.v) TKV_CUDA_CHECK(cudaMemcpyAsync(h.v, a.v_out, kvb, cudaMemcpyDeviceToHost, s));
    if (h.logits)
        TKV_CUDA_CHECK(cudaMemcpyAsync(h.logits, a.logits_out, size_t(c.vocab_padded()) * 4, cudaMemcpyDeviceToHost, s));
    if (h.argmax) TKV_CUDA_CHECK(cudaMemcpyAsync(h.argmax, a.argmax_out, 4, cudaMemcpyDeviceToHost, s));
    TKV_CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace tkv
