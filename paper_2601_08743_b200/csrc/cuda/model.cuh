// Device model: weights initialised on the GPU from the reference's counter hash and the
// prefill forward used by query_attend / prefill / encode_group (attention.hpp:207-414).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <vector>

#include "attn_tc.cuh"
#include "kernels.cuh"

namespace tkv {

struct ModelCfg {
    int num_layers = 2, num_heads = 4, kv_heads = 4, head_dim = 16, ffn = 256, vocab = 0;
    double rotary_base = 10000.0;
    uint64_t seed = 1;
    int mlp = 0;   // 0 = SiLU (reference), 1 = SwiGLU
    int norm = 0;  // 0 = LayerNorm w/o affine (reference), 1 = RMSNorm
    DType dtype = DType::bf16;  // bf16: tensor-core path; f32/f64: reference-precision path
    double eps = 1e-5;
    int hidden() const { return num_heads * head_dim; }
    int kv_dim() const { return kv_heads * head_dim; }
    int vocab_padded() const { return (vocab + 255) / 256 * 256; }
};

// Pinned host + device staging ring for per-call metadata (segment lists, attention tiles,
// positions). Chunks are reused only after every stream that may read them drained.
class StagingRing {
   public:
    explicit StagingRing(size_t bytes);
    ~StagingRing();
    // copies `n` bytes of `src` into the ring and returns the device pointer; the device-side copy (an
    // SM kernel reading the mapped ring, so it never queues behind DMA page copies) runs at flush()
    void* upload(const void* src, size_t n, cudaStream_t s);
    // copy every upload since the last flush to HBM (one kernel on `s`): call before a kernel reads them
    void flush(cudaStream_t s);
    // make room for n more bytes without wrapping (wraps, with a device sync, now if needed)
    void reserve(size_t n);
    long launches() const { return launches_; }  // copy kernels launched so far (gpu_launches claim)

   private:
    uint8_t* host_ = nullptr;
    uint8_t* mapped_ = nullptr;  // device view of host_
    long launches_ = 0;
    size_t pend_begin_ = 0, pend_end_ = 0;  // ring bytes uploaded but not yet copied
    uint8_t* dev_ = nullptr;
    size_t cap_ = 0, off_ = 0;
};

// cos/sin of pos * base^(-2k/d) for pos < max_pos, k < d/2, built on the host in double with
// the reference's expressions (rotary.hpp:31-39); f64 copy for exact paths, f32 for bf16.
class RopeTables {
   public:
    RopeTables(int head_dim, double base);
    ~RopeTables();
    void ensure(int max_pos);  // synchronises the device before regrowing
    const double* cos_d() const { return cos_d_; }
    const double* sin_d() const { return sin_d_; }
    const float* cos_f() const { return cos_f_; }
    const float* sin_f() const { return sin_f_; }
    int max_pos() const { return max_pos_; }

   private:
    int d_;
    double base_;
    int max_pos_ = 0;
    double *cos_d_ = nullptr, *sin_d_ = nullptr;
    float *cos_f_ = nullptr, *sin_f_ = nullptr;
};

struct FwdArgs {
    int M = 0;                          // own rows, all sequences concatenated
    const int32_t* tokens = nullptr;    // device [M]
    const int32_t* pos = nullptr;       // device [M] global positions
    const int64_t* pos64 = nullptr;     // device [M] (reference-precision path)
    const int32_t* group = nullptr;     // device [M] (mode 1)
    const int32_t* group_host = nullptr;  // host copy (mode 1 on the tcgen05 attention)
    int n_seqs = 0;
    const AttnSeq* seqs = nullptr;      // device
    const AttnSeq* seqs_host = nullptr; // host copy (tile planning)
    int mode = 0;                       // 0: own rows see all ctx + causal own; 1: block-causal groups
    const void* ctx_k = nullptr;        // [L][ctx_rows][kv_dim] rotated cached keys (model dtype)
    const void* ctx_v = nullptr;
    long ctx_rows = 0;
    // Layer-streamed prefix (bf16 path): when gather_segs is set, ctx_k / ctx_v hold ONE layer and
    // layer l's prefix is gathered (+RoPE) from the pool pages right before layer l's attention.
    const uint8_t* gather_pool = nullptr;
    size_t gather_page_bytes = 0;
    const int32_t* gather_pages = nullptr;  // device
    const GatherSeg* gather_segs = nullptr; // device
    int gather_n_segs = 0, gather_rows = 0;
    const int4* gather_chunks = nullptr;    // device: {seg, t0, rows, 0} (bf16 fast path)
    size_t gather_pool_bytes = 0;           // pool extent (paged mode's TMA view of the pool)
    const int32_t* seq_seg0 = nullptr;      // device [n_seqs]: first gather segment of each sequence
    const cudaEvent_t* layer_ready = nullptr;  // optional [L]: layer l's prefix K/V has landed (layer-ordered loads)
    bool paged_v = false, paged_k = false;  // both: the tcgen05 attention reads the prefix from the
                                            // pages (K rotated in smem); else the gather fills the slab
    int gather_n_chunks = 0;
    DType gather_in = DType::bf16;
    void* kraw_out = nullptr;           // optional [L][M][kv_dim] pre-rotation keys (offline encode)
    void* v_out = nullptr;              // optional [L][M][kv_dim]
    void* krot_out = nullptr;           // optional [L][M][kv_dim] rotated own keys (prefill's k_rot)
    void* hidden_out = nullptr;         // optional [M][hidden] final hidden (f32 for bf16 path, T otherwise)
    const int32_t* logit_rows = nullptr;  // optional device [n_logit_rows] rows to run the head on
    const int32_t* logit_rows_host = nullptr;  // host copy (reference-precision path)
    int n_logit_rows = 0;
    float* logits_out = nullptr;        // [n_logit_rows][vocab_padded]
    int32_t* argmax_out = nullptr;      // optional [n_logit_rows]
};

// One sequence through the forward with HOST buffers (the parity wrappers: tkv_model_forward and
// the C++ attention.hpp templates). Outputs are in the model dtype except hidden for bf16 models
// (f32 residual stream). positions nullable (= n_ctx + i).
struct HostFwd {
    const int32_t* tokens = nullptr;
    const int64_t* positions = nullptr;
    const int32_t* groups = nullptr;
    int n = 0, mode = 0, n_ctx = 0;
    const void* ctx_k = nullptr;
    const void* ctx_v = nullptr;
    void *hidden = nullptr, *kraw = nullptr, *krot = nullptr, *v = nullptr;
    float* logits = nullptr;  // [vocab_padded] of the last row
    int32_t* argmax = nullptr;
};
class Model;
void forward_host(Model& m, cudaStream_t s, const HostFwd& h);

class Model {
   public:
    Model(const ModelCfg& cfg, cudaStream_t s);
    ~Model();
    const ModelCfg& cfg() const { return cfg_; }
    // regenerate every weight for another counter-hash seed in the existing buffers (the drop-in
    // API's tests build one model per seed; a new Model would pin another staging ring each time)
    void reseed(uint64_t seed, cudaStream_t s);
    void forward(const FwdArgs& a, cudaStream_t s);
    RopeTables& rope() { return rope_; }
    StagingRing& ring() { return ring_; }
    size_t weight_bytes() const { return weight_bytes_; }
    // per-forward kernel launch count (for the bench's gpu_launches claim)
    long launches() const { return launches_; }
    // raw weight pointers (tests)
    const void* embedding() const { return emb_; }
    const void* head() const { return head_; }

    // Optional CUDA-event timing of every GEMM / attention launch (bench roofline). Records
    // accumulate across forwards until collect_timing(), which needs the stream drained.
    void set_timing(bool on) { timing_ = on; }
    // attention kernel: 0 = tcgen05 where supported (head_dim 128), 1 = mma.sync everywhere
    void set_attention_impl(int impl) { attn_impl_ = impl; }
    int attention_impl() const { return attn_impl_; }
    void add_timed(cudaEvent_t a, cudaEvent_t b, double flops);  // flops < 0 tags a gather moving -flops bytes
    void collect_timing(double& gemm_ms, double& gemm_flops, double& gather_ms, double& attn_ms, double& gather_bytes);
    cudaEvent_t timing_event();

   private:
    struct TimedRec {
        cudaEvent_t a, b;
        double flops;
        int kind;  // 0 gemm, 1 attention, 2 gather
    };
    std::vector<TimedRec> timed_;
    std::vector<cudaEvent_t> ev_pool_;
    size_t ev_used_ = 0;
    bool timing_ = false;
    int attn_impl_ = 0;

    struct Layer {
        void *wqkv = nullptr, *wq = nullptr, *wk = nullptr, *wv = nullptr, *wo = nullptr;
        void *w_in = nullptr, *w_gate = nullptr, *w_out = nullptr;
    };
    void alloc_weights(cudaStream_t s);
    void ensure_ws(int M, cudaStream_t s);
    void forward_bf16(const FwdArgs& a, cudaStream_t s);
    void forward_ref(const FwdArgs& a, cudaStream_t s);

    ModelCfg cfg_;
    RopeTables rope_;
    StagingRing ring_;
    void* emb_ = nullptr;
    void* head_ = nullptr;
    std::vector<Layer> layers_;
    std::vector<void*> allocs_;
    size_t weight_bytes_ = 0;
    // workspace
    int ws_rows_ = 0;
    void* ws_ = nullptr;
    long launches_ = 0;
    size_t pend_begin_ = 0, pend_end_ = 0;  // ring bytes uploaded but not yet copied
};

}  // namespace tkv
