// Launchers for every device kernel of the online path (host-callable, stream-ordered).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

namespace tkv {

enum class DType : int { f32 = 0, bf16 = 1, f64 = 2 };

inline size_t dtype_size(DType d) { return d == DType::bf16 ? 2 : (d == DType::f32 ? 4 : 8); }

// ---- init.cu: weight init from the counter hash (proj/include/tablekv/model.hpp:80-87) -----
// dst row (interleaved) <- source row r of a [rows x cols] matrix whose element i is
// float(signed_unit(mix3(seed, tag_stream, i)) * scale). interleave_block == 0 means rows
// land contiguously at dst_row0 + r; otherwise source row r lands at
// (r / ib) * 2ib + slot * ib + r % ib (SwiGLU gate/up interleave for the fused epilogue).
void launch_fill_matrix(void* dst, DType dt, long rows, long cols, long dst_row0, uint64_t seed, uint64_t tag_stream,
                        double scale, int interleave_block, int slot, cudaStream_t s);

// ---- kvload.cu: slow tier -> paged HBM pool ------------------------------------------------
constexpr int kMaxPagesPerCopy = 256;
struct PageList {
    int32_t n;
    int32_t page[kMaxPagesPerCopy];
};
// SM-driven copy of a table image from mapped pinned host memory into its pool pages with
// coalesced 16-byte loads/stores (the north-star "vectorised H2D"); bytes % 16 == 0.
void launch_h2d_pages(const void* src_mapped, size_t bytes, uint8_t* pool, size_t page_bytes, const PageList& pages,
                      int n_ctas, cudaStream_t s);

// ---- gather.cu: assemble (proj/include/tablekv/attention.hpp:300-362) ----------------------
struct GatherSeg {
    int32_t page_off;  // index of the table's first page id in the page-id array
    int32_t tokens;    // table token count T
    int32_t pos0;      // global position of the table's first token (cursor)
    int32_t out_row0;  // first output row (segments are contiguous in output rows)
};
// Out layout: out_k / out_v are [L][out_rows][kvdim]; the table image in the pool is the
// .kv layout [K: L][T][kvdim] then [V: L][T][kvdim] (table_kv.hpp:45-48) addressed through
// its pages. K is rotated at pos0 + t (interleaved pairs); V is copied.
// exact (f32 in/out): cos/sin double tables, double arithmetic without contraction =>
// bit-identical to the reference's rotated_copy. fast: f32 math, any in/out dtype.
void launch_gather_rope(const uint8_t* pool, size_t page_bytes, const int32_t* d_page_ids, const GatherSeg* d_segs,
                        int n_segs, int total_rows, int L, int kvdim, int head_dim, DType in_dt, DType out_dt,
                        const double* cos_d, const double* sin_d, const float* cos_f, const float* sin_f,
                        void* out_k, void* out_v, long out_rows, cudaStream_t s, int l0 = 0, int nl = -1);
// Serving fast path: bf16 image -> bf16 one-layer slab for layer l, one CTA per chunk of <= 8 rows
// of one segment (gather_chunks builds the list once per window on the host).
int gather_chunks(const GatherSeg* segs, int n_segs, std::vector<int4>& out);
void launch_gather_rope_bf16(const uint8_t* pool, size_t page_bytes, const int32_t* d_page_ids, const GatherSeg* d_segs,
                             const int4* d_chunks, int n_chunks, int L, int l, int kvdim, int head_dim, const float* cos_f,
                             const float* sin_f, void* out_k, void* out_v, long out_rows, cudaStream_t s, bool k_head_major = false);
// k_head_major (K only, out_v null): out_k is [kv head][out_rows][head_dim], so one kv head's
// 128-key tile is a contiguous 32 KB block for the attention's TMA.
bool gather_use_tma();
// (l0, nl): gather only layers [l0, l0 + nl) of the L-layer images into out layers [0, nl) — the
// serving path streams one layer of prefix at a time just before that layer's attention.

// ---- rope tables ------------------------------------------------------------------------------
// Host-built [max_pos][head_dim/2] tables: angle = pos * pow(base, -2k/d) in double, std::cos /
// std::sin (rotary.hpp:31-39), so device rotation uses the reference's exact factors.

// ---- simt.cu: reference-precision (double-accumulate) forward pieces, any T in {float,double} --
void launch_embed(const void* emb, DType dt, const int32_t* tokens, int n, int hidden, void* x, cudaStream_t s);
void launch_layer_norm_ref(const void* x, void* out, DType dt, int rows, int hidden, int rms, double eps, cudaStream_t s);
void launch_matmul_ref(const void* w, const void* x, void* y, DType dt, int rows_out, int cols_in, int tokens,
                       int act_silu, cudaStream_t s);
void launch_add_ref(void* x, const void* y, DType dt, long n, cudaStream_t s);
void launch_mul_ref(void* x, const void* y, DType dt, long n, cudaStream_t s);
void launch_rope_ref(void* x, DType dt, const int64_t* positions, int n, int heads, int head_dim,
                     const double* cos_d, const double* sin_d, int table_pos, cudaStream_t s);
// attention over [ctx ; own] per sequence; mask mode 0: own rows see all ctx + causal own,
// mode 1: block-causal by group id (BlockMask::allows, attention.hpp:37-39), no ctx.
struct AttnSeq {
    int32_t q_row0;    // first own row in q / own k / own v (token rows)
    int32_t n_own;
    int32_t ctx_row0;  // first ctx row in ctx k / v
    int32_t n_ctx;
};
void launch_attend_ref(const void* q, const void* k_own, const void* v_own, const void* k_ctx, const void* v_ctx,
                       const int32_t* group, const AttnSeq* seqs, int n_seqs, int total_q, void* out, DType dt,
                       int num_heads, int kv_heads, int head_dim, int mode, cudaStream_t s,
                       const AttnSeq* seqs_host = nullptr);

}  // namespace tkv
