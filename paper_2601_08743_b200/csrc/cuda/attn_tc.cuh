#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace tkv {

struct AttnArgs {
    const __nv_bfloat16* q;      // [M][Hq*d] rotated queries
    const __nv_bfloat16* k_own;  // [M][Hkv*d] rotated own keys
    const __nv_bfloat16* v_own;  // [M][Hkv*d]
    const __nv_bfloat16* k_ctx;  // [ctx rows][Hkv*d] rotated cached keys (this layer)
    const __nv_bfloat16* v_ctx;
    const int32_t* group;        // [M] group id per own row (mode 1)
    const AttnSeq* seqs;         // device
    const int4* tiles;           // device: {seq, tok0, kv head, 0}
    __nv_bfloat16* out;          // [M][Hq*d]
    int num_heads, kv_heads, head_dim, mode;
    float scale;                 // 1/sqrt(d)
    const uint8_t* vpool = nullptr;      // paged mode: pool base (below)
    long pool_rows = 0;                  // paged mode: pool bytes / (kv_heads * head_dim * 2)
    int page_shift = 0, layer = 0, layers = 0;
    const int32_t* page_ids = nullptr;   // window page-id list (GatherSeg::page_off indexes it)
    const GatherSeg* segs = nullptr;     // window segments, ascending out_row0 (= ctx rows)
    int n_segs = 0;
    int prefetch = 0;                    // tiles ahead pulled into L2 (0 = off)
    long k_hm_rows = 0;                  // > 0: k_ctx is head-major [kv head][k_hm_rows][head_dim]
    // paged prefix (tcgen05 kernel): cached-prefix K and V rows come straight from the table pages
    // by TMA over the pool (rows of kv_heads * head_dim bf16, 2^rows_shift rows per page) and K is
    // rotated in shared memory at its prefix positions with the f32 RoPE tables [pos][head_dim/2];
    // vpool = pool base, page_ids / segs / layer / layers locate the rows, no slab
    bool kpaged = false;
    const int32_t* seq_seg0 = nullptr;   // paged mode: first segment of each sequence (no search)
    int rows_shift = 0;
    const float* cos_f = nullptr;
    const float* sin_f = nullptr;
    const int32_t* row_lo = nullptr;  // mode 1 on the tcgen05 kernel: first visible own key per row
                                      // (start of the row's group block; 0 for query rows)
};

// tokens per CTA tile for a GQA ratio (rows per CTA / G)
int attn_rows_per_tile(int num_heads, int kv_heads);
void attention_bf16(const AttnArgs& a, int n_tiles, cudaStream_t s);

// tcgen05 / TMEM / TMA attention (head_dim 128); work items {seq, tok0, kv head} with tok0 stepping
// by attn_tc5_rows_per_tile; ctx_rows / own_rows = row extents of the k_ctx/v_ctx and k_own/v_own
// buffers (TMA bounds).
bool attention_tc5_supported(const AttnArgs& a);
int attn_tc5_rows_per_tile(int num_heads, int kv_heads);
void attention_tc5(const AttnArgs& a, const int4* work, int n_work, long ctx_rows, long own_rows, cudaStream_t s);

}  // namespace tkv
