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
};

// tokens per CTA tile for a GQA ratio (64 rows / G)
int attn_rows_per_tile(int num_heads, int kv_heads);
void attention_bf16(const AttnArgs& a, int n_tiles, cudaStream_t s);

}  // namespace tkv
