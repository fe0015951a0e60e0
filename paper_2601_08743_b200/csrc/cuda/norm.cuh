#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tkv {

// x[m] = f32(embedding[tok[m]]), xn[m] = bf16(norm(x[m]))
void embed_norm_bf16(const void* emb, const int32_t* tokens, int rows, int hidden, float* x, void* xn, int rms, float eps,
                     cudaStream_t s);
// xn[r] = bf16(norm(x[rows_idx ? rows_idx[r] : r]))
void norm_bf16(const float* x, const int32_t* rows_idx, int rows, int hidden, void* xn, int rms, float eps, cudaStream_t s);
// per row: lowest index of the maximum (first-token argmax)
void argmax_rows(const float* logits, int rows, int vocab, long ld, int32_t* out_idx, float* out_val, cudaStream_t s);
void f32_to_bf16(const float* in, void* out, long n, cudaStream_t s);

}  // namespace tkv
