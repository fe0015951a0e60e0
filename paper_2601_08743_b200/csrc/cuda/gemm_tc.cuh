// bf16 x bf16 -> f32 tcgen05 GEMM with fused epilogues: C[M][N] = A[M][K] . B[N][K]^T.
// A = activations (row-major, K contiguous), B = weights in the reference's row-major
// [out][in] layout (model.hpp:49-51), so both operands are K-major for UMMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tkv {

enum class Epi : int {
    store_bf16 = 0,   // out_bf16[m][n]
    store_f32 = 1,    // out_f32[m][n]
    resid_f32 = 2,    // resid[m][n] += acc          (O-proj / down-proj, residual stream)
    silu_bf16 = 3,    // out_bf16[m][n] = silu(acc)  (reference non-gated MLP)
    swiglu_bf16 = 4,  // 16-col interleaved [gate|up]: out[m][n/2] = silu(g) * u
    qkv_rope = 5,     // split q | k | v, interleaved RoPE on q, k at pos[m]
};

struct EpiParams {
    Epi kind = Epi::store_bf16;
    void* out = nullptr;        // bf16/f32 output or residual (f32)
    long ldo = 0;               // output row stride (elements)
    // qkv_rope
    void* q_out = nullptr;      // [M][q_cols] bf16
    void* k_out = nullptr;      // [M][kv_cols] bf16 (rotated)
    void* k_raw_out = nullptr;  // optional [M][kv_cols] bf16 pre-rotation (offline encode keeps it)
    void* v_out = nullptr;      // [M][kv_cols] bf16
    int q_cols = 0, kv_cols = 0, head_dim = 0;
    const int32_t* pos = nullptr;        // [M] global positions
    const float* cos_f = nullptr;        // [max_pos][head_dim/2]
    const float* sin_f = nullptr;
    // RMSNorm folded into the GEMMs (no norm kernel between a residual update and the next
    // projection). Producer (resid_f32): xb_out[m][n] = bf16(updated residual) and ss_out[m][n / 128]
    // = sum of squares of its 128-column chunk, written by the one thread that owns that row of
    // the tile (no atomics: fixed order, deterministic). Consumer: the A operand is that bf16(x);
    // every accumulator row is scaled by rsqrt(sum_c ss_in[m][c] / ss_n + eps) before the epilogue
    // op, i.e. norm(x) . W = rs(x) * (x . W) with the rounding of x instead of norm(x).
    void* xb_out = nullptr;        // [M][ldo] bf16
    float* ss_out = nullptr;       // [M][ldo / 128]
    const float* ss_in = nullptr;  // [M][ss_chunks]
    int ss_chunks = 0;
    float ss_n = 1.f, eps = 0.f;
};
constexpr int kNormChunk = 128;  // columns per sum-of-squares partial

// Launch on stream; A, B device pointers (bf16 bits), K % 8 == 0, N % 32 == 0.
void gemm_bf16(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s);

// Non-persistent one-tile-per-CTA variant (the first version; A/B comparisons).
void gemm_bf16_classic(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s);

// Simple SIMT bf16 GEMM with the same epilogues (correctness reference for tests only).
void gemm_bf16_simt(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s);

}  // namespace tkv
