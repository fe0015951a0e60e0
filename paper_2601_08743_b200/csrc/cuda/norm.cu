// bf16-path row kernels: embedding gather fused with the first norm, per-layer norms
// (LayerNorm without affine, attention.hpp:84-104, or RMSNorm), final norm of the last row of
// each sequence, and the first-token argmax. One warp per row, f32 statistics, 16-byte I/O.
#include <algorithm>

#include "common.cuh"
#include "norm.cuh"

namespace tkv {

namespace {

// x: f32 row (hidden), writes bf16 normalised row
__device__ __forceinline__ void norm_row(const float* x, __nv_bfloat16* out, int hidden, int rms, float eps, int lane) {
    float s = 0.f, ss = 0.f;
    for (int i = lane * 4; i < hidden; i += 128) {
        const float4 v = *reinterpret_cast<const float4*>(x + i);
        s += v.x + v.y + v.z + v.w;
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    s = warp_sum(s);
    ss = warp_sum(ss);
    float mean = rms ? 0.f : s / hidden;
    float var = rms ? ss / hidden : fmaxf(ss / hidden - mean * mean, 0.f);
    if (!rms) {  // second pass for a numerically safe variance
        float d2 = 0.f;
        for (int i = lane * 4; i < hidden; i += 128) {
            const float4 v = *reinterpret_cast<const float4*>(x + i);
            d2 += (v.x - mean) * (v.x - mean) + (v.y - mean) * (v.y - mean) + (v.z - mean) * (v.z - mean) +
                  (v.w - mean) * (v.w - mean);
        }
        var = warp_sum(d2) / hidden;
    }
    const float inv = rsqrtf(var + eps);
    for (int i = lane * 4; i < hidden; i += 128) {
        const float4 v = *reinterpret_cast<const float4*>(x + i);
        *reinterpret_cast<uint2*>(out + i) =
            make_uint2(pack_bf16x2((v.x - mean) * inv, (v.y - mean) * inv), pack_bf16x2((v.z - mean) * inv, (v.w - mean) * inv));
    }
}

__global__ void embed_norm_kernel(const __nv_bfloat16* __restrict__ emb, const int32_t* __restrict__ tok, int rows,
                                  int hidden, float* __restrict__ x, __nv_bfloat16* __restrict__ xn, int rms, float eps) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const __nv_bfloat16* e = emb + long(tok[row]) * hidden;
    float* xr = x + long(row) * hidden;
    for (int i = lane * 4; i < hidden; i += 128) {
        const uint2 raw = *reinterpret_cast<const uint2*>(e + i);
        const float2 a = unpack_bf16x2(raw.x), b = unpack_bf16x2(raw.y);
        *reinterpret_cast<float4*>(xr + i) = make_float4(a.x, a.y, b.x, b.y);
    }
    __syncwarp();
    norm_row(xr, xn + long(row) * hidden, hidden, rms, eps, lane);
}

__global__ void norm_kernel(const float* __restrict__ x, const int32_t* __restrict__ rows_idx, int rows, int hidden,
                            __nv_bfloat16* __restrict__ xn, int rms, float eps) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const long src = rows_idx ? rows_idx[row] : row;
    norm_row(x + src * hidden, xn + long(row) * hidden, hidden, rms, eps, lane);
}

__global__ void argmax_kernel(const float* __restrict__ logits, int rows, int vocab, long ld, int32_t* __restrict__ out_idx,
                              float* __restrict__ out_val) {
    const int row = blockIdx.x;
    const float* r = logits + long(row) * ld;
    float best = -INFINITY;
    int bi = 0x7fffffff;
    auto take = [&](float v, int i) {
        if (v > best || (v == best && i < bi)) best = v, bi = i;
    };
    int i0 = 0;
    if ((reinterpret_cast<uintptr_t>(r) & 15) == 0) {  // 16-byte loads, two in flight per thread
        const int n4 = vocab >> 2;
        const float4* r4 = reinterpret_cast<const float4*>(r);
        int j = threadIdx.x;
        for (; j + int(blockDim.x) < n4; j += 2 * blockDim.x) {
            const float4 a = __ldg(r4 + j), b = __ldg(r4 + j + blockDim.x);
            take(a.x, 4 * j), take(a.y, 4 * j + 1), take(a.z, 4 * j + 2), take(a.w, 4 * j + 3);
            const int k = 4 * (j + blockDim.x);
            take(b.x, k), take(b.y, k + 1), take(b.z, k + 2), take(b.w, k + 3);
        }
        for (; j < n4; j += blockDim.x) {
            const float4 a = __ldg(r4 + j);
            take(a.x, 4 * j), take(a.y, 4 * j + 1), take(a.z, 4 * j + 2), take(a.w, 4 * j + 3);
        }
        i0 = n4 << 2;
    }
    for (int i = i0 + threadIdx.x; i < vocab; i += blockDim.x) take(r[i], i);
    __shared__ float sv[32];
    __shared__ int si[32];
    for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) best = ov, bi = oi;
    }
    if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = best, si[threadIdx.x >> 5] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (sv[w] > best || (sv[w] == best && si[w] < bi)) best = sv[w], bi = si[w];
        out_idx[row] = bi;
        if (out_val) out_val[row] = best;
    }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace

void embed_norm_bf16(const void* emb, const int32_t* tokens, int rows, int hidden, float* x, void* xn, int rms, float eps,
                     cudaStream_t s) {
    if (rows == 0) return;
    if (hidden % 4) throw std::invalid_argument("hidden must be a multiple of 4");
    embed_norm_kernel<<<ceil_div(rows, 8), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(emb), tokens, rows, hidden, x,
                                                        static_cast<__nv_bfloat16*>(xn), rms, eps);
    TKV_CUDA_CHECK(cudaGetLastError());
}

void norm_bf16(const float* x, const int32_t* rows_idx, int rows, int hidden, void* xn, int rms, float eps, cudaStream_t s) {
    if (rows == 0) return;
    norm_kernel<<<ceil_div(rows, 8), 256, 0, s>>>(x, rows_idx, rows, hidden, static_cast<__nv_bfloat16*>(xn), rms, eps);
    TKV_CUDA_CHECK(cudaGetLastError());
}

void argmax_rows(const float* logits, int rows, int vocab, long ld, int32_t* out_idx, float* out_val, cudaStream_t s) {
    if (rows == 0) return;
    argmax_kernel<<<rows, 1024, 0, s>>>(logits, rows, vocab, ld, out_idx, out_val);
    TKV_CUDA_CHECK(cudaGetLastError());
}

void f32_to_bf16(const float* in, void* out, long n, cudaStream_t s) {
    if (n == 0) return;
    f32_to_bf16_kernel<<<std::min<long>(ceil_div(n, 256), 4096), 256, 0, s>>>(in, static_cast<__nv_bfloat16*>(out), n);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
