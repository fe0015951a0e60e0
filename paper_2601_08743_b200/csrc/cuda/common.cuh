// Shared device helpers for the TableCache B200 kernels (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <stdexcept>
#include <string>

namespace tkv {

#define TKV_CUDA_CHECK(expr)                                                                    \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            throw ::tkv::CudaError(_e, std::string(#expr) + " @ " + __FILE__ + ":" +            \
                                           std::to_string(__LINE__));                           \
    } while (0)

struct CudaError : std::runtime_error {
    cudaError_t code;
    CudaError(cudaError_t c, const std::string& where)
        : std::runtime_error(std::string("CUDA ") + cudaGetErrorName(c) + " (" + cudaGetErrorString(c) + ") at " + where),
          code(c) {}
};

// ---- counter hash (bit-identical to proj/include/tablekv/rng.hpp:9-30) -----------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// mix3(seed, tag, i) = splitmix64(h0 + i * golden) with h0 depending only on (seed, tag).
__host__ __device__ __forceinline__ uint64_t mix3_prefix(uint64_t seed, uint64_t tag) {
    uint64_t h = splitmix64(seed ^ 0x243f6a8885a308d3ull);
    return splitmix64(h ^ splitmix64(tag));
}

__host__ __device__ __forceinline__ double signed_unit(uint64_t x) {
    return static_cast<double>(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
}

__host__ __device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return uint16_t((u >> 16) | 0x40);  // NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

inline int ceil_div(long a, long b) { return int((a + b - 1) / b); }

constexpr int kNumSMs = 148;

// Opt `func` in to `bytes` of dynamic shared memory on the CURRENT device. The attribute is
// per device, so the opt-in is remembered per (device, kernel) and raised only when a larger
// size is asked for; thread-safe (the C ABI may be called from any thread, on any device).
void ensure_smem_optin(const void* func, int bytes);
// SM count of the current device (cached per device).
int device_sm_count();

#ifdef __CUDACC__
// ---- bf16 ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
    return __bfloat1622float2(v);
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

#endif  // __CUDACC__

}  // namespace tkv
