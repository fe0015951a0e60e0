// microbenchmark: MUFU ex2 throughput per SM, f32 vs f16x2 vs bf16x2 (elements per clock per SM)
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

constexpr int N_IT = 4096;

__global__ void k_f32(float* out, float seed, long long* clk) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = seed * (threadIdx.x + i) * 1e-6f - 1.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void k_f16x2(float* out, float seed, long long* clk) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) {
        __half2 h = __floats2half2_rn(seed * (threadIdx.x + i) * 1e-6f - 1.f, -0.5f);
        x[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += __half2float(reinterpret_cast<__half2*>(&x[i])->x);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
__global__ void k_bf16x2(float* out, float seed, long long* clk) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(seed * (threadIdx.x + i) * 1e-6f - 1.f, -0.5f);
        x[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x[i]));
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += __bfloat162float(reinterpret_cast<__nv_bfloat162*>(&x[i])->x);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
// f32 input -> cvt to f16x2 -> ex2 f16x2 -> (the softmax's real chain): measures the cvt cost too
__global__ void k_cvt_f16x2(float* out, float seed, long long* clk) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = seed * (threadIdx.x + i) * 1e-6f - 1.f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < N_IT / 2; ++it)
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
            uint32_t h;
            asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x[i + 1]), "f"(x[i]));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
            float lo, hi;
            asm volatile("{.reg .f16 l, h;\nmov.b32 {l, h}, %2;\ncvt.f32.f16 %0, l;\ncvt.f32.f16 %1, h;}" : "=f"(lo), "=f"(hi) : "r"(h));
            x[i] = lo - 1.f, x[i + 1] = hi - 1.f;
        }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    float* out;
    long long* clk;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&clk, 148 * 8);
    long long h[148];
    const char* names[4] = {"f32 (1 elem/lane)", "f16x2 (2 elem/lane)", "bf16x2 (2 elem/lane)", "cvt f32->f16x2 + ex2 + cvt back (2 elem/lane)"};
    for (int threads : {256, 512, 1024}) {
        for (int k = 0; k < 4; ++k) {
            for (int rep = 0; rep < 2; ++rep) {
                if (k == 0) k_f32<<<148, threads>>>(out, 1.f, clk);
                if (k == 1) k_f16x2<<<148, threads>>>(out, 1.f, clk);
                if (k == 2) k_bf16x2<<<148, threads>>>(out, 1.f, clk);
                if (k == 3) k_cvt_f16x2<<<148, threads>>>(out, 1.f, clk);
            }
            cudaDeviceSynchronize();
            cudaMemcpy(h, clk, 148 * 8, cudaMemcpyDeviceToHost);
            double instr = double(threads) * N_IT * 8 / (k == 3 ? 2 : 1);  // lane-instructions per SM
            double elems = instr * (k == 0 ? 1 : 2);
            printf("threads %4d %-48s: %.2f lane-instr/clk/SM, %.2f elem/clk/SM (%lld clk)\n", threads, names[k], instr / h[0],
                   elems / h[0], h[0]);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
