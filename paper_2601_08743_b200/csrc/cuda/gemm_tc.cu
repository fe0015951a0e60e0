// tcgen05 / TMEM / TMA GEMM for sm_100a with fused epilogues (the QKV/O/MLP/head projections
// of query_attend, proj/include/tablekv/attention.hpp:387-411, as dense tensor-core work).
//
// CTA tile 128 x BN x 64 (bf16, 128-byte swizzle), STAGES-deep TMA->smem ring guarded by
// mbarriers, one elected thread issues tcgen05.mma (M=128, N=BN, K=16) into a TMEM f32
// accumulator, tcgen05.commit releases smem slots and finally signals the epilogue; all four
// warps then drain TMEM (tcgen05.ld 32x32b, one accumulator row per thread) through the fused
// epilogue (RoPE / SiLU / SwiGLU / residual add) straight to global memory.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <mutex>

#include "common.cuh"
#include "gemm_tc.cuh"

namespace tkv {

namespace {

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// 32 lanes x 32 columns of 32-bit accumulators: thread i gets row (lane base + i), 32 columns.
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: rows 128 B apart, 8-row groups
// 1024 B apart (SBO), LBO unused (=1), version 1 (sm100), layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}

// Instruction descriptor: D f32, A/B bf16, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// ------------------------------------------------------------------ fused epilogue
// v[0..31] = accumulator row m, columns n0..n0+31 (n0 % 32 == 0).
__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i)
        d[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                          pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
}

// 32 accumulator columns starting at col0 (a multiple of 32 inside one head of head_dim >= 32):
// 16 interleaved pairs whose cos/sin are 16 consecutive table entries -> 4 + 4 float4 loads
// (scalar loads here made the QKV epilogue, not the MMA, the bound of that GEMM)
__device__ __forceinline__ void rope32(float* v, int col0, int head_dim, int pos, const float* cos_f, const float* sin_f) {
    const int half = head_dim >> 1;
    if (head_dim & 31) {  // small heads: 32 columns span several heads
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            const int k = ((col0 + i) % head_dim) >> 1;
            const float c = cos_f[long(pos) * half + k], s = sin_f[long(pos) * half + k];
            const float a = v[i], b = v[i + 1];
            v[i] = fmaf(a, c, -b * s);
            v[i + 1] = fmaf(a, s, b * c);
        }
        return;
    }
    const int k0 = (col0 % head_dim) >> 1;
    const float4* c4 = reinterpret_cast<const float4*>(cos_f + long(pos) * half + k0);
    const float4* s4 = reinterpret_cast<const float4*>(sin_f + long(pos) * half + k0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 c = __ldg(c4 + q), s = __ldg(s4 + q);
        const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int i = 8 * q + 2 * e;
            const float a = v[i], b = v[i + 1];
            v[i] = fmaf(a, cc[e], -b * ss[e]);
            v[i + 1] = fmaf(a, ss[e], b * cc[e]);
        }
    }
}

__device__ __forceinline__ float silu_f(float z) { return z / (1.0f + __expf(-z)); }

// norm-fold consumer: the row's RMS scale from the producer's partials (1 when not folded)
__device__ __forceinline__ float ep_row_scale(const EpiParams& ep, int m, int M) {
    if (!ep.ss_in || m >= M) return 1.f;
    const float4* p = reinterpret_cast<const float4*>(ep.ss_in + long(m) * ep.ss_chunks);
    float acc = 0.f;
    for (int i = 0; i < ep.ss_chunks / 4; ++i) {
        const float4 x = __ldg(p + i);
        acc += (x.x + x.y) + (x.z + x.w);
    }
    return rsqrtf(acc / ep.ss_n + ep.eps);
}
// norm-fold producer: one 128-column partial of the row's sum of squares
__device__ __forceinline__ void ep_store_ssq(const EpiParams& ep, int m, int M, int n_end, float& ssq) {
    if (ep.ss_out && m < M) ep.ss_out[long(m) * (ep.ldo / kNormChunk) + (n_end - 1) / kNormChunk] = ssq;
    ssq = 0.f;
}

// returns the sum of squares of the updated residual values (resid_f32 with xb_out), else 0
__device__ float epilogue32(const EpiParams& ep, int m, int n0, float* v, float rs = 1.f) {
    if (rs != 1.f) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= rs;
    }
    switch (ep.kind) {
        case Epi::store_bf16:
            store_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + long(m) * ep.ldo + n0, v);
            break;
        case Epi::store_f32: {
            float4* d = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + long(m) * ep.ldo + n0);
#pragma unroll
            for (int i = 0; i < 8; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            break;
        }
        case Epi::resid_f32: {
            float4* d = reinterpret_cast<float4*>(static_cast<float*>(ep.out) + long(m) * ep.ldo + n0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float4 r = d[i];
                r.x += v[4 * i], r.y += v[4 * i + 1], r.z += v[4 * i + 2], r.w += v[4 * i + 3];
                d[i] = r;
                v[4 * i] = r.x, v[4 * i + 1] = r.y, v[4 * i + 2] = r.z, v[4 * i + 3] = r.w;
            }
            if (ep.xb_out) {
                store_bf16x32(static_cast<__nv_bfloat16*>(ep.xb_out) + long(m) * ep.ldo + n0, v);
                float s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int i = 0; i < 32; ++i) s2[i & 3] = fmaf(v[i], v[i], s2[i & 3]);
                return (s2[0] + s2[1]) + (s2[2] + s2[3]);
            }
            break;
        }
        case Epi::silu_bf16:
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = silu_f(v[i]);
            store_bf16x32(static_cast<__nv_bfloat16*>(ep.out) + long(m) * ep.ldo + n0, v);
            break;
        case Epi::swiglu_bf16: {
            float o[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] = silu_f(v[i]) * v[16 + i];
            uint4* d = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + long(m) * ep.ldo + n0 / 2);
#pragma unroll
            for (int i = 0; i < 2; ++i)
                d[i] = make_uint4(pack_bf16x2(o[8 * i], o[8 * i + 1]), pack_bf16x2(o[8 * i + 2], o[8 * i + 3]),
                                  pack_bf16x2(o[8 * i + 4], o[8 * i + 5]), pack_bf16x2(o[8 * i + 6], o[8 * i + 7]));
            break;
        }
        case Epi::qkv_rope: {
            const int pos = ep.pos[m];
            if (n0 < ep.q_cols) {
                rope32(v, n0, ep.head_dim, pos, ep.cos_f, ep.sin_f);
                store_bf16x32(static_cast<__nv_bfloat16*>(ep.q_out) + long(m) * ep.q_cols + n0, v);
            } else if (n0 < ep.q_cols + ep.kv_cols) {
                const int c = n0 - ep.q_cols;
                if (ep.k_raw_out) store_bf16x32(static_cast<__nv_bfloat16*>(ep.k_raw_out) + long(m) * ep.kv_cols + c, v);
                rope32(v, c, ep.head_dim, pos, ep.cos_f, ep.sin_f);
                store_bf16x32(static_cast<__nv_bfloat16*>(ep.k_out) + long(m) * ep.kv_cols + c, v);
            } else {
                const int c = n0 - ep.q_cols - ep.kv_cols;
                store_bf16x32(static_cast<__nv_bfloat16*>(ep.v_out) + long(m) * ep.kv_cols + c, v);
            }
            break;
        }
    }
    return 0.f;
}

// ------------------------------------------------------------------ the kernel
constexpr int BM = 128, BK = 64;

template <int BN, int STAGES>
struct Smem {
    static constexpr int a_bytes = BM * BK * 2;
    static constexpr int b_bytes = BN * BK * 2;
    static constexpr int stage_bytes = a_bytes + b_bytes;
    static constexpr int bars_off = STAGES * stage_bytes;
    static constexpr int total = bars_off + (2 * STAGES + 1) * 8 + 16 + 1024;  // + alignment slack
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                   const __grid_constant__ EpiParams ep) {
    using S = Smem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::bars_off);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES), done = smem_u32(bars + 2 * STAGES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 2) {  // TMEM: BN f32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer
        for (int kb = 0; kb < nk; ++kb) {
            const int st = kb % STAGES;
            mbar_wait(empty0 + 8 * st, ((kb / STAGES) & 1) ^ 1);
            const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
            mbar_expect_tx(full0 + 8 * st, S::stage_bytes);
            tma_load_2d(sa, &tmA, full0 + 8 * st, kb * BK, m0);
            tma_load_2d(sa + S::a_bytes, &tmB, full0 + 8 * st, kb * BK, n0);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer
        constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
        for (int kb = 0; kb < nk; ++kb) {
            const int st = kb % STAGES;
            mbar_wait(full0 + 8 * st, (kb / STAGES) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
            const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + S::a_bytes);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)  // +32 bytes per K=16 step inside the swizzle atom
                tc_mma(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            tc_commit(empty0 + 8 * st);
        }
        tc_commit(done);
    }
    __syncwarp();

    // ---- epilogue: warp w owns TMEM lanes [32w, 32w+32) = tile rows
    mbar_wait(done, 0);
    tc_fence_after();
    const int m = m0 + warp * 32 + lane;
    const float rs = ep_row_scale(ep, m, M);
    float ssq = 0.f;
    for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c, v);
        if (m < M && n0 + c < N) ssq += epilogue32(ep, m, n0 + c, v, rs);
        if (((c + 32) % kNormChunk) == 0) ep_store_ssq(ep, m, M, n0 + c + 32, ssq);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(BN));
}

// ------------------------------------------------------------------ persistent kernel
// One CTA per SM looping over tiles (static round robin, M-fastest raster: consecutive tiles
// share the weight tile B while the activation panel A stays L2-resident, so weights stream from
// HBM once). Warp 0 = TMA producer, warp 1 = MMA issuer, warps 2-5 = epilogue. The accumulator is
// double-buffered in TMEM (2 x BN columns) so the epilogue of tile i overlaps the MMAs of i+1.
constexpr int kPersistThreads = 192;

template <int BN, int STAGES>
struct SmemP {
    static constexpr int a_bytes = BM * BK * 2;
    static constexpr int b_bytes = BN * BK * 2;
    static constexpr int stage_bytes = a_bytes + b_bytes;
    static constexpr int bars_off = STAGES * stage_bytes;
    static constexpr int n_bars = 2 * STAGES + 4;  // full, empty, tmem_full[2], tmem_empty[2]
    static constexpr int total = bars_off + n_bars * 8 + 16 + 1024;
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kPersistThreads, 1)
    gemm_tc_persistent(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                       int K, const __grid_constant__ EpiParams ep) {
    using S = SmemP<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::bars_off);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::n_bars);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = (M + BM - 1) / BM, nt = (N + BN - 1) / BN, tiles = mt * nt;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull0 + 8 * i, 1);
            mbar_init(tempty0 + 8 * i, 4);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 2) {  // 2 accumulators x BN f32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int m0 = (t % mt) * BM, n0 = (t / mt) * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait(empty0 + 8 * st, ((it / STAGES) & 1) ^ 1);
                    const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
                    mbar_expect_tx(full0 + 8 * st, S::stage_bytes);
                    tma_load_2d(sa, &tmA, full0 + 8 * st, kb * BK, m0);
                    tma_load_2d(sa + S::a_bytes, &tmB, full0 + 8 * st, kb * BK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            int it = 0, local = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
                const int acc = local & 1;
                mbar_wait(tempty0 + 8 * acc, ((local >> 1) & 1) ^ 1);  // epilogue drained this buffer
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * BN);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait(full0 + 8 * st, (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
                    const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + S::a_bytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) tc_mma(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    tc_commit(empty0 + 8 * st);
                }
                tc_commit(tfull0 + 8 * acc);
            }
        }
    } else {
        // ---- epilogue warps 2..5: TMEM lane quarter = warp % 4
        const int q = warp & 3;
        int local = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++local) {
            const int acc = local & 1;
            const int m0 = (t % mt) * BM, n0 = (t / mt) * BN;
            mbar_wait(tfull0 + 8 * acc, (local >> 1) & 1);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
            const float rs = ep_row_scale(ep, m, M);
            float ssq = 0.f;
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c), v);
                if (m < M && n0 + c < N) ssq += epilogue32(ep, m, n0 + c, v, rs);
                if (((c + 32) % kNormChunk) == 0) ep_store_ssq(ep, m, M, n0 + c + 32, ssq);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

// ------------------------------------------------------------------ cluster-pair kernel (B multicast)
// Same warp roles and TMEM double buffer as gemm_tc_persistent, but CTAs run in clusters of two
// that own vertically adjacent 128 x 256 tiles (same weight columns): each CTA TMA-loads its own
// A tile and HALF of the shared 256 x 64 B tile with .multicast::cluster into both CTAs' smem, so
// every weight byte leaves L2 once per pair instead of once per CTA (48 -> 32 KB of L2 reads per
// CTA per 64-deep K step). Each MMA commit releases the stage in both CTAs (empty count 2).
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// bounded: a protocol error traps (launch failure) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_b(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    for (long spin = 0; spin < (1L << 28); ++spin) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(bar), "r"(parity)
                     : "memory");
        if (done) return;
    }
    __trap();
}
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"(mask)
                 : "memory");
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPersistThreads, 1)
    gemm_tc_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                 const __grid_constant__ EpiParams ep) {
    constexpr int BN = 256;
    using S = SmemP<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::bars_off);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + S::n_bars);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = int(cluster_rank());
    const int cid = blockIdx.x >> 1, n_cl = gridDim.x >> 1;
    const int mt = (M + BM - 1) / BM, mt2 = (mt + 1) / 2, nt = N / BN, units = mt2 * nt;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 2);  // both CTAs' MMAs must be done with the stage
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull0 + 8 * i, 1);
            mbar_init(tempty0 + 8 * i, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();  // the peer's barriers are initialised before any multicast lands in them
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: own A tile + half of the pair's B tile, multicast
            int it = 0;
            for (int u = cid; u < units; u += n_cl) {
                const int m0 = (2 * (u % mt2) + rank) * BM, n0 = (u / mt2) * BN;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait_b(empty0 + 8 * st, ((it / STAGES) & 1) ^ 1);
                    const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
                    mbar_expect_tx(full0 + 8 * st, S::stage_bytes);
                    tma_load_2d(sa, &tmA, full0 + 8 * st, kb * BK, m0);
                    tma_load_2d_mc(sa + S::a_bytes + rank * (S::b_bytes / 2), &tmB, full0 + 8 * st, kb * BK, n0 + rank * (BN / 2),
                                   uint16_t(3));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer (this CTA's 128 rows)
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
            int it = 0, local = 0;
            for (int u = cid; u < units; u += n_cl, ++local) {
                const int acc = local & 1;
                mbar_wait_b(tempty0 + 8 * acc, ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * BN);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait_b(full0 + 8 * st, (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + st * S::stage_bytes);
                    const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + S::a_bytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) tc_mma(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    tc_commit_mc(empty0 + 8 * st, uint16_t(3));  // frees the slot in both CTAs
                }
                tc_commit(tfull0 + 8 * acc);
            }
        }
    } else {
        const int q = warp & 3;
        int local = 0;
        for (int u = cid; u < units; u += n_cl, ++local) {
            const int acc = local & 1;
            const int m0 = (2 * (u % mt2) + rank) * BM, n0 = (u / mt2) * BN;
            mbar_wait_b(tfull0 + 8 * acc, (local >> 1) & 1);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
            const float rs = ep_row_scale(ep, m, M);
            float ssq = 0.f;
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c), v);
                if (m < M) ssq += epilogue32(ep, m, n0 + c, v, rs);
                if (((c + 32) % kNormChunk) == 0) ep_store_ssq(ep, m, M, n0 + c + 32, ssq);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

// ------------------------------------------------------------------ CTA-pair UMMA kernel (cta_group::2)
// The Blackwell 2-SM GEMM: a cluster of two CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256) issued by the leader. Each CTA TMA-loads its own 128 rows of
// A and its own 128 rows (N half) of B into its own smem; the MMA reads A from both SMs and B from
// both SMs, and each SM's TMEM receives its 128 accumulator rows. Per SM and 64-deep K step that is
// 32 KB of TMA writes + 32 KB of MMA reads of shared memory instead of 48 + 48 KB — the single-CTA
// 128 x 256 tile needs 188 B/clk of smem bandwidth at full MMA rate, more than the SM has.
__device__ __forceinline__ uint32_t map_to_rank(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tc_mma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_commit2_mc(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"(mask)
                 : "memory");
}

template <int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPersistThreads, 1)
    gemm_tc_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                const __grid_constant__ EpiParams ep) {
    constexpr int BN = 256;                 // pair tile 256 x 256; each CTA holds 128 rows of A and of B
    constexpr int a_bytes = BM * BK * 2, b_bytes = 128 * BK * 2, stage_bytes = a_bytes + b_bytes;  // 32 KB
    constexpr int bars_off = STAGES * stage_bytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + bars_off);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * STAGES), tempty0 = smem_u32(bars + 2 * STAGES + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1, n_cl = gridDim.x >> 1;
    const int mt = (M + BM - 1) / BM, mt2 = (mt + 1) / 2, nt = N / BN, units = mt2 * nt;
    const int nk = (K + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 2);   // leader's: one expect_tx arrive per CTA
            mbar_init(empty0 + 8 * i, 1);  // each CTA's: the leader's multicast commit
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(tfull0 + 8 * i, 1);
            mbar_init(tempty0 + 8 * i, 8);  // leader's: 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 2) {  // pair allocation: the same columns in both SMs' TMEM
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer (both CTAs): own A rows + own B half, signalling the leader
            int it = 0;
            for (int u = cid; u < units; u += n_cl) {
                const int m0 = (2 * (u % mt2) + int(rank)) * BM, n0 = (u / mt2) * BN + int(rank) * 128;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait_b(empty0 + 8 * st, ((it / STAGES) & 1) ^ 1);
                    const uint32_t sa = smem_u32(smem + st * stage_bytes);
                    const uint32_t fb = map_to_rank(full0 + 8 * st, 0);
                    mbar_arrive_expect_tx_cluster(fb, stage_bytes);
                    tma_load_2d_2sm(sa, &tmA, fb, kb * BK, m0);
                    tma_load_2d_2sm(sa + a_bytes, &tmB, fb, kb * BK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {  // ---- MMA issuer: M = 256 across the pair
            constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, BN);
            int it = 0, local = 0;
            for (int u = cid; u < units; u += n_cl, ++local) {
                const int acc = local & 1;
                mbar_wait_b(tempty0 + 8 * acc, ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + uint32_t(acc * BN);
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int st = it % STAGES;
                    mbar_wait_b(full0 + 8 * st, (it / STAGES) & 1);
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + st * stage_bytes);
                    const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + a_bytes);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) tc_mma2(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    tc_commit2_mc(empty0 + 8 * st, uint16_t(3));
                }
                tc_commit2_mc(tfull0 + 8 * acc, uint16_t(3));
            }
        }
    } else {
        const int q = warp & 3;
        const uint32_t te_leader = map_to_rank(tempty0, 0);
        int local = 0;
        for (int u = cid; u < units; u += n_cl, ++local) {
            const int acc = local & 1;
            const int m0 = (2 * (u % mt2) + int(rank)) * BM, n0 = (u / mt2) * BN;
            mbar_wait_b(tfull0 + 8 * acc, (local >> 1) & 1);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
            const float rs = ep_row_scale(ep, m, M);
            float ssq = 0.f;
            for (int c = 0; c < BN; c += 32) {
                float v[32];
                tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c), v);
                if (m < M) ssq += epilogue32(ep, m, n0 + c, v, rs);
                if (((c + 32) % kNormChunk) == 0) ep_store_ssq(ep, m, M, n0 + c + 32, ssq);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(te_leader + 8 * acc);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN));
}

// ------------------------------------------------------------------ SIMT reference
__global__ void gemm_simt_kernel(const __nv_bfloat16* __restrict__ A, const __nv_bfloat16* __restrict__ B, int M, int N,
                                 int K, EpiParams ep) {
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    const int chunks = N / 32;
    if (idx >= long(M) * chunks) return;
    const int m = int(idx / chunks), n0 = int(idx % chunks) * 32;
    float v[32];
    for (int j = 0; j < 32; ++j) {
        float acc = 0.f;
        for (int k = 0; k < K; ++k)
            acc = fmaf(__bfloat162float(A[long(m) * K + k]), __bfloat162float(B[long(n0 + j) * K + k]), acc);
        v[j] = acc;
    }
    epilogue32(ep, m, n0, v);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        TKV_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

CUtensorMap make_map_2d(const void* base, int rows, int cols, int box_rows) {
    CUtensorMap map;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return map;
}

template <int BN, int STAGES>
void launch_tc(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    using S = Smem<BN, STAGES>;
    ensure_smem_optin(reinterpret_cast<const void*>(gemm_tc_kernel<BN, STAGES>), S::total);
    const CUtensorMap ta = make_map_2d(A, M, K, BM);
    const CUtensorMap tb = make_map_2d(B, N, K, BN);
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
    gemm_tc_kernel<BN, STAGES><<<grid, 128, S::total, s>>>(ta, tb, M, N, K, ep);
    TKV_CUDA_CHECK(cudaGetLastError());
}

int sm_count() { return device_sm_count(); }

template <int BN, int STAGES>
void launch_persistent(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    using S = SmemP<BN, STAGES>;
    ensure_smem_optin(reinterpret_cast<const void*>(gemm_tc_persistent<BN, STAGES>), S::total);
    const CUtensorMap ta = make_map_2d(A, M, K, BM);
    const CUtensorMap tb = make_map_2d(B, N, K, BN);
    const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    gemm_tc_persistent<BN, STAGES><<<std::min(tiles, sm_count()), kPersistThreads, S::total, s>>>(ta, tb, M, N, K, ep);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

template <int STAGES>
void launch_pair(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    using S = SmemP<256, STAGES>;
    ensure_smem_optin(reinterpret_cast<const void*>(gemm_tc_pair<STAGES>), S::total);
    const CUtensorMap ta = make_map_2d(A, M, K, BM);
    const CUtensorMap tb = make_map_2d(B, N, K, 128);  // half of a 256-column B tile per CTA
    const int units = (((M + BM - 1) / BM + 1) / 2) * (N / 256);
    const int grid = 2 * std::max(1, std::min(units, sm_count() / 2));
    gemm_tc_pair<STAGES><<<grid, kPersistThreads, S::total, s>>>(ta, tb, M, N, K, ep);
    TKV_CUDA_CHECK(cudaGetLastError());
}

template <int STAGES>
void launch_2sm(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    constexpr int total = STAGES * (BM * BK * 2 + 128 * BK * 2) + (2 * STAGES + 4) * 8 + 16 + 1024;
    ensure_smem_optin(reinterpret_cast<const void*>(gemm_tc_2sm<STAGES>), total);
    const CUtensorMap ta = make_map_2d(A, M, K, BM);
    const CUtensorMap tb = make_map_2d(B, N, K, 128);
    const int units = (((M + BM - 1) / BM + 1) / 2) * (N / 256);
    const int grid = 2 * std::max(1, std::min(units, sm_count() / 2));
    gemm_tc_2sm<STAGES><<<grid, kPersistThreads, total, s>>>(ta, tb, M, N, K, ep);
    TKV_CUDA_CHECK(cudaGetLastError());
}

int gemm_mode() {  // TKV_GEMM = single | pair | 2sm (A/B measurements); default single
    static int mode = -1;
    if (mode < 0) {
        const char* e = std::getenv("TKV_GEMM");
        const std::string v = e ? e : "";
        mode = v == "pair" ? 1 : v == "2sm" ? 2 : 0;
    }
    return mode;
}

void gemm_bf16(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    if (M == 0) return;
    if (K % 8 || N % 32) throw std::invalid_argument("gemm_bf16: need K % 8 == 0 and N % 32 == 0");
    if ((ep.ss_out && (N % kNormChunk || ep.ldo != N)) || (ep.ss_in && ep.ss_chunks % 4))
        throw std::invalid_argument("gemm_bf16: folded norm needs 128-column partials");
    // persistent warp-specialised kernel; 128x256 tiles when N allows, else 128x128 with a deeper ring
    if (N % 256 == 0 && M > 128 && gemm_mode() == 2)
        launch_2sm<6>(A, B, M, N, K, ep, s);
    else if (N % 256 == 0 && M > 128 && gemm_mode() == 1)
        launch_pair<4>(A, B, M, N, K, ep, s);
    else if (N % 256 == 0)
        launch_persistent<256, 4>(A, B, M, N, K, ep, s);
    else
        launch_persistent<128, 6>(A, B, M, N, K, ep, s);
}

void gemm_bf16_classic(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    if (M == 0) return;
    if (K % 8 || N % 32) throw std::invalid_argument("gemm_bf16: need K % 8 == 0 and N % 32 == 0");
    // one tile per CTA (round-1 kernel), kept for A/B comparisons
    const long tiles256 = long((N + 255) / 256) * ((M + BM - 1) / BM);
    if (N % 256 == 0 && tiles256 >= 2 * kNumSMs)
        launch_tc<256, 4>(A, B, M, N, K, ep, s);
    else
        launch_tc<128, 3>(A, B, M, N, K, ep, s);
}

void gemm_bf16_simt(const void* A, const void* B, int M, int N, int K, const EpiParams& ep, cudaStream_t s) {
    if (M == 0) return;
    if (ep.ss_in || ep.ss_out) throw std::invalid_argument("gemm_bf16_simt: no folded-norm epilogue");
    const long n = long(M) * (N / 32);
    gemm_simt_kernel<<<ceil_div(n, 128), 128, 0, s>>>(static_cast<const __nv_bfloat16*>(A),
                                                      static_cast<const __nv_bfloat16*>(B), M, N, K, ep);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
