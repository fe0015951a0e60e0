// tcgen05 attention (sm_100a) for head_dim 128: S = Q.K^T and O += P.V on the 5th-gen tensor
// cores with the accumulators in TMEM — the Blackwell form of detail::attend
// (proj/include/tablekv/attention.hpp:129-176) for the serving path's [cached prefix ; own rows].
//
// CTA = (sequence, kv head, chunk of 128 query rows; rows = tokens x the G q-heads of the kv head).
// Warp 0: two TMA producer lanes — K tiles (64 keys, two 64-column SW128 boxes) on a 3-deep ring
// released as soon as Q.K^T is done, V tiles on a 2-deep ring released after P.V — from the prefix
// slab or the own-row buffer (a tile never straddles the two). Warp 1: MMA issuer. Warps 2-9:
// softmax — TMEM lane i = query row i, two warps per lane quarter split the 64 S columns (row max
// exchanged through smem), so 8 warps share the exp2/FMA work that bounds this kernel. TMEM: S double-buffered (2 x 64 cols) so
// S(t+1) overlaps softmax(t); O (128 cols) accumulates P.V across tiles. P goes through a
// double-buffered SW128 smem tile (A operand); V is the MN-major B operand straight from its TMA
// tile. Online softmax with conditional rescale (O in TMEM is rescaled only when a row max grows
// by more than 2^8), masks as in attn_tc.cu (mode 0 prefix+causal, mode 1 block-causal groups).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "attn_tc.cuh"
#include "common.cuh"

namespace tkv {

namespace {

constexpr int BM = 128, BN = 64, D = 128;
constexpr int kThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax (2 column halves)
constexpr int kKStages = 3, kVStages = 2;
constexpr int kQHalf = BM * 64 * 2;        // Q: two [128 rows][64 dims] SW128 blocks, 16 KB each
constexpr int kKVHalf = BN * 64 * 2;       // K/V tile: two [64 keys][64 dims] SW128 blocks, 8 KB each
constexpr int kKVTile = 2 * kKVHalf;       // 16 KB
constexpr int kPTile = BM * BN * 2;        // P: [128 rows][64 keys], one SW128 block, 16 KB
// smem: Q | K ring | V ring | P0 P1 | barriers
constexpr int kQOff = 0, kK0 = 2 * kQHalf, kV0 = kK0 + kKStages * kKVTile, kP0 = kV0 + kVStages * kKVTile;
constexpr int kBarOff = kP0 + 2 * kPTile;
constexpr int kNumBars = 2 * kKStages + 2 * kVStages + 2 + 2 + 2 + 2;
constexpr int kXOff = kBarOff + kNumBars * 8 + 16;   // [2 halves][128 rows] row-max exchange, then row sums
constexpr int kSmem = kXOff + 2 * 2 * BM * 4 + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
// Bounded wait: a protocol bug traps (launch error) after ~10^8 polls instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity) {
    uint32_t done = 0;
    for (long spin = 0; spin < (1L << 27); ++spin) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done)
                     : "r"(b), "r"(parity)
                     : "memory");
        if (done) return;
    }
    __trap();
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint32_t b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%"
        "22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t addr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%"
        "21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
        "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
        "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
        "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
}

// K-major SW128 descriptor (rows 128 B apart, 8-row groups 1024 B apart)
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// MN-major SW128 descriptor for V [keys][dims]: the two 64-dim blocks LBO = 8 KB apart, 8-key groups
// SBO = 1 KB apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(kKVHalf >> 4) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}
// f16-kind instruction descriptor: D f32, A/B bf16, A K-major, B K- or MN-major, M=128, N=n
__host__ __device__ constexpr uint32_t idesc(bool b_mn, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(b_mn) << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

// byte offset of (row r, 16-byte chunk c) in SW128 storage whose 64-column blocks are `half` bytes apart
__device__ __forceinline__ uint32_t sw_off(int r, int c, int half) { return uint32_t((c >> 3) * half + r * 128 + (((c & 7) ^ (r & 7)) << 4)); }

struct Tc5Args {
    AttnArgs a;
    const int4* work;  // {seq, tok0, kvh, 0}
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap mk_ctx, const __grid_constant__ CUtensorMap mv_ctx,
                    const __grid_constant__ CUtensorMap mk_own, const __grid_constant__ CUtensorMap mv_own,
                    const __grid_constant__ Tc5Args args) {
    const AttnArgs& a = args.a;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t s0 = smem_u32(sm);
    const uint32_t bars = s0 + kBarOff;
    // barrier slots: K_FULL[3] K_EMPTY[3] V_FULL[2] V_EMPTY[2] S_FULL[2] S_FREE[2] P_FULL[2] PV_DONE[2]
    auto b_kfull = [&](int i) { return bars + uint32_t(i) * 8; };
    auto b_kempty = [&](int i) { return bars + uint32_t(kKStages + i) * 8; };
    auto b_vfull = [&](int i) { return bars + uint32_t(2 * kKStages + i) * 8; };
    auto b_vempty = [&](int i) { return bars + uint32_t(2 * kKStages + kVStages + i) * 8; };
    auto b_sfull = [&](int i) { return bars + uint32_t(2 * kKStages + 2 * kVStages + i) * 8; };
    auto b_sfree = [&](int i) { return bars + uint32_t(2 * kKStages + 2 * kVStages + 2 + i) * 8; };
    auto b_pfull = [&](int i) { return bars + uint32_t(2 * kKStages + 2 * kVStages + 4 + i) * 8; };
    auto b_pvdone = [&](int i) { return bars + uint32_t(2 * kKStages + 2 * kVStages + 6 + i) * 8; };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kBarOff + kNumBars * 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 w = args.work[blockIdx.x];
    const AttnSeq sq = a.seqs[w.x];
    const int tok0 = w.y, kvh = w.z;
    const int G = a.num_heads / a.kv_heads;
    const int qw = a.num_heads * D;
    const int n_tok = min(BM / G, sq.n_own - tok0);
    const int rows = n_tok * G;
    // key tiles: the cached prefix in BN-key tiles, then the own rows up to the chunk's causal bound
    const int own_end = tok0 + n_tok;
    const int n_ctx_tiles = (sq.n_ctx + BN - 1) / BN;
    const int n_tiles = n_ctx_tiles + (own_end + BN - 1) / BN;

    // ---- setup: barriers, TMEM, Q tile (cp.async with the SW128 pattern, all threads)
    if (threadIdx.x == 0) {
        for (int i = 0; i < kKStages; ++i) mbar_init(b_kfull(i), 1), mbar_init(b_kempty(i), 1);
        for (int i = 0; i < kVStages; ++i) mbar_init(b_vfull(i), 1), mbar_init(b_vempty(i), 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(b_sfull(i), 1);
            mbar_init(b_sfree(i), 8);
            mbar_init(b_pfull(i), 8);
            mbar_init(b_pvdone(i), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int idx = threadIdx.x; idx < BM * 16; idx += kThreads) {
        const int r = idx >> 4, c = idx & 15;
        const bool ok = r < rows;
        const __nv_bfloat16* src = a.q + long(sq.q_row0 + tok0 + (ok ? r / G : 0)) * qw + (kvh * G + r % G) * D + c * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s0 + kQOff + sw_off(r, c, kQHalf)), "l"(src),
                     "r"(ok ? 16 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core reads
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tS0 = tmem, tO = tmem + 2 * BN;

    auto tile_row = [&](int t, bool& ctx) {
        ctx = t < n_ctx_tiles;
        return ctx ? sq.ctx_row0 + t * BN : sq.q_row0 + (t - n_ctx_tiles) * BN;
    };

    if (warp == 0) {
        // ---- TMA producers: lane 0 streams K tiles (released right after Q.K^T), lane 16 V tiles
        if (lane == 0) {
            for (int t = 0; t < n_tiles; ++t) {
                const int st = t % kKStages;
                mbar_wait(b_kempty(st), ((t / kKStages) & 1) ^ 1);
                bool ctx;
                const int row = tile_row(t, ctx);
                const uint32_t dk = s0 + kK0 + st * kKVTile;
                mbar_expect_tx(b_kfull(st), kKVTile);
                for (int h = 0; h < 2; ++h) tma_2d(dk + h * kKVHalf, ctx ? &mk_ctx : &mk_own, b_kfull(st), kvh * D + h * 64, row);
            }
        } else if (lane == 16) {
            for (int t = 0; t < n_tiles; ++t) {
                const int st = t % kVStages;
                mbar_wait(b_vempty(st), ((t / kVStages) & 1) ^ 1);
                bool ctx;
                const int row = tile_row(t, ctx);
                const uint32_t dv = s0 + kV0 + st * kKVTile;
                mbar_expect_tx(b_vfull(st), kKVTile);
                for (int h = 0; h < 2; ++h) tma_2d(dv + h * kKVHalf, ctx ? &mv_ctx : &mv_own, b_vfull(st), kvh * D + h * 64, row);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            const uint32_t id_qk = idesc(false, BN), id_pv = idesc(true, D);
            const uint32_t qa = s0 + kQOff;
            auto pv = [&](int t) {
                const int sp = t & 1, sv = t % kVStages;
                mbar_wait(b_pfull(sp), (t >> 1) & 1);
                mbar_wait(b_vfull(sv), (t / kVStages) & 1);
                fence_after();
                const uint32_t pa = s0 + kP0 + sp * kPTile, va = s0 + kV0 + sv * kKVTile;
#pragma unroll
                for (int k = 0; k < BN / 16; ++k)  // K = keys: A = P (K-major), B = V (MN-major)
                    mma(tO, desc_k(pa + k * 32), desc_mn(va + k * 16 * 128), id_pv, (t > 0 || k > 0) ? 1u : 0u);
                commit(b_pvdone(sp));
                commit(b_vempty(sv));
            };
            for (int t = 0; t < n_tiles; ++t) {
                const int sk = t % kKStages, ss = t & 1;
                mbar_wait(b_kfull(sk), (t / kKStages) & 1);
                mbar_wait(b_sfree(ss), ((t >> 1) & 1) ^ 1);
                fence_after();
                const uint32_t ka = s0 + kK0 + sk * kKVTile;
#pragma unroll
                for (int k = 0; k < D / 16; ++k)  // K = head dim: A = Q, B = K (both K-major)
                    mma(tS0 + ss * BN, desc_k(qa + (k >> 2) * kQHalf + (k & 3) * 32),
                        desc_k(ka + (k >> 2) * kKVHalf + (k & 3) * 32), id_qk, k > 0 ? 1u : 0u);
                commit(b_sfull(ss));
                commit(b_kempty(sk));
                if (t > 0) pv(t - 1);
            }
            if (n_tiles > 0) pv(n_tiles - 1);
        }
    } else {
        // ---- softmax warps 2..9: lane quarter q4 = warp % 4 (TMEM lanes = query rows), column half
        // h = (warp - 2) / 4 handles S columns [32h, 32h + 32) and O columns [64h, 64h + 64)
        const int q4 = warp & 3, h = (warp - 2) >> 2;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = uint32_t(q4 * 32) << 16;
        const bool live = r < rows;
        const int tok = tok0 + min(r, rows - 1) / G;
        const int grp = a.mode == 1 ? a.group[sq.q_row0 + tok] : -1;
        const float sl2 = a.scale * 1.4426950408889634f;
        const int causal = sq.n_ctx + tok;  // last visible combined key index
        float* xmax = reinterpret_cast<float*>(sm + kXOff);  // [2][BM]
        float* xsum = xmax + 2 * BM;                          // [2][BM]
        float m_run = -INFINITY, l_run = 0.f;
        for (int t = 0; t < n_tiles; ++t) {
            const int st = t & 1;
            const bool ctx = t < n_ctx_tiles;
            const int base_j = (ctx ? t * BN : sq.n_ctx + (t - n_ctx_tiles) * BN) + 32 * h;  // key index of my column 0
            const int seg_end = ctx ? sq.n_ctx : sq.n_ctx + sq.n_own;
            mbar_wait(b_sfull(st), (t >> 1) & 1);
            fence_after();
            float s[32];
            tmem_ld32(tS0 + st * BN + lane_off + 32 * h, s);
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_sfree(st));
            float mx = -INFINITY;
            if (a.mode == 0 && ctx && base_j + 32 <= sq.n_ctx) {  // full prefix columns: nothing masked
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    s[c] *= sl2;
                    mx = fmaxf(mx, s[c]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int j = base_j + c;
                    bool ok = j < seg_end && j <= causal;
                    if (a.mode == 1 && ok) ok = grp == -1 || a.group[sq.q_row0 + j - sq.n_ctx] == grp;
                    s[c] = ok ? s[c] * sl2 : -INFINITY;
                    mx = fmaxf(mx, s[c]);
                }
            }
            // row max over both halves
            xmax[h * BM + r] = mx;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            mx = fmaxf(mx, xmax[(h ^ 1) * BM + r]);
            asm volatile("bar.sync 2, 256;" ::: "memory");  // exchange slot reusable next tile
            // conditional rescale: keep the running max unless it grows by more than 8 (x256)
            const bool grow = mx > m_run + 8.f;
            if (t > 0 && __any_sync(0xffffffffu, grow)) {
                mbar_wait(b_pvdone((t - 1) & 1), ((t - 1) >> 1) & 1);  // O is stable after P(t-1).V
                fence_after();
                const float corr = grow ? exp2f(m_run - mx) : 1.f;
#pragma unroll
                for (int c = 0; c < 64; c += 32) {
                    float o[32];
                    tmem_ld32(tO + lane_off + 64 * h + c, o);
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[i] *= corr;
                    tmem_st32(tO + lane_off + 64 * h + c, o);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                if (grow) l_run *= corr;
            }
            if (grow) m_run = mx;
            const float base = m_run == -INFINITY ? 0.f : m_run;
            // P(t) -> smem buffer st (free once P(t-2).V has completed)
            if (t >= 2) mbar_wait(b_pvdone(st), ((t - 2) >> 1) & 1);
            const uint32_t pbuf = s0 + kP0 + st * kPTile;
            float sum = 0.f;
#pragma unroll
            for (int c = 0; c < 32; c += 8) {
                float p[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    p[i] = live ? exp2f(s[c + i] - base) : 0.f;
                    sum += p[i];
                }
                asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(pbuf + sw_off(r, 4 * h + (c >> 3), kPTile)),
                             "r"(pack_bf16x2(p[0], p[1])), "r"(pack_bf16x2(p[2], p[3])), "r"(pack_bf16x2(p[4], p[5])),
                             "r"(pack_bf16x2(p[6], p[7]))
                             : "memory");
            }
            l_run += sum;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_pfull(st));
        }
        // ---- epilogue: O / l -> bf16 rows (each half stores its 64 columns)
        xsum[h * BM + r] = l_run;
        if (n_tiles > 0) {
            mbar_wait(b_pvdone((n_tiles - 1) & 1), ((n_tiles - 1) >> 1) & 1);
            fence_after();
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const float l_tot = xsum[r] + xsum[BM + r];
        const float inv = l_tot > 0.f ? 1.f / l_tot : 0.f;
        __nv_bfloat16* dst = a.out + long(sq.q_row0 + tok) * qw + (kvh * G + r % G) * D + 64 * h;
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
            float o[32];
            tmem_ld32(tO + lane_off + 64 * h + c, o);
            if (live) {
#pragma unroll
                for (int i = 0; i < 32; i += 8)
                    *reinterpret_cast<uint4*>(dst + c + i) =
                        make_uint4(pack_bf16x2(o[i] * inv, o[i + 1] * inv), pack_bf16x2(o[i + 2] * inv, o[i + 3] * inv),
                                   pack_bf16x2(o[i + 4] * inv, o[i + 5] * inv), pack_bf16x2(o[i + 6] * inv, o[i + 7] * inv));
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// [rows][cols] bf16 (cols contiguous), box = 64 cols x 128 rows, 128-byte swizzle
CUtensorMap rows_map(const void* base, long rows, int cols) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(std::max(1L, rows))};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, cuuint32_t(BN)}, es[2] = {1, 1};  // 64 cols x BN rows
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (attention) failed: " + std::to_string(int(r)));
    return m;
}

}  // namespace

bool attention_tc5_supported(const AttnArgs& a) {
    return a.head_dim == 128 && a.num_heads % a.kv_heads == 0 && BM % (a.num_heads / a.kv_heads) == 0;
}

int attn_tc5_rows_per_tile(int num_heads, int kv_heads) { return BM / (num_heads / kv_heads); }

void attention_tc5(const AttnArgs& a, const int4* work, int n_work, long ctx_rows, long own_rows, cudaStream_t s) {
    if (n_work == 0) return;
    if (!attention_tc5_supported(a)) throw std::invalid_argument("tcgen05 attention needs head_dim 128");
    static bool attr = false;
    if (!attr) {
        TKV_CUDA_CHECK(cudaFuncSetAttribute(attn_tc5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
        attr = true;
    }
    const int kvd = a.kv_heads * D;
    const CUtensorMap mkc = rows_map(a.k_ctx, ctx_rows, kvd), mvc = rows_map(a.v_ctx, ctx_rows, kvd);
    const CUtensorMap mko = rows_map(a.k_own, own_rows, kvd), mvo = rows_map(a.v_own, own_rows, kvd);
    Tc5Args args{a, work};
    attn_tc5_kernel<<<n_work, kThreads, kSmem, s>>>(mkc, mvc, mko, mvo, args);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
