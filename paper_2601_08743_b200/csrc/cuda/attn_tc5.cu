// tcgen05 attention (sm_100a) for head_dim 128: S = Q.K^T and O += P.V on the 5th-gen tensor
// cores with the accumulators in TMEM — the Blackwell form of detail::attend
// (proj/include/tablekv/attention.hpp:129-176) for the serving path's [cached prefix ; own rows].
//
// Work item = (sequence, kv head, 2 x 128 query rows; rows = tokens x the G q-heads of the kv head):
// two Q tiles share every 128-key K/V tile and run as two softmax streams that ping-pong on the
// tensor core (the FlashAttention-4 structure). Persistent: one CTA per SM walks the items
// (heaviest first); every role keeps a running tile counter, so rings and mbarrier phases run on
// from one item into the next. An item whose tokens all fit the first Q tile is single-stream:
// stream 1 sits it out, so stream 1's barriers count their own items / tiles (j1, g1).
// Warp 0: TMA lanes (lane 0: the item's two Q tiles + K tiles, lane 16: V tiles; 2-deep rings of
// 32 KB tiles) from the prefix slab or the own-row buffer (a tile never straddles the two).
// Paged prefix (the serving path): cached-prefix tiles come straight from the tables' pool pages,
// no slab at all — V by warps 2-3 (16-byte cp.async into the swizzled tile), K by warpgroup 3
// (warps 12-15, one per SM sub-partition): 16-byte cp.async of the raw rows, then RoPE applied in
// place in shared memory (assemble's rotation at the key's prefix position, attention.hpp:300-362)
// before the tile is handed to the tensor core. Own-row tiles (already rotated) stay on TMA.
// Warp 1: MMA issuer, order PV_0(t) QK_0(t+1) PV_1(t) QK_1(t+1): S_s = Q_s.K^T (SS) into TMEM, then
// O_s += P_s.V with P_s read from TMEM (TS: the A operand stays in tensor memory, so P never
// touches shared memory and each PV reads only V from smem).
// Warpgroups 1 / 2 (warps 4-7 / 8-11, registers raised with setmaxnreg): softmax of stream 0 / 1 — TMEM lane = query row, each thread owns one row:
// loads its 128 S values, row max, conditional rescale of O in TMEM (only when the max grows by
// more than 2^8), P = exp2(S*scale*log2e - m) packed to bf16 and stored over S's columns.
// Masks: mode 0 — own rows see every cached prefix row + causal own (query_attend,
// attention.hpp:368-414); mode 1 — block-causal prefill over contiguous group blocks (prefill /
// encode_group, attention.hpp:210-294): a row sees [its group block's first row, itself].
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "attn_tc.cuh"
#include "common.cuh"

namespace tkv {

namespace {

constexpr int BM = 128, BN = 128, D = 128;
// warpgroup 0: warp 0 TMA (Q; K / V in slab mode), warp 1 MMA, warps 2 / 3 paged K / V TMA
// issuers; warpgroups 1 / 2: softmax of Q0 / Q1; warpgroup 3: paged K rotation in smem
constexpr int kThreads = 512;
constexpr int kKLoadThreads = 128;
#ifndef TKV_ATTN_KSTAGES
#define TKV_ATTN_KSTAGES 3  // three K slots: the paged-K loader rotates tile g-1 while tile g lands
#endif
#ifndef TKV_ATTN_VSTAGES
#define TKV_ATTN_VSTAGES 2
#endif
constexpr int kKStages = TKV_ATTN_KSTAGES, kVStages = TKV_ATTN_VSTAGES;
constexpr int kQHalf = BM * 64 * 2;        // Q tile: two [128 rows][64 dims] SW128 blocks, 16 KB each
constexpr int kQTile = 2 * kQHalf;         // 32 KB; one per stream
constexpr int kKVHalf = BN * 64 * 2;       // K/V tile: two [128 keys][64 dims] SW128 blocks, 16 KB each
constexpr int kKVTile = 2 * kKVHalf;       // 32 KB
// smem: Q0 Q1 | K ring | V ring | barriers
constexpr int kQOff = 0, kK0 = 2 * kQTile, kV0 = kK0 + kKStages * kKVTile;
constexpr int kBarOff = kV0 + kVStages * kKVTile;
// QFULL[2] QEMPTY[2] KFULL[K] KEMPTY[K] VFULL[V] VEMPTY[V], per stream: SFULL PFULL PVDONE OFREE,
// then KLAND[K] (paged: raw K rows landed, before the in-place rotation publishes KFULL)
#ifndef TKV_ATTN_PHALF
#define TKV_ATTN_PHALF 0
#endif
// TKV_ATTN_PHALF=1: P is published in two halves (keys 0-63, then 64-127) so PV's first four
// k-steps run while the softmax computes the second half (adds a per-stream PHALF barrier)
constexpr bool kPHalf = TKV_ATTN_PHALF != 0;
constexpr int kStreamBars = kPHalf ? 5 : 4;
constexpr int kNumBars = 4 + 2 * kKStages + 2 * kVStages + 2 * kStreamBars + kKStages;
constexpr int kSmem = kBarOff + kNumBars * 8 + 16 + 1024;
static_assert(kSmem <= 227 * 1024, "attention smem over the per-CTA limit");
#ifndef TKV_ATTN_SINGLE_STREAM
#define TKV_ATTN_SINGLE_STREAM 1
#endif
// an item whose tokens all fit the first Q tile runs stream 0 alone (no Q1 load, QK1 / PV1 or
// stream-1 softmax); 0 keeps both streams on every item (A/B)
constexpr bool kSingleStreamItems = TKV_ATTN_SINGLE_STREAM != 0;
#ifndef TKV_ATTN_Q_PREFETCH
#define TKV_ATTN_Q_PREFETCH 1
#endif
constexpr bool kQPrefetch = TKV_ATTN_Q_PREFETCH != 0;  // L2 prefetch of the next item's Q tiles (0: A/B)
// TMEM columns: S_s (f32, P_s as packed bf16 over its first 64 columns) at 128 s, O_s at 256 + 128 s
constexpr int kTmemCols = 512;

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
// L2 prefetch of a future tile (no smem, no barrier): the rings are 2 deep, so a tile's HBM latency
// under load (several us with K and V streaming on every SM) is hidden by pulling it into L2 early
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* m, int x, int y, int z) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(m)), "r"(x),
                 "r"(y), "r"(z)
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
__device__ __forceinline__ void tmem_ld32_async(uint32_t addr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%"
        "22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
// D (TMEM) += A (TMEM, K-major) x B (smem descriptor)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// pins registers filled by an asynchronous tcgen05.ld after the wait that completes it (the
// compiler cannot hoist their uses above this volatile asm)
__device__ __forceinline__ void reg_fence32(uint32_t* v) {
    asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]), "+r"(v[8]),
                 "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]),
                 "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]),
                 "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31]));
}
// packed f32x2 arithmetic (sm_100: FFMA2 / FADD2 issue two lanes' worth per instruction)
__device__ __forceinline__ uint64_t pack_f32x2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint64_t pack_u32x2(uint32_t a, uint32_t b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ void unpack_f32x2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fsub2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
#ifdef TKV_ATTN_EXP_EMU
// 2^x for two lanes on the FMA pipe (x >= -127): x = j + f with j = rint(x) from the 1.5*2^23
// magic add, 2^f on [-0.5, 0.5] by a degree-3 polynomial (rel. error < 1e-3, below bf16 P's
// rounding), exponent j added to the result's bits
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t x) {
    const uint64_t magic = pack_f32x2(12582912.f, 12582912.f), nmagic = pack_f32x2(-12582912.f, -12582912.f);
    const uint64_t t = fadd2(x, magic);
    const uint64_t j = fadd2(t, nmagic);
    uint64_t f;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(f) : "l"(x), "l"(j));
    uint64_t p = ffma2(f, pack_f32x2(0.0555041f, 0.0555041f), pack_f32x2(0.2402265f, 0.2402265f));
    p = ffma2(p, f, pack_f32x2(0.6931472f, 0.6931472f));
    p = ffma2(p, f, pack_f32x2(1.f, 1.f));
    uint32_t plo, phi, tlo, thi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(plo), "=r"(phi) : "l"(p));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(tlo), "=r"(thi) : "l"(t));
    return pack_u32x2(plo + (tlo << 23), phi + (thi << 23));
}
#endif
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
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
// Paged ctx tiles use a group-interleaved layout: 8-row group g, 64-column half h at g * 2 KB +
// h * 1 KB (each block one SW128 atom), so one 3-D TMA box {64 cols, 8 rows, 2 halves} fills a whole
// group. K-major (K tile, B of S = Q.K^T): 8-row groups SBO = 2 KB apart; the second 64 head dims
// +1 KB. MN-major (V tile, B of O += P.V): the two 64-dim blocks LBO = 1 KB apart, 8-key groups
// SBO = 2 KB apart.
constexpr int kGrp = 2048, kGrpHalf = 1024;
__device__ __forceinline__ uint64_t desc_k_grp(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(kGrp >> 4) << 32) | (uint64_t(1) << 46) |
           (uint64_t(2) << 61);
}
__device__ __forceinline__ uint64_t desc_mn_grp(uint32_t saddr) {
    return uint64_t((saddr & 0x3FFFF) >> 4) | (uint64_t(kGrpHalf >> 4) << 16) | (uint64_t(kGrp >> 4) << 32) |
           (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// smem byte offset of 16-byte chunk c (0..15) of tile row rr in a grouped paged tile
__device__ __forceinline__ uint32_t grp_off(int rr, int c) {
    return uint32_t((rr >> 3) * kGrp + (c >> 3) * kGrpHalf + (rr & 7) * 128 + (((c & 7) ^ (rr & 7)) << 4));
}

// f16-kind instruction descriptor: D f32, A/B bf16, A K-major, B K- or MN-major, M=128, N=n
__host__ __device__ constexpr uint32_t idesc(bool b_mn, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(b_mn) << 16) | (uint32_t(n >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}


// Walks the window's table segments along increasing prefix rows: the pool row of a cached table
// image row ([K: L][T][kv_dim] then [V: L][T][kv_dim], table_kv.hpp:45-48) for layer slot `ls`
// (l for K, L + l for V). Rows only grow along a lane's walk through an item, so each lookup
// advances the cursor instead of searching (one binary search per item).
struct SegCursor {
    int seg, next_row0;  // current segment; first row of the next one (INT_MAX past the end)
    GatherSeg sg;
    __device__ __forceinline__ void seek(const AttnArgs& a, int vr) {
        int lo = 0, hi = a.n_segs - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.segs[mid].out_row0 <= vr) lo = mid; else hi = mid - 1;
        }
        seg = lo;
        sg = a.segs[lo];
        next_row0 = lo + 1 < a.n_segs ? a.segs[lo + 1].out_row0 : 0x7fffffff;
    }
    // start at a known segment (the sequence's first) and walk forward to the one holding vr
    __device__ __forceinline__ void start(const AttnArgs& a, int s0, int vr) {
        seg = s0;
        sg = a.segs[s0];
        next_row0 = s0 + 1 < a.n_segs ? a.segs[s0 + 1].out_row0 : 0x7fffffff;
        advance(a, vr);
    }
    __device__ __forceinline__ void advance(const AttnArgs& a, int vr) {
        while (vr >= next_row0) {
            ++seg;
            sg = a.segs[seg];
            next_row0 = seg + 1 < a.n_segs ? a.segs[seg + 1].out_row0 : 0x7fffffff;
        }
    }
    // the pool row (pool viewed as [page_bytes / row_bytes rows per page]) holding window row vr
    __device__ __forceinline__ long pool_row(const AttnArgs& a, int vr, int ls) {
        advance(a, vr);
        const long off = long(ls) * sg.tokens + (vr - sg.out_row0);  // in rows of the table image
        const long rpp = 1L << a.rows_shift;                        // rows per page
        return (long(__ldg(a.page_ids + sg.page_off + (off >> a.rows_shift))) << a.rows_shift) + (off & (rpp - 1));
    }
    // rows vr..vr+7 are consecutive pool rows: one segment and one page (after pool_row(vr))
    __device__ __forceinline__ bool run8(const AttnArgs& a, int vr, int ls) const {
        const long off = long(ls) * sg.tokens + (vr - sg.out_row0);
        return vr + 8 <= next_row0 && vr - sg.out_row0 + 8 <= sg.tokens && ((off & ((1L << a.rows_shift) - 1)) + 8) <= (1L << a.rows_shift);
    }
};

struct Tc5Args {
    AttnArgs a;
    const int4* work;  // {seq, tok0, kvh, 0}, tok0 a multiple of 2·BM/G, heaviest first
    int n_work;
    uint32_t* trace;   // debug timeline of CTA 0 (TKV_ATTN_TRACE), else null
};

constexpr int kTraceEvents = 24;  // TKV_ATTN_TRACE rows of 1024 timestamps (attn_trace.py)
__device__ __forceinline__ uint32_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return uint32_t(t);
}
#define TR(ev, idx)                                                                                  \
    do {                                                                                             \
        if (args.trace && blockIdx.x == 0 && (idx) < 1024) args.trace[(ev) * 1024 + (idx)] = gtime(); \
    } while (0)

__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int x, int y, int z, int w) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(x), "r"(y), "r"(z)
                 : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc5_kernel(const __grid_constant__ CUtensorMap mq, const __grid_constant__ CUtensorMap mk_ctx,
                    const __grid_constant__ CUtensorMap mv_ctx, const __grid_constant__ CUtensorMap mk_own,
                    const __grid_constant__ CUtensorMap mv_own, const __grid_constant__ CUtensorMap mp4,
                    const __grid_constant__ CUtensorMap mp2, const __grid_constant__ Tc5Args args) {
    const AttnArgs& a = args.a;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t s0 = smem_u32(sm);
    const uint32_t bars = s0 + kBarOff;
    auto bar = [&](int i) { return bars + uint32_t(i) * 8; };
    auto b_qfull = [&](int st) { return bar(st); };
    auto b_qempty = [&](int st) { return bar(2 + st); };
    auto b_kfull = [&](int i) { return bar(4 + i); };
    auto b_kempty = [&](int i) { return bar(4 + kKStages + i); };
    auto b_vfull = [&](int i) { return bar(4 + 2 * kKStages + i); };
    auto b_vempty = [&](int i) { return bar(4 + 2 * kKStages + kVStages + i); };
    constexpr int kSB = 4 + 2 * kKStages + 2 * kVStages;
    auto b_sfull = [&](int st) { return bar(kSB + st * kStreamBars); };
    auto b_pfull = [&](int st) { return bar(kSB + st * kStreamBars + 1); };
    auto b_pvdone = [&](int st) { return bar(kSB + st * kStreamBars + 2); };
    auto b_ofree = [&](int st) { return bar(kSB + st * kStreamBars + 3); };
    auto b_kland = [&](int i) { return bar(kSB + 2 * kStreamBars + i); };
    auto b_phalf = [&](int st) { return bar(kSB + st * kStreamBars + 4); };  // kPHalf only
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + kBarOff + kNumBars * 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = a.num_heads / a.kv_heads;
    const int TQ = BM / G;  // tokens per Q tile
    const int qw = a.num_heads * D;

    if (threadIdx.x == 0) {
        TR(10, 0);
        for (int st = 0; st < 2; ++st) {
            mbar_init(b_qfull(st), 1);
            mbar_init(b_qempty(st), 1);
            mbar_init(b_sfull(st), 1);
            mbar_init(b_pfull(st), 4);
            if (kPHalf) mbar_init(b_phalf(st), 4);
            mbar_init(b_pvdone(st), 1);
            mbar_init(b_ofree(st), 4);
        }
        // slab mode: K / V tiles from the TMA lanes (1 arrival each). Paged mode: raw K rows land on
        // KLAND (the K issuer warp arms it), warpgroup 3 rotates them and all 128 threads arrive on
        // KFULL; V tiles land on VFULL armed by the V issuer warp.
        for (int i = 0; i < kKStages; ++i)
            mbar_init(b_kfull(i), a.kpaged ? kKLoadThreads : 1), mbar_init(b_kempty(i), 1), mbar_init(b_kland(i), 1);
        for (int i = 0; i < kVStages; ++i) mbar_init(b_vfull(i), 1), mbar_init(b_vempty(i), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    // per-item geometry (every role derives the same values)
    struct Item {
        AttnSeq sq;
        int tok0, kvh, n_tok, n_ctx_tiles, n_tiles;
        bool two;  // stream 1 has live rows (else the item is single-stream: no Q1, no QK1 / PV1, no softmax 1)
    };
    auto item = [&](int w) {
        const int4 wi = args.work[w];
        Item it;
        it.sq = a.seqs[wi.x];
        it.tok0 = wi.y;
        it.kvh = wi.z;
        it.n_tok = min(2 * TQ, it.sq.n_own - it.tok0);
        it.n_ctx_tiles = (it.sq.n_ctx + BN - 1) / BN;
        it.n_tiles = it.n_ctx_tiles + (it.tok0 + it.n_tok + BN - 1) / BN;  // own keys up to the item's causal bound
        it.two = it.n_tok > TQ || !kSingleStreamItems;
        return it;
    };
    auto tile_row = [&](const Item& it, int t, bool& ctx) {
        ctx = t < it.n_ctx_tiles;
        return ctx ? it.sq.ctx_row0 + t * BN : it.sq.q_row0 + (t - it.n_ctx_tiles) * BN;
    };

    // registers move to the softmax warpgroups (each thread holds a 128-column S row)
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    if (warp == 0) {
        if (lane == 0) {  // ---- TMA: the item's two Q tiles, then its K tiles
            long g = 0;
            int j = 0, j1 = 0;  // items so far; items with stream 1 so far
            for (int w = blockIdx.x; w < args.n_work; w += gridDim.x, ++j) {
                const Item it = item(w);
                for (int st = 0; st < (it.two ? 2 : 1); ++st) {
                    mbar_wait(b_qempty(st), ((st ? j1 : j) & 1) ^ 1);
                    mbar_expect_tx(b_qfull(st), kQTile);
                    for (int h = 0; h < 2; ++h)
                        tma_3d(s0 + kQOff + st * kQTile + h * kQHalf, &mq, b_qfull(st), h * 64, it.kvh * G,
                               it.sq.q_row0 + it.tok0 + st * TQ);
                }
                j1 += it.two;
                TR(8, j);
                // the next item's Q tiles into L2 now: their TMA load can only issue once this item's
                // last QK has read the Q buffers, and a cold load then sits on the item boundary
                // (several us under the K/V streams — most of a short item's time at C2)
                if (kQPrefetch && w + int(gridDim.x) < args.n_work) {
                    const Item nx = item(w + gridDim.x);
                    for (int st = 0; st < (nx.two ? 2 : 1); ++st)
                        for (int h = 0; h < 2; ++h) tma_prefetch_3d(&mq, h * 64, nx.kvh * G, nx.sq.q_row0 + nx.tok0 + st * TQ);
                }
                if (a.kpaged) continue;  // paged mode: K tiles come from the K issuer warp
                auto prefetch_kv = [&](int t) {  // K always; V here only when it comes by TMA
                    bool ctx;
                    const int row = tile_row(it, t, ctx);
                    for (int h = 0; h < 2; ++h) {
                        const bool hm = ctx && a.k_hm_rows;
                        tma_prefetch_2d(ctx ? &mk_ctx : &mk_own, hm ? h * 64 : it.kvh * D + h * 64, hm ? int(it.kvh * a.k_hm_rows) + row : row);
                        tma_prefetch_2d(ctx ? &mv_ctx : &mv_own, it.kvh * D + h * 64, row);
                    }
                };
                const int pf = a.prefetch;
                for (int t = kKStages; t < min(pf, it.n_tiles); ++t) prefetch_kv(t);
                for (int t = 0; t < it.n_tiles; ++t, ++g) {
                    if (pf && t + pf < it.n_tiles) prefetch_kv(t + pf);
                    const int sk = int(g % kKStages);
                    mbar_wait(b_kempty(sk), int((g / kKStages) & 1) ^ 1);
                    TR(0, g);
                    bool ctx;
                    const int row = tile_row(it, t, ctx);
                    const uint32_t dk = s0 + kK0 + sk * kKVTile;
                    mbar_expect_tx(b_kfull(sk), kKVTile);
                    const bool hm = ctx && a.k_hm_rows;  // head-major slab: the head's block, rows within it
                    for (int h = 0; h < 2; ++h)
                        tma_2d(dk + h * kKVHalf, ctx ? &mk_ctx : &mk_own, b_kfull(sk), hm ? h * 64 : it.kvh * D + h * 64,
                               hm ? int(it.kvh * a.k_hm_rows) + row : row);
                }
            }
        } else if (lane == 16 && !a.kpaged) {  // ---- TMA: V tiles (slab mode)
            long g = 0;
            for (int w = blockIdx.x; w < args.n_work; w += gridDim.x) {
                const Item it = item(w);
                for (int t = 0; t < it.n_tiles; ++t, ++g) {
                    const int sv = int(g % kVStages);
                    mbar_wait(b_vempty(sv), int((g / kVStages) & 1) ^ 1);
                    TR(1, g);
                    bool ctx;
                    const int row = tile_row(it, t, ctx);
                    const uint32_t dv = s0 + kV0 + sv * kKVTile;
                    mbar_expect_tx(b_vfull(sv), kKVTile);
                    for (int h = 0; h < 2; ++h) tma_2d(dv + h * kKVHalf, ctx ? &mv_ctx : &mv_own, b_vfull(sv), it.kvh * D + h * 64, row);
                }
            }
        }
    } else if ((warp == 2 || warp == 3) && a.kpaged) {
        // ---- paged issuers: warp 2 the K tiles (onto KLAND), warp 3 the V tiles (onto VFULL).
        // Cached-prefix tiles come straight from the tables' pool pages by TMA over the pool viewed
        // as [pool rows][kv_heads * 128] (mk_ctx: 8-row boxes, mv_ctx: 1-row boxes, 128-byte
        // swizzle): lane j < 16 owns rows [8j, 8j + 8) of the tile; when those 8 rows are one run of
        // one table segment inside one page they move as one 8-row box per 64-column half, else row
        // by row. Own-row tiles (rotated by the QKV epilogue) by TMA from the own-row buffers.
        const bool is_k = warp == 2;
        const int ls = is_k ? a.layer : a.layers + a.layer;  // layer slot of the table image
        SegCursor cur;
        long g = 0;
        for (int w = blockIdx.x; w < args.n_work; w += gridDim.x) {
            const Item it = item(w);
            if (it.n_ctx_tiles && lane < 16) {
                const int vr0 = it.sq.ctx_row0 + min(8 * lane, it.sq.n_ctx - 1);
                if (a.seq_seg0) cur.start(a, a.seq_seg0[args.work[w].x], vr0);
                else cur.seek(a, vr0);
            }
            for (int t = 0; t < it.n_tiles; ++t, ++g) {
                const int stg = int(g % (is_k ? kKStages : kVStages));
                const long lap = g / (is_k ? kKStages : kVStages);
                mbar_wait(is_k ? b_kempty(stg) : b_vempty(stg), int(lap & 1) ^ 1);
                if (lane == 0) TR(is_k ? 0 : 1, g);
                bool ctx;
                const int row = tile_row(it, t, ctx);
                const uint32_t dst = s0 + (is_k ? kK0 : kV0) + stg * kKVTile;
                const uint32_t fb = is_k ? b_kland(stg) : b_vfull(stg);
                if (!ctx) {
                    if (lane == 0) {
                        mbar_expect_tx(fb, kKVTile);
                        for (int h = 0; h < 2; ++h) tma_2d(dst + h * kKVHalf, is_k ? &mk_own : &mv_own, fb, it.kvh * D + h * 64, row);
                    }
                    continue;
                }
                const int key0 = t * BN + 8 * lane;
                const int nv = lane < 16 ? max(0, min(8, it.sq.n_ctx - key0)) : 0;
                if (!is_k && t * BN + BN > it.sq.n_ctx) {  // V rows past the prefix: finite zeros (P is 0 there)
                    for (int i = lane; i < (t * BN + BN - it.sq.n_ctx) * 16; i += 32) {
                        const int rr = it.sq.n_ctx - t * BN + (i >> 4), c = i & 15;
                        asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(dst + grp_off(rr, c)), "r"(0u) : "memory");
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                }
                uint32_t bytes = uint32_t(nv) * D * 2;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
                __syncwarp();
                if (lane == 0) mbar_expect_tx(fb, bytes);
                __syncwarp();
                if (nv > 0) {
                    const int vr = it.sq.ctx_row0 + key0;
                    const uint32_t gdst = dst + lane * kGrp;  // this lane's 8-row group (grouped layout)
                    long pr = cur.pool_row(a, vr, ls);
#ifdef TKV_ATTN_FAKE_CLEAN  // timing probe only (wrong rows at boundaries): every full group as one box
                    if (nv == 8) {
#else
                    if (nv == 8 && cur.run8(a, vr, ls)) {
#endif
                        tma_4d(gdst, &mk_ctx, fb, 0, int(pr), 0, it.kvh);  // both halves of 8 rows of this head
                    } else {
                        // runs of consecutive pool rows inside the group, each as 4 / 2 / 1-row boxes
                        // per 64-column half (the swizzle follows the smem address, so a box may
                        // start at any row of the atom)
                        int r0 = 0;
                        while (r0 < nv) {
                            int n = 1;
                            long pn = pr;
                            while (r0 + n < nv) {
                                pn = cur.pool_row(a, vr + r0 + n, ls);
                                if (pn != pr + n) break;
                                ++n;
                            }
                            for (int r = r0; r < r0 + n;) {
                                const int len = (r0 + n - r) >= 4 ? 4 : (r0 + n - r) >= 2 ? 2 : 1;
                                const CUtensorMap* mp = len == 4 ? &mp4 : len == 2 ? &mp2 : &mv_ctx;
                                for (int h = 0; h < 2; ++h)
                                    tma_2d(gdst + h * kGrpHalf + r * 128, mp, fb, it.kvh * D + h * 64, int(pr + (r - r0)));
                                r += len;
                            }
                            r0 += n;
                            pr = pn;  // first row of the next run (when the run broke on pn)
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            const uint32_t id_qk = idesc(false, BN), id_pv = idesc(true, D);
            // cursor over the flattened (item, tile) sequence of this CTA
            // stream 1's barriers run on their own counters (j1: items with stream 1 before this
            // one, g1: stream-1 tiles before this one) because single-stream items skip them
            struct Cur {
                int w, j, j1, t, n, nct;  // nct: the item's cached-prefix tiles (grouped layout when paged)
                long gi, g1;
                bool two;
            };
            auto set_item = [&](Cur& c) {
                if (c.w < args.n_work) {
                    const Item it = item(c.w);
                    c.n = it.n_tiles, c.nct = it.n_ctx_tiles, c.two = it.two;
                } else {
                    c.n = 0, c.nct = 0, c.two = false;
                }
            };
            auto first_tile = [&](Cur& c) {
                c.w = blockIdx.x, c.j = 0, c.j1 = 0, c.t = 0, c.gi = 0, c.g1 = 0;
                set_item(c);
                return c.w < args.n_work;
            };
            auto advance = [&](Cur c) {
                ++c.gi;
                c.g1 += c.two;
                if (++c.t == c.n) {
                    c.t = 0, c.w += gridDim.x, ++c.j;
                    c.j1 += c.two;
                    set_item(c);
                }
                return c;
            };
            auto qk = [&](const Cur& c, int st) {  // S_st = Q_st . K(c)^T
                const int sk = int(c.gi % kKStages);
                if (st == 0) {
                    mbar_wait(b_kfull(sk), int((c.gi / kKStages) & 1));
                    TR(2, c.gi);
                }
                if (c.t == 0) mbar_wait(b_qfull(st), (st ? c.j1 : c.j) & 1);
                fence_after();
                const uint32_t qa = s0 + kQOff + st * kQTile, ka = s0 + kK0 + sk * kKVTile;
                const bool grp = a.kpaged && c.t < c.nct;  // paged cached-prefix tile: grouped layout
#pragma unroll
                for (int k = 0; k < D / 16; ++k)  // K = head dim: A = Q_st, B = K (both K-major)
                    mma(tmem + st * BN, desc_k(qa + (k >> 2) * kQHalf + (k & 3) * 32),
                        grp ? desc_k_grp(ka + (k >> 2) * kGrpHalf + (k & 3) * 32) : desc_k(ka + (k >> 2) * kKVHalf + (k & 3) * 32),
                        id_qk, k > 0 ? 1u : 0u);
                commit(b_sfull(st));
                if (st == 0) TR(19, c.gi);
                if (c.t + 1 == c.n) commit(b_qempty(st));
                if (st == 1 || !c.two) commit(b_kempty(sk));
            };
            auto pv = [&](const Cur& c, int st) {  // O_st += P_st . V(c), P_st from TMEM
                const int sv = int(c.gi % kVStages);
                if (st == 0) {
                    mbar_wait(b_vfull(sv), int((c.gi / kVStages) & 1));
                    TR(11, c.gi);
                }
                const int pph = int((st ? c.g1 : c.gi) & 1);
                mbar_wait(kPHalf ? b_phalf(st) : b_pfull(st), pph);
                TR(st == 0 ? 4 : 18, c.gi);
                if (c.t == 0) mbar_wait(b_ofree(st), ((st ? c.j1 : c.j) & 1) ^ 1);  // the previous item's epilogue read O_st
                fence_after();
                const uint32_t va = s0 + kV0 + sv * kKVTile;
                const bool grp = a.kpaged && c.t < c.nct;
#pragma unroll
                for (int k = 0; k < BN / 16; ++k) {  // K = keys: A = P (TMEM, 8 columns per 16 keys), B = V (MN-major)
                    if (kPHalf && k == BN / 32) {  // keys 64-127: the second half of P
                        mbar_wait(b_pfull(st), pph);
                        fence_after();
                    }
                    mma_ts(tmem + 256 + st * D, tmem + st * BN + k * 8,
                           grp ? desc_mn_grp(va + k * 2 * kGrp) : desc_mn(va + k * 16 * 128), id_pv, (c.t > 0 || k > 0) ? 1u : 0u);
                }
                commit(b_pvdone(st));
                if (st == 1 || !c.two) commit(b_vempty(sv));
                TR(16 + st, c.gi);
            };
            Cur cur;
            if (first_tile(cur)) {
                qk(cur, 0);
                if (cur.two) qk(cur, 1);
                while (true) {
                    const Cur nxt = advance(cur);
                    const bool more = nxt.w < args.n_work;
                    // PV_s(t) then QK_s(t+1): the tensor pipe executes in issue order, so QK_s(t+1)
                    // overwrites S_s / P_s only after PV_s(t) — or stream s's last PV of an earlier
                    // item — has consumed P_s
                    pv(cur, 0);
                    if (more) qk(nxt, 0);
                    if (cur.two) pv(cur, 1);
                    if (more && nxt.two) qk(nxt, 1);
                    TR(3, cur.gi);
                    if (!more) break;
                    cur = nxt;
                }
            }
        }
    }
    } else if (warp >= 12) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;");
        if (a.kpaged) {
            // ---- paged K rotation: once a tile's raw rows have landed (KLAND), every thread rotates
            // its chunks in place — interleaved pairs k = 4c..4c+3 of its rows at their prefix
            // positions p (assemble, attention.hpp:300-362): a' = a cos - b sin, b' = a sin + b cos in
            // f32, rounded to bf16 (the gather's formula) — writes zeros into rows past the prefix,
            // and publishes the tile on KFULL. cos/sin of p come from the f32 table at the thread's
            // first row and advance by R(2 theta_k) per row step (its rows are 2 apart).
            const int kt = threadIdx.x - 384;
            const int kw = kt >> 5;                   // warp kw owns tile rows [32 kw, 32 kw + 32)
            const int c = lane & 15, hl = lane >> 4;  // chunk of the head row; rows 32 kw + 2i + hl
            constexpr int kRowStep = 2;
            const int half = D / 2;
            // packed f32x2 math: lane q of the pair vectors holds pairs (2q, 2q + 1) of the chunk
            uint64_t CD[2], SD[2], NSD[2];  // R(kRowStep theta_k), k = 4c..4c+3
            {
                const float4 x = __ldg(reinterpret_cast<const float4*>(a.cos_f + kRowStep * half + 4 * c));
                const float4 y = __ldg(reinterpret_cast<const float4*>(a.sin_f + kRowStep * half + 4 * c));
                CD[0] = pack_f32x2(x.x, x.y), CD[1] = pack_f32x2(x.z, x.w);
                SD[0] = pack_f32x2(y.x, y.y), SD[1] = pack_f32x2(y.z, y.w);
                NSD[0] = pack_f32x2(-y.x, -y.y), NSD[1] = pack_f32x2(-y.z, -y.w);
            }
            long g = 0;
            for (int w = blockIdx.x; w < args.n_work; w += gridDim.x) {
                const Item it = item(w);
                for (int t = 0; t < it.n_tiles; ++t, ++g) {
                    const int sk = int(g % kKStages);
                    mbar_wait(b_kland(sk), int((g / kKStages) & 1));
#ifdef TKV_ATTN_NO_ROTATE  // timing probe only: K published unrotated
                    if (false) {
#else
                    if (t < it.n_ctx_tiles) {
#endif
                        const uint32_t dk = s0 + kK0 + sk * kKVTile;
                        const int pos0 = t * BN + 32 * kw + hl;
                        uint64_t CS[2] = {0ull, 0ull}, SN[2] = {0ull, 0ull};
                        if (pos0 < it.sq.n_ctx) {
                            const float4 x = __ldg(reinterpret_cast<const float4*>(a.cos_f + long(pos0) * half + 4 * c));
                            const float4 y = __ldg(reinterpret_cast<const float4*>(a.sin_f + long(pos0) * half + 4 * c));
                            CS[0] = pack_f32x2(x.x, x.y), CS[1] = pack_f32x2(x.z, x.w);
                            SN[0] = pack_f32x2(y.x, y.y), SN[1] = pack_f32x2(y.z, y.w);
                        }
#pragma unroll 4
                        for (int i = 0; i < 16; ++i) {
                            const int rr = 32 * kw + 2 * i + hl;
                            const uint32_t at = dk + grp_off(rr, c);  // grouped paged tile
                            uint32_t wv[4] = {0u, 0u, 0u, 0u};
                            if (pos0 + 2 * i < it.sq.n_ctx) {
                                asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                             : "=r"(wv[0]), "=r"(wv[1]), "=r"(wv[2]), "=r"(wv[3])
                                             : "r"(at));
#pragma unroll
                                for (int q = 0; q < 2; ++q) {
                                    const uint32_t w0 = wv[2 * q], w1 = wv[2 * q + 1];
                                    const uint64_t X0 = pack_u32x2(w0 << 16, w1 << 16);                  // a of the pairs
                                    const uint64_t X1 = pack_u32x2(w0 & 0xffff0000u, w1 & 0xffff0000u);  // b
                                    const uint64_t A = fsub2(fmul2(X0, CS[q]), fmul2(X1, SN[q]));        // a c - b s
                                    const uint64_t B = ffma2(X0, SN[q], fmul2(X1, CS[q]));              // a s + b c
                                    float a0, a1, b0, b1;
                                    unpack_f32x2(A, a0, a1);
                                    unpack_f32x2(B, b0, b1);
                                    wv[2 * q] = pack_bf16x2(a0, b0);
                                    wv[2 * q + 1] = pack_bf16x2(a1, b1);
                                    const uint64_t cn = ffma2(SN[q], NSD[q], fmul2(CS[q], CD[q]));  // c cd - s sd
                                    SN[q] = ffma2(CS[q], SD[q], fmul2(SN[q], CD[q]));               // s cd + c sd
                                    CS[q] = cn;
                                }
                            }
                            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(at), "r"(wv[0]), "r"(wv[1]), "r"(wv[2]), "r"(wv[3])
                                         : "memory");
                        }
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    mbar_arrive(b_kfull(sk));
                    if (kt == 0) TR(9, g);
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 176;");
        // ---- softmax: stream st = Q tile, lane quarter q4 = warp % 4 (TMEM lanes = rows); every
        // thread owns one query row and all 128 columns of each S tile
        const int st = (warp - 4) >> 2, q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_off = uint32_t(q4 * 32) << 16;
        const uint32_t tS = tmem + st * BN + lane_off;
        const uint32_t tO = tmem + 256 + st * D + lane_off;
        const float sl2 = a.scale * 1.4426950408889634f;
        long g = 0;
        int j = 0;
        for (int w = blockIdx.x; w < args.n_work; w += gridDim.x, ++j) {
            const Item it = item(w);
            if (st == 1 && !it.two) continue;  // single-stream item: stream 1's counters do not move
            const AttnSeq& sq = it.sq;
            const int tok_local = st * TQ + r / G;  // token within the item
            const bool live = tok_local < it.n_tok;
            const int tok = it.tok0 + min(tok_local, it.n_tok - 1);
            const int causal = sq.n_ctx + tok;  // last visible combined key index
            // block-causal prefill (BlockMask::allows, attention.hpp:37-39) with contiguous group
            // blocks: a row sees own keys [first key of its group block, itself]
            const int lo = a.mode == 1 ? a.row_lo[sq.q_row0 + tok] : 0;
            float m_run = -INFINITY, l_run = 0.f;
            // a warp whose 32 rows are all past the item's tokens (short suffixes) skips the TMEM
            // reads, exponentials and P writes: its O rows are never stored, so its P may stay
            // whatever S left there; it still paces on S-ready / PV-done so its arrivals stay in phase
            const bool wdead = __all_sync(0xffffffffu, !live);
            for (int t = 0; t < it.n_tiles; ++t) {
                const long gi = g + t;
                const bool ctx = t < it.n_ctx_tiles;
                const int base_j = ctx ? t * BN : sq.n_ctx + (t - it.n_ctx_tiles) * BN;  // key index of column 0
                const int seg_end = ctx ? sq.n_ctx : sq.n_ctx + sq.n_own;
                mbar_wait(b_sfull(st), int(gi & 1));
                if (warp == 4 && lane == 0) TR(5, gi);
                if (warp == 8 && lane == 0) TR(20, gi);  // stream 1's S ready
                if (wdead) {
                    __syncwarp();
                    if (lane == 0 && kPHalf) mbar_arrive(b_phalf(st));
                    if (lane == 0) mbar_arrive(b_pfull(st));
                    continue;
                }
                fence_after();
                // S row -> registers, row max, conditional rescale, then exponentials -> P over S's first
                // 64 columns (TKV_ATTN_TWOPASS: the round-1 variant reading S twice in 32-column chunks)
                const bool masked = !(ctx && base_j + BN <= sq.n_ctx);  // full prefix tiles skip the mask
                const int lim = masked ? min(seg_end, causal + 1) - base_j : BN;  // columns [lo_c, lim) visible
                const int lo_c = masked ? lo - base_j : 0;
                auto mask_chunk = [&](uint32_t* v, int c0) {
                    if (masked) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (c0 + i >= lim || c0 + i < lo_c) v[i] = 0xff800000u;  // -inf
                    }
                };
#ifdef TKV_ATTN_TWOPASS
                uint32_t ua[32], ub[32];
#endif
                // row max as four independent 3-input max chains (FMNMX3)
                float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
                auto max_chunk = [&](const uint32_t* v) {
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            m4[q] = fmaxf(fmaxf(m4[q], __uint_as_float(v[i + 2 * q])), __uint_as_float(v[i + 2 * q + 1]));
                };
#ifndef TKV_ATTN_TWOPASS
                // one pass: the whole 128-column S row into registers (4 loads, one wait) — TMEM reads
                // run at 64 B/clk per SM, so S is read once per tile, not twice
                uint32_t sv[128];
#pragma unroll
                for (int k = 0; k < 4; ++k) tmem_ld32_async(tS + 32 * k, sv + 32 * k);
                tmem_wait_ld();
#pragma unroll
                for (int k = 0; k < 4; ++k) reg_fence32(sv + 32 * k);
                if (warp == 4 && lane == 0) TR(12, gi);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    mask_chunk(sv + 32 * k, 32 * k);
                    max_chunk(sv + 32 * k);
                }
#else
                tmem_ld32_async(tS, ua);
                tmem_wait_ld();
                reg_fence32(ua);
                if (warp == 4 && lane == 0) TR(12, gi);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    uint32_t* cur = (k & 1) ? ub : ua;
                    uint32_t* nxt = (k & 1) ? ua : ub;
                    if (k < 3) tmem_ld32_async(tS + 32 * (k + 1), nxt);
                    mask_chunk(cur, 32 * k);
                    max_chunk(cur);
                    if (k < 3) {
                        tmem_wait_ld();
                        reg_fence32(nxt);
                    }
                }
#endif
                float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                mx *= sl2;  // scale > 0: the max commutes with it
                // conditional rescale: keep the running max unless it grows by more than 8 (x256)
                // (O is rescaled after P is written, before P is published: the S registers are dead
                // by then, and PV(t) cannot start before the P-ready arrival)
                const bool grow = mx > m_run + 8.f;
                const bool any_grow = t > 0 && __any_sync(0xffffffffu, grow);
                const float corr = grow ? ex2(m_run - mx) : 1.f;
                if (grow) l_run *= corr, m_run = mx;
                if (warp == 4 && lane == 0) TR(13, gi);
                // rows past the item's tokens get P = 0 through the bias (-inf)
                const float nb = !live ? -INFINITY : (m_run == -INFINITY ? 0.f : -m_run);
                // pass 2: x*scale*log2e - m on column pairs (FFMA2), exp2 on the MUFU, row sum in two
                // packed accumulators (FADD2), P as bf16 pairs over S's first 64 columns (chunk k's P
                // lands on columns [16k, 16k+16), all of which pass 2 has already read)
                const uint64_t sl2x2 = pack_f32x2(sl2, sl2), nbx2 = pack_f32x2(nb, nb);
                uint64_t acc[2] = {0ull, 0ull};
                auto rescale_o = [&]() {
                    mbar_wait(b_pvdone(st), int((gi - 1) & 1));  // O is stable after P(t-1).V
                    fence_after();
#pragma unroll
                    for (int c = 0; c < D; c += 32) {
                        float o[32];
                        tmem_ld32(tO + c, o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= corr;
                        tmem_st32(tO + c, o);
                    }
                };
#ifdef TKV_ATTN_TWOPASS
                tmem_ld32_async(tS, ua);
                tmem_wait_ld();
                reg_fence32(ua);
#endif
#pragma unroll
                for (int k = 0; k < 4; ++k) {
#ifndef TKV_ATTN_TWOPASS
                    uint32_t* cur = sv + 32 * k;  // already masked
#else
                    uint32_t* cur = (k & 1) ? ub : ua;
                    uint32_t* nxt = (k & 1) ? ua : ub;
                    if (k < 3) tmem_ld32_async(tS + 32 * (k + 1), nxt);
                    mask_chunk(cur, 32 * k);
#endif
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        float a0, a1;
                        const uint64_t ax2 = ffma2(pack_u32x2(cur[i], cur[i + 1]), sl2x2, nbx2);
                        unpack_f32x2(ax2, a0, a1);
                        float p0, p1;
#ifdef TKV_ATTN_EXP_EMU  // measured slower, build knob only
                        if (i >= 32 - 2 * TKV_ATTN_EXP_EMU) {  // the chunk's last pairs on the FMA pipe
                            unpack_f32x2(ex2_poly2(pack_f32x2(fmaxf(a0, -127.f), fmaxf(a1, -127.f))), p0, p1);
                        } else
#endif
                        {
#ifdef TKV_ATTN_NO_EXP_PROBE  // timing probe only (wrong P): the exponentials skipped
                            p0 = a0;
                            p1 = a1;
#else
                            p0 = ex2(a0);
                            p1 = ex2(a1);
#endif
                        }
#ifdef TKV_ATTN_PTRUNC  // measured slower (DESIGN §8 "Measured and not kept"); kept as a build knob
                        // bf16 P by truncation (one PRMT per pair on the ALU instead of an F2FP), and
                        // the row sum over the same truncated values so O / l stays consistent
                        const uint32_t b0 = __float_as_uint(p0) & 0xffff0000u, b1 = __float_as_uint(p1) & 0xffff0000u;
                        acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], pack_u32x2(b0, b1));
                        pk[i >> 1] = __byte_perm(b0, b1, 0x7632);
#else
                        acc[(i >> 1) & 1] = fadd2(acc[(i >> 1) & 1], pack_f32x2(p0, p1));
                        pk[i >> 1] = pack_bf16x2(p0, p1);
#endif
                    }
                    tmem_st16(tS + 16 * k, pk);
                    if (kPHalf && k == 1) {  // keys 0-63 of P (and O rescaled) before PV's first half
                        if (any_grow) rescale_o();
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(b_phalf(st));
                    }
#ifdef TKV_ATTN_TWOPASS
                    if (k < 3) {
                        tmem_wait_ld();
                        reg_fence32(nxt);
                    }
#endif
                }
                float s0, s1, s2, s3;
                unpack_f32x2(acc[0], s0, s1);
                unpack_f32x2(acc[1], s2, s3);
                l_run += (s0 + s1) + (s2 + s3);
                if (warp == 4 && lane == 0) TR(14, gi);
                if (warp == 8 && lane == 0) TR(21, gi);  // stream 1's exponentials done
                if (!kPHalf && any_grow) rescale_o();
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(b_pfull(st));
                if (warp == 4 && lane == 0) TR(6, gi);
                if (warp == 8 && lane == 0) TR(15, gi);  // stream 1's P ready
            }
            // ---- epilogue: O / l -> bf16 row, then O free for the next item
            const long gl = g + it.n_tiles - 1;
            mbar_wait(b_pvdone(st), int(gl & 1));
            fence_after();
            const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
            __nv_bfloat16* dst = a.out + long(sq.q_row0 + tok) * qw + (it.kvh * G + r % G) * D;
#pragma unroll
            for (int c = 0; c < (wdead ? 0 : D); c += 32) {
                float o[32];
                tmem_ld32(tO + c, o);
                if (live) {
#pragma unroll
                    for (int i = 0; i < 32; i += 8)
                        *reinterpret_cast<uint4*>(dst + c + i) =
                            make_uint4(pack_bf16x2(o[i] * inv, o[i + 1] * inv), pack_bf16x2(o[i + 2] * inv, o[i + 3] * inv),
                                       pack_bf16x2(o[i + 4] * inv, o[i + 5] * inv), pack_bf16x2(o[i + 6] * inv, o[i + 7] * inv));
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(b_ofree(st));
            if (warp == 4 && lane == 0) TR(7, j);
            g += it.n_tiles;
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
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

// [rows][cols] bf16 (cols contiguous), box = 64 cols x box_rows rows, 128-byte swizzle
CUtensorMap rows_map(const void* base, long rows, int cols, int box_rows = BN) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(std::max(1L, rows))};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    const cuuint32_t box[2] = {64, cuuint32_t(box_rows)}, es[2] = {1, 1};  // 64 cols x box_rows rows
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (attention) failed: " + std::to_string(int(r)));
    return m;
}

// the pool as a 4-D tensor {64 cols, rows, 2 halves (128 B apart), kv heads (256 B apart)}: a
// {64, 8, 2, 1} box lands as the [half][8 rows][64] pair of SW128 atoms of one group of a grouped
// paged tile
CUtensorMap pool_group_map(const void* base, long rows, int kvd) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {64, cuuint64_t(std::max(1L, rows)), 2, cuuint64_t(kvd / D)};
    const cuuint64_t strides[3] = {cuuint64_t(kvd) * 2, 128, 256};
    const cuuint32_t box[4] = {64, 8, 2, 1}, es[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (pool groups) failed: " + std::to_string(int(r)));
    return m;
}

// queries [rows][heads][128] bf16: box = 64 dims x G heads x BM/G tokens, so the tile lands as
// BM rows (token-major, head-minor) of 128 bytes with the 128-byte swizzle
CUtensorMap q_map(const void* base, long rows, int heads, int G) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {cuuint64_t(D), cuuint64_t(heads), cuuint64_t(std::max(1L, rows))};
    const cuuint64_t strides[2] = {cuuint64_t(D) * 2, cuuint64_t(heads) * D * 2};
    const cuuint32_t box[3] = {64, cuuint32_t(G), cuuint32_t(BM / G)}, es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (attention Q) failed: " + std::to_string(int(r)));
    return m;
}

}  // namespace

bool attention_tc5_supported(const AttnArgs& a) {
    return a.head_dim == 128 && a.num_heads % a.kv_heads == 0 && BM % (a.num_heads / a.kv_heads) == 0;
}

int attn_tc5_rows_per_tile(int num_heads, int kv_heads) { return 2 * BM / (num_heads / kv_heads); }

void attention_tc5(const AttnArgs& a, const int4* work, int n_work, long ctx_rows, long own_rows, cudaStream_t s) {
    if (n_work == 0) return;
    if (!attention_tc5_supported(a)) throw std::invalid_argument("tcgen05 attention needs head_dim 128");
    if (a.mode == 1 && !a.row_lo) throw std::invalid_argument("tcgen05 block-mask attention needs per-row group starts");
    ensure_smem_optin(reinterpret_cast<const void*>(attn_tc5_kernel), kSmem);
    const int kvd = a.kv_heads * D;
    // paged mode: the pool as [pool rows][kv_dim] — 8-row boxes (mkc) and single-row boxes (mvc)
    // paged mode: the pool as [pool rows][kv_dim] — one {64 cols, 8 rows, 2 halves} box per 8-row
    // group (mkc, 3-D view with the halves as a dimension) and 4 / 2 / 1-row boxes of one half for
    // the runs between table and page boundaries (mp4, mp2, mvc)
    const CUtensorMap mkc = a.kpaged ? pool_group_map(a.vpool, a.pool_rows, kvd)
                            : a.k_hm_rows ? rows_map(a.k_ctx, a.k_hm_rows * a.kv_heads, D) : rows_map(a.k_ctx, ctx_rows, kvd);
    const CUtensorMap mvc = a.kpaged ? rows_map(a.vpool, a.pool_rows, kvd, 1) : rows_map(a.v_ctx, ctx_rows, kvd);
    const CUtensorMap mp4 = a.kpaged ? rows_map(a.vpool, a.pool_rows, kvd, 4) : mvc;
    const CUtensorMap mp2 = a.kpaged ? rows_map(a.vpool, a.pool_rows, kvd, 2) : mvc;
    const CUtensorMap mko = rows_map(a.k_own, own_rows, kvd), mvo = rows_map(a.v_own, own_rows, kvd);
    const CUtensorMap mq = q_map(a.q, own_rows, a.num_heads, a.num_heads / a.kv_heads);
    static const char* trace_path = std::getenv("TKV_ATTN_TRACE");
    uint32_t* trace = nullptr;
    if (trace_path) {
        TKV_CUDA_CHECK(cudaMalloc(&trace, kTraceEvents * 1024 * 4));
        TKV_CUDA_CHECK(cudaMemsetAsync(trace, 0, kTraceEvents * 1024 * 4, s));
    }
    Tc5Args args{a, work, n_work, trace};
    const int n_sm = device_sm_count();
    attn_tc5_kernel<<<std::min(n_work, n_sm), kThreads, kSmem, s>>>(mq, mkc, mvc, mko, mvo, mp4, mp2, args);
    TKV_CUDA_CHECK(cudaGetLastError());
    if (trace) {  // debug only: CTA 0's timeline of the latest launch
        std::vector<uint32_t> h(kTraceEvents * 1024);
        TKV_CUDA_CHECK(cudaStreamSynchronize(s));
        TKV_CUDA_CHECK(cudaMemcpy(h.data(), trace, h.size() * 4, cudaMemcpyDeviceToHost));
        cudaFree(trace);
        if (FILE* f = std::fopen(trace_path, "wb")) {
            std::fwrite(h.data(), 4, h.size(), f);
            std::fclose(f);
        }
    }
}

}  // namespace tkv
