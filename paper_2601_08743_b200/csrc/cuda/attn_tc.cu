// Tensor-core attention over [cached prefix ; own rows] — detail::attend of the serving path
// (proj/include/tablekv/attention.hpp:129-176, used by query_attend :406-407 and prefill :238).
//
// CTA = (sequence, kv head, chunk of up to 256 query rows). With GQA the rows are tokens x the G
// query heads sharing that kv head, so for a cached query (tens of suffix tokens) ONE CTA holds
// all of its rows for a kv head and every K/V tile fetched from L2/HBM feeds 16 warps. K/V tiles
// of 32 keys stream through a 4-stage cp.async ring in XOR-swizzled smem (3 tiles in flight while
// one is consumed); S = Q.K^T and O += P.V run on mma.sync m16n8k16 (bf16 in, f32 acc) with an
// online softmax in registers; tiles entirely inside the cached prefix skip the mask, warps whose
// rows are all padding skip the math. Masks: mode 0 (rows see every cached row + causal own rows),
// mode 1 (block-causal by group id, BlockMask::allows, attention.hpp:37-39).
#include "attn_tc.cuh"
#include "common.cuh"

namespace tkv {

namespace {

constexpr int kWarps = 16;
constexpr int kRows = 16 * kWarps;  // query rows per CTA
constexpr int kKeys = 32;           // keys per tile
constexpr int kStages = 4;
constexpr int kThreads = 32 * kWarps;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// smem tile [rows][D] bf16; 16-byte chunk c of row r lives at chunk (c ^ (r & 7)) when the row
// has >= 8 chunks (conflict-free ldmatrix), unswizzled otherwise.
template <int D>
__device__ __forceinline__ uint32_t tile_off(int r, int c16) {
    constexpr int CPR = D / 8;
    const int pc = CPR >= 8 ? (c16 ^ (r & 7)) : c16;
    return uint32_t((r * CPR + pc) * 16);
}

template <int D>
struct AttnSmem {
    static constexpr int q_bytes = kRows * D * 2;
    static constexpr int kv_bytes = kKeys * D * 2;  // one K or V tile
    static constexpr int stage_bytes = 2 * kv_bytes;
    static constexpr int total = q_bytes + kStages * stage_bytes;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1) attn_kernel(AttnArgs a) {
    using S = AttnSmem<D>;
    extern __shared__ __align__(128) uint8_t sm[];
    const uint32_t sQ = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t sKV0 = sQ + S::q_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int4 tile = a.tiles[blockIdx.x];
    const AttnSeq sq = a.seqs[tile.x];
    const int tok0 = tile.y, kvh = tile.z;
    const int G = a.num_heads / a.kv_heads;
    const int qw = a.num_heads * D, kw = a.kv_heads * D;
    constexpr int CPR = D / 8;
    const int tok_cap = kRows / G;  // tokens per CTA
    const int n_tok = min(tok_cap, sq.n_own - tok0);
    const int rows = n_tok * G;

    // ---- Q rows: r = (token tok0 + r / G, head kvh * G + r % G)
    for (int idx = threadIdx.x; idx < kRows * CPR; idx += kThreads) {
        const int r = idx / CPR, c = idx % CPR;
        const bool ok = r < rows;
        const __nv_bfloat16* src = a.q + long(sq.q_row0 + tok0 + (ok ? r / G : 0)) * qw + (kvh * G + r % G) * D + c * 8;
        cp_async16(sQ + tile_off<D>(r, c), src, ok);
    }
    cp_commit();

    const int n_keys = sq.n_ctx + sq.n_own;
    const int key_end = min(n_keys, sq.n_ctx + tok0 + n_tok);  // causal bound of the last row
    const int n_tiles = (key_end + kKeys - 1) / kKeys;

    auto load_kv = [&](int t) {
        if (t < n_tiles) {
            const uint32_t dk = sKV0 + uint32_t(t % kStages) * S::stage_bytes, dv = dk + S::kv_bytes;
            for (int idx = threadIdx.x; idx < kKeys * CPR; idx += kThreads) {
                const int r = idx / CPR, c = idx % CPR;
                const int j = t * kKeys + r;
                const bool ok = j < key_end;
                const bool ctx = j < sq.n_ctx;
                const long row = !ok ? 0 : (ctx ? long(sq.ctx_row0 + j) : long(sq.q_row0 + j - sq.n_ctx));
                const __nv_bfloat16* kb = (ctx ? a.k_ctx : a.k_own) + row * kw + kvh * D + c * 8;
                const __nv_bfloat16* vb = (ctx ? a.v_ctx : a.v_own) + row * kw + kvh * D + c * 8;
                cp_async16(dk + tile_off<D>(r, c), ok ? kb : a.k_own, ok);
                cp_async16(dv + tile_off<D>(r, c), ok ? vb : a.v_own, ok);
            }
        }
        cp_commit();  // always commit so group counting stays uniform
    };
#pragma unroll
    for (int t = 0; t < kStages - 1; ++t) load_kv(t);

    const int g8 = lane >> 2, tq = lane & 3;
    const int r_lo = warp * 16 + g8, r_hi = r_lo + 8;
    const bool warp_live = warp * 16 < rows;
    const int tok_lo = min(tok0 + r_lo / G, sq.n_own - 1), tok_hi = min(tok0 + r_hi / G, sq.n_own - 1);
    const int grp_lo = a.mode == 1 ? a.group[sq.q_row0 + tok_lo] : -1;
    const int grp_hi = a.mode == 1 ? a.group[sq.q_row0 + tok_hi] : -1;
    const int warp_key_end = sq.n_ctx + min(tok0 + (warp * 16 + 15) / G, sq.n_own - 1) + 1;  // causal bound of the warp
    const int q_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8, q_half = lane >> 4;

    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    const float sl2 = a.scale * 1.4426950408889634f;

    for (int t = 0; t < n_tiles; ++t) {
        load_kv(t + kStages - 1);
        cp_wait<kStages - 1>();  // tile t (and Q) landed for this thread
        __syncthreads();
        const int j0 = t * kKeys;
        if (warp_live && j0 < warp_key_end) {
            const uint32_t sK = sKV0 + uint32_t(t % kStages) * S::stage_bytes, sV = sK + S::kv_bytes;
            float s[4][4];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                uint32_t q0, q1, q2, q3;
                ldsm_x4(sQ + tile_off<D>(q_row, kk * 2 + q_half), q0, q1, q2, q3);
#pragma unroll
                for (int nb = 0; nb < 4; nb += 2) {
                    const int r = nb * 8 + (lane & 7) + (lane >> 4) * 8;
                    const int c = kk * 2 + ((lane >> 3) & 1);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(sK + tile_off<D>(r, c), b0, b1, b2, b3);
                    mma16816(s[nb], q0, q1, q2, q3, b0, b1);
                    mma16816(s[nb + 1], q0, q1, q2, q3, b2, b3);
                }
            }
            float mx_lo = m_lo, mx_hi = m_hi;
            if (a.mode == 0 && j0 + kKeys <= sq.n_ctx) {  // inside the cached prefix: all visible
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        s[nb][e] *= sl2;
                        s[nb][2 + e] *= sl2;
                        mx_lo = fmaxf(mx_lo, s[nb][e]);
                        mx_hi = fmaxf(mx_hi, s[nb][2 + e]);
                    }
            } else {
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = j0 + nb * 8 + 2 * tq + e;
                        bool ok_lo = j <= sq.n_ctx + tok_lo, ok_hi = j <= sq.n_ctx + tok_hi;
                        if (a.mode == 1 && j < n_keys) {
                            const int gj = a.group[sq.q_row0 + j - sq.n_ctx];
                            ok_lo = ok_lo && (grp_lo == -1 || grp_lo == gj);
                            ok_hi = ok_hi && (grp_hi == -1 || grp_hi == gj);
                        }
                        s[nb][e] = ok_lo ? s[nb][e] * sl2 : -INFINITY;
                        s[nb][2 + e] = ok_hi ? s[nb][2 + e] * sl2 : -INFINITY;
                        mx_lo = fmaxf(mx_lo, s[nb][e]);
                        mx_hi = fmaxf(mx_hi, s[nb][2 + e]);
                    }
            }
            mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
            mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
            mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
            mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
            const float base_lo = mx_lo == -INFINITY ? 0.f : mx_lo, base_hi = mx_hi == -INFINITY ? 0.f : mx_hi;
            const float corr_lo = exp2f(m_lo - base_lo), corr_hi = exp2f(m_hi - base_hi);
            m_lo = mx_lo;
            m_hi = mx_hi;
            float sum_lo = 0.f, sum_hi = 0.f;
            uint32_t p[4][2];
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) {
                const float p0 = exp2f(s[nb][0] - base_lo), p1 = exp2f(s[nb][1] - base_lo);
                const float p2 = exp2f(s[nb][2] - base_hi), p3 = exp2f(s[nb][3] - base_hi);
                sum_lo += p0 + p1;
                sum_hi += p2 + p3;
                p[nb][0] = pack_bf16x2(p0, p1);
                p[nb][1] = pack_bf16x2(p2, p3);
            }
            l_lo = l_lo * corr_lo + sum_lo;
            l_hi = l_hi * corr_hi + sum_hi;
#pragma unroll
            for (int i = 0; i < D / 8; ++i) {
                o[i][0] *= corr_lo;
                o[i][1] *= corr_lo;
                o[i][2] *= corr_hi;
                o[i][3] *= corr_hi;
            }
#pragma unroll
            for (int kb = 0; kb < kKeys / 16; ++kb) {
                const uint32_t a0 = p[2 * kb][0], a1 = p[2 * kb][1], a2 = p[2 * kb + 1][0], a3 = p[2 * kb + 1][1];
#pragma unroll
                for (int nd = 0; nd < D / 8; nd += 2) {
                    const int r = kb * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
                    const int c = nd + (lane >> 4);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4_t(sV + tile_off<D>(r, c), b0, b1, b2, b3);
                    mma16816(o[nd], a0, a1, a2, a3, b0, b1);
                    mma16816(o[nd + 1], a0, a1, a2, a3, b2, b3);
                }
            }
        }
        __syncthreads();  // slot t % kStages is refilled by the next iteration's load
    }
    cp_wait<0>();
    if (!warp_live) return;

    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
    const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
    const int h_lo = kvh * G + r_lo % G, h_hi = kvh * G + r_hi % G;
#pragma unroll
    for (int nd = 0; nd < D / 8; ++nd) {
        const int col = nd * 8 + 2 * tq;
        if (r_lo < rows)
            *reinterpret_cast<uint32_t*>(a.out + long(sq.q_row0 + tok0 + r_lo / G) * qw + h_lo * D + col) =
                pack_bf16x2(o[nd][0] * inv_lo, o[nd][1] * inv_lo);
        if (r_hi < rows)
            *reinterpret_cast<uint32_t*>(a.out + long(sq.q_row0 + tok0 + r_hi / G) * qw + h_hi * D + col) =
                pack_bf16x2(o[nd][2] * inv_hi, o[nd][3] * inv_hi);
    }
}

template <int D>
void launch_d(const AttnArgs& a, int n_tiles, cudaStream_t s) {
    const int smem = AttnSmem<D>::total;
    ensure_smem_optin(reinterpret_cast<const void*>(attn_kernel<D>), smem);
    attn_kernel<D><<<n_tiles, kThreads, smem, s>>>(a);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

int attn_rows_per_tile(int num_heads, int kv_heads) { return kRows / (num_heads / kv_heads); }

void attention_bf16(const AttnArgs& a, int n_tiles, cudaStream_t s) {
    if (n_tiles == 0) return;
    if ((a.num_heads % a.kv_heads) || (kRows % (a.num_heads / a.kv_heads)))
        throw std::invalid_argument("attention: num_heads / kv_heads must divide 256");
    switch (a.head_dim) {
        case 16: launch_d<16>(a, n_tiles, s); break;
        case 32: launch_d<32>(a, n_tiles, s); break;
        case 64: launch_d<64>(a, n_tiles, s); break;
        case 128: launch_d<128>(a, n_tiles, s); break;
        default: throw std::invalid_argument("attention: head_dim must be 16, 32, 64 or 128");
    }
}

}  // namespace tkv
