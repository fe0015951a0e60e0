// Tensor-core attention over [cached prefix ; own rows] — detail::attend of the serving path
// (proj/include/tablekv/attention.hpp:129-176, used by query_attend :406-407 and prefill :238).
//
// CTA = (sequence, kv head, tile of 64 query rows). With GQA the 64 rows are
// 64/G tokens x the G query heads sharing that kv head, so every K/V tile is read once for
// all of them. K/V tiles (64 keys) stream through a double-buffered cp.async ring into
// XOR-swizzled smem; S = Q.K^T and O += P.V run on mma.sync m16n8k16 (bf16 in, f32 acc) with
// an online softmax in registers. Masks: mode 0 (query rows see every cached row + causal
// own rows), mode 1 (block-causal by group id, BlockMask::allows, attention.hpp:37-39).
#include "attn_tc.cuh"
#include "common.cuh"

namespace tkv {

namespace {

constexpr int kRows = 64;  // query rows per CTA (4 warps x 16)
constexpr int kKeys = 64;  // keys per tile

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

// smem tile [64 rows][D] bf16; 16-byte chunk c of row r lives at chunk (c ^ (r & 7)) when the
// row has >= 8 chunks (conflict-free ldmatrix), unswizzled for D = 16.
template <int D>
__device__ __forceinline__ uint32_t tile_off(int r, int c16) {
    constexpr int CPR = D / 8;  // 16-byte chunks per row
    const int pc = CPR >= 8 ? (c16 ^ (r & 7)) : c16;
    return uint32_t((r * CPR + pc) * 16);
}

template <int D>
__global__ void __launch_bounds__(128) attn_kernel(AttnArgs a) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int TB = kRows * D * 2;  // bytes per tile
    const uint32_t sQ = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t sK0 = sQ + TB, sV0 = sQ + 2 * TB;  // K/V buffers: [buf][K,V] at +TB*(1 + 2*buf + {0,1})

    const int4 tile = a.tiles[blockIdx.x];
    const AttnSeq sq = a.seqs[tile.x];
    const int tok0 = tile.y, kvh = tile.z;
    const int G = a.num_heads / a.kv_heads;
    const int qw = a.num_heads * D, kw = a.kv_heads * D;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int CPR = D / 8;

    // ---- Q tile: row r = (token tok0 + r / G, head kvh * G + r % G)
    for (int idx = threadIdx.x; idx < kRows * CPR; idx += 128) {
        const int r = idx / CPR, c = idx % CPR;
        const int tok = tok0 + r / G;
        const bool ok = tok < sq.n_own;
        const __nv_bfloat16* src = a.q + long(sq.q_row0 + (ok ? tok : 0)) * qw + (kvh * G + r % G) * D + c * 8;
        cp_async16(sQ + tile_off<D>(r, c), src, ok);
    }
    cp_commit();

    const int n_keys = sq.n_ctx + sq.n_own;
    const int last_tok = min(sq.n_own - 1, tok0 + (kRows / G) - 1);
    const int key_end = min(n_keys, sq.n_ctx + last_tok + 1);  // causal bound for the tile
    const int n_tiles = (key_end + kKeys - 1) / kKeys;

    auto load_kv = [&](int t, int buf) {
        const uint32_t dk = sK0 + uint32_t(2 * buf) * TB, dv = dk + TB;
        for (int idx = threadIdx.x; idx < kKeys * CPR; idx += 128) {
            const int r = idx / CPR, c = idx % CPR;
            const int j = t * kKeys + r;
            const bool ok = j < key_end;
            const long row = !ok ? 0 : (j < sq.n_ctx ? long(sq.ctx_row0 + j) : long(sq.q_row0 + j - sq.n_ctx));
            const __nv_bfloat16* kb = (j < sq.n_ctx ? a.k_ctx : a.k_own) + row * kw + kvh * D + c * 8;
            const __nv_bfloat16* vb = (j < sq.n_ctx ? a.v_ctx : a.v_own) + row * kw + kvh * D + c * 8;
            cp_async16(dk + tile_off<D>(r, c), ok ? kb : a.k_own, ok);
            cp_async16(dv + tile_off<D>(r, c), ok ? vb : a.v_own, ok);
        }
        cp_commit();
    };

    if (n_tiles > 0) load_kv(0, 0);

    // per-thread rows: g and g + 8 inside the warp's 16
    const int g = lane >> 2, tq = lane & 3;
    const int r_lo = warp * 16 + g, r_hi = r_lo + 8;
    const int tok_lo = min(tok0 + r_lo / G, sq.n_own - 1), tok_hi = min(tok0 + r_hi / G, sq.n_own - 1);
    const int grp_lo = a.mode == 1 ? a.group[sq.q_row0 + tok_lo] : -1;
    const int grp_hi = a.mode == 1 ? a.group[sq.q_row0 + tok_hi] : -1;

    cp_wait<0>();  // Q (and first K/V) landed
    __syncthreads();
    uint32_t qf[D / 16][4];
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(sQ + tile_off<D>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
    }

    float o[D / 8][4];
#pragma unroll
    for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;
    const float sl2 = a.scale * 1.4426950408889634f;

    for (int t = 0; t < n_tiles; ++t) {
        const int buf = t & 1;
        if (t + 1 < n_tiles) {
            load_kv(t + 1, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const uint32_t sK = sK0 + uint32_t(2 * buf) * TB, sV = sK + TB;

        // ---- S = Q K^T (16 x 64 per warp)
        float s[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) s[nb][0] = s[nb][1] = s[nb][2] = s[nb][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
            for (int nb = 0; nb < 8; nb += 2) {
                const int r = nb * 8 + (lane & 7) + (lane >> 4) * 8;
                const int c = kk * 2 + ((lane >> 3) & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(sK + tile_off<D>(r, c), b0, b1, b2, b3);
                mma16816(s[nb], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b0, b1);
                mma16816(s[nb + 1], qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], b2, b3);
            }
        }
        // ---- mask + online softmax (base-2)
        float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = t * kKeys + nb * 8 + 2 * tq + e;
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
        uint32_t p[8][2];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
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
        // ---- O += P V
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {  // 16 keys per step
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
        __syncthreads();  // buffer `buf` is refilled two iterations later
    }

    // ---- normalise and store (rows past n_own are padding)
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
    const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
    const int t_lo = tok0 + r_lo / G, t_hi = tok0 + r_hi / G;
    const int h_lo = kvh * G + r_lo % G, h_hi = kvh * G + r_hi % G;
#pragma unroll
    for (int nd = 0; nd < D / 8; ++nd) {
        const int col = nd * 8 + 2 * tq;
        if (t_lo < sq.n_own)
            *reinterpret_cast<uint32_t*>(a.out + long(sq.q_row0 + t_lo) * qw + h_lo * D + col) =
                pack_bf16x2(o[nd][0] * inv_lo, o[nd][1] * inv_lo);
        if (t_hi < sq.n_own)
            *reinterpret_cast<uint32_t*>(a.out + long(sq.q_row0 + t_hi) * qw + h_hi * D + col) =
                pack_bf16x2(o[nd][2] * inv_hi, o[nd][3] * inv_hi);
    }
}

template <int D>
void launch_d(const AttnArgs& a, int n_tiles, cudaStream_t s) {
    const int smem = 5 * kRows * D * 2;  // Q + 2 x (K, V)
    static bool attr = false;
    if (!attr) {
        TKV_CUDA_CHECK(cudaFuncSetAttribute(attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr = true;
    }
    attn_kernel<D><<<n_tiles, 128, smem, s>>>(a);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

int attn_rows_per_tile(int num_heads, int kv_heads) { return kRows / (num_heads / kv_heads); }

void attention_bf16(const AttnArgs& a, int n_tiles, cudaStream_t s) {
    if (n_tiles == 0) return;
    if ((a.num_heads % a.kv_heads) || (kRows % (a.num_heads / a.kv_heads)))
        throw std::invalid_argument("attention: num_heads / kv_heads must divide 64");
    switch (a.head_dim) {
        case 16: launch_d<16>(a, n_tiles, s); break;
        case 32: launch_d<32>(a, n_tiles, s); break;
        case 64: launch_d<64>(a, n_tiles, s); break;
        case 128: launch_d<128>(a, n_tiles, s); break;
        default: throw std::invalid_argument("attention: head_dim must be 16, 32, 64 or 128");
    }
}

}  // namespace tkv
