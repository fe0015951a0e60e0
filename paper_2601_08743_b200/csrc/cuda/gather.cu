// Prefix assembly: the device form of assemble() (proj/include/tablekv/attention.hpp:300-362).
//
// One warp per output token row. The warp finds its table segment (binary search over the
// contiguous output ranges), then for each layer and for K and V reads the row out of the
// table's pool pages with 16-byte vector loads, rotates K at the token's global position
// (cursor + t, interleaved pairs, rotary.hpp:21-51) and writes the row into the per-layer
// prefix slab. HBM-bound: algorithmic bytes = rows * 2L * kvdim * (in + out element size).
#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

namespace tkv {

namespace {

template <int EPV>
struct Vec;  // EPV elements held as float
template <>
struct Vec<4> { float v[4]; };
template <>
struct Vec<8> { float v[8]; };

__device__ __forceinline__ void load_in(const uint8_t* p, DType dt, float* f, int& n) {
    const uint4 raw = *reinterpret_cast<const uint4*>(p);
    if (dt == DType::f32) {
        f[0] = __uint_as_float(raw.x);
        f[1] = __uint_as_float(raw.y);
        f[2] = __uint_as_float(raw.z);
        f[3] = __uint_as_float(raw.w);
        n = 4;
    } else {
        float2 a = unpack_bf16x2(raw.x), b = unpack_bf16x2(raw.y), c = unpack_bf16x2(raw.z), d = unpack_bf16x2(raw.w);
        f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y; f[4] = c.x; f[5] = c.y; f[6] = d.x; f[7] = d.y;
        n = 8;
    }
}

__device__ __forceinline__ void store_out(uint8_t* p, DType dt, const float* f, int n) {
    if (dt == DType::f32) {
        for (int i = 0; i < n; i += 4)
            *reinterpret_cast<uint4*>(p + i * 4) =
                make_uint4(__float_as_uint(f[i]), __float_as_uint(f[i + 1]), __float_as_uint(f[i + 2]), __float_as_uint(f[i + 3]));
    } else if (n == 8) {
        *reinterpret_cast<uint4*>(p) =
            make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
    } else {
        *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]));
    }
}

__global__ void gather_rope_kernel(const uint8_t* __restrict__ pool, long page_bytes, const int32_t* __restrict__ page_ids,
                                   const GatherSeg* __restrict__ segs, int n_segs, int total_rows, int L, int kvdim,
                                   int head_dim, DType in_dt, DType out_dt, const double* __restrict__ cos_d,
                                   const double* __restrict__ sin_d, const float* __restrict__ cos_f,
                                   const float* __restrict__ sin_f, uint8_t* __restrict__ out_k,
                                   uint8_t* __restrict__ out_v, long out_rows, int l0, int nl) {
    const int warps = blockDim.x >> 5;
    const int row = blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= total_rows) return;
    int lo = 0, hi = n_segs - 1;
    while (lo < hi) {  // last segment with out_row0 <= row
        const int mid = (lo + hi + 1) >> 1;
        if (segs[mid].out_row0 <= row) lo = mid; else hi = mid - 1;
    }
    const GatherSeg sg = segs[lo];
    const int t = row - sg.out_row0;
    const long pos = sg.pos0 + t;
    const int half = head_dim >> 1;
    const int isz = in_dt == DType::f32 ? 4 : 2, osz = out_dt == DType::f32 ? 4 : 2;
    const int epv = 16 / isz;  // elements per input vector
    const long row_in = long(kvdim) * isz;
    const int nvec = int(row_in / 16);
    const bool exact = (in_dt == DType::f32 && out_dt == DType::f32 && cos_d != nullptr);
    for (int kv = 0; kv < 2; ++kv) {
        uint8_t* out = kv == 0 ? out_k : out_v;
        for (int l = l0; l < l0 + nl; ++l) {
            const long base = ((long(kv) * L + l) * sg.tokens + t) * row_in;
            uint8_t* orow = out + ((long(l - l0) * out_rows) + row) * long(kvdim) * osz;
            for (int vi = lane; vi < nvec; vi += 32) {
                const long off = base + long(vi) * 16;
                const long pg = off / page_bytes;
                const uint8_t* src = pool + long(page_ids[sg.page_off + pg]) * page_bytes + (off - pg * page_bytes);
                float f[8];
                int n;
                load_in(src, in_dt, f, n);
                const int e0 = vi * epv;
                if (kv == 0 && pos != 0) {
                    for (int i = 0; i < n; i += 2) {
                        const int k = ((e0 + i) % head_dim) >> 1;
                        if (exact) {
                            // a*c - b*s, a*s + b*c in double, each product rounded (no FMA contraction),
                            // exactly like the reference's double arithmetic (rotary.hpp:44-47)
                            const double c = cos_d[pos * half + k], s = sin_d[pos * half + k];
                            const double a = f[i], b = f[i + 1];
                            f[i] = float(__dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s)));
                            f[i + 1] = float(__dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c)));
                        } else {
                            const float c = cos_f[pos * half + k], s = sin_f[pos * half + k];
                            const float a = f[i], b = f[i + 1];
                            f[i] = fmaf(a, c, -b * s);
                            f[i + 1] = fmaf(a, s, b * c);
                        }
                    }
                }
                store_out(orow + long(e0) * osz, out_dt, f, n);
            }
        }
    }
}

// Serving fast path (bf16 image -> bf16 slab, one layer): CTA = one chunk of <= kChunkRows rows
// of ONE table segment (host-built list: no per-row segment search), warp = one row; every lane
// issues all of its 16-byte K and V loads (page addressing by shift: power-of-two pages) before
// rotating K and storing.
constexpr int kChunkRows = 8;

__global__ void __launch_bounds__(256) gather_rope_bf16_kernel(const uint8_t* __restrict__ pool, int page_shift,
                                                               const int32_t* __restrict__ page_ids,
                                                               const GatherSeg* __restrict__ segs, const int4* __restrict__ chunks,
                                                               int L, int l, int kvdim, int head_dim,
                                                               const float* __restrict__ cos_f, const float* __restrict__ sin_f,
                                                               uint8_t* __restrict__ out_k, uint8_t* __restrict__ out_v) {
    const int4 ch = chunks[blockIdx.x];  // {seg, t0, rows, 0}
    const int r = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (r >= ch.z) return;
    const GatherSeg sg = segs[ch.x];
    const int t = ch.y + r;
    const long pos = sg.pos0 + t;
    const int vpr = kvdim >> 3;  // 16-byte vectors per row (8 bf16)
    const long row_in = long(kvdim) * 2;
    const long pmask = (1L << page_shift) - 1;
    const int half = head_dim >> 1;
    const int32_t* pages = page_ids + sg.page_off;
    for (int v0 = 0; v0 < vpr; v0 += 128) {
        uint4 kv[2][4];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (c == 1 && !out_v) break;  // K only: the attention reads V from the pages
            const long base = ((long(c) * L + l) * sg.tokens + t) * row_in;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int vi = v0 + lane + 32 * q;
                if (vi < vpr) {
                    const long off = base + long(vi) * 16;
                    kv[c][q] = *reinterpret_cast<const uint4*>(pool + (long(pages[off >> page_shift]) << page_shift) + (off & pmask));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int vi = v0 + lane + 32 * q;
            if (vi >= vpr) continue;
            uint4 w = kv[0][q];
            if (pos != 0) {
                const int k0 = ((vi * 8) % head_dim) >> 1;  // first rotary pair of this vector
                const float4 c = *reinterpret_cast<const float4*>(cos_f + pos * half + k0);
                const float4 sn = *reinterpret_cast<const float4*>(sin_f + pos * half + k0);
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
                const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 ab = unpack_bf16x2(wp[e]);
                    wp[e] = pack_bf16x2(fmaf(ab.x, cc[e], -ab.y * ss[e]), fmaf(ab.x, ss[e], ab.y * cc[e]));
                }
            }
            const long o = (long(sg.out_row0 + t) * kvdim + long(vi) * 8) * 2;
            *reinterpret_cast<uint4*>(out_k + o) = w;
            if (out_v) *reinterpret_cast<uint4*>(out_v + o) = kv[1][q];
        }
    }
}

// TMA-staged variant: CTA = up to kTmaRows rows of one table segment for one layer. One thread
// moves the rows' K and V bytes (contiguous runs of the table image, split only at page
// boundaries) into shared memory with cp.async.bulk, all threads rotate K in place, then bulk
// stores write both runs into the slab — the loads/stores are a handful of bulk copies per CTA
// instead of 16-byte LSU traffic.
constexpr int kTmaRows = 16;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(256) gather_rope_tma_kernel(const uint8_t* __restrict__ pool, int page_shift,
                                                              const int32_t* __restrict__ page_ids,
                                                              const GatherSeg* __restrict__ segs, const int4* __restrict__ chunks,
                                                              int L, int l, int kvdim, int head_dim,
                                                              const float* __restrict__ cos_f, const float* __restrict__ sin_f,
                                                              uint8_t* __restrict__ out_k, uint8_t* __restrict__ out_v,
                                                              long hm_rows) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const int4 ch = chunks[blockIdx.x];  // {seg, t0, rows, 0}
    const GatherSeg sg = segs[ch.x];
    const long row_bytes = long(kvdim) * 2;
    const uint32_t run = uint32_t(ch.z * row_bytes);
    const uint32_t s_k = uint32_t(__cvta_generic_to_shared(sm)), s_v = s_k + run;
    const uint32_t b = uint32_t(__cvta_generic_to_shared(&bar));
    const long pmask = (1L << page_shift) - 1;
    const int32_t* pages = page_ids + sg.page_off;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int n_kv = out_v ? 2 : 1;  // K only when the attention reads V from the pages itself
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n_kv * run) : "memory");
        for (int kv = 0; kv < n_kv; ++kv) {
            long off = ((long(kv) * L + l) * sg.tokens + ch.y) * row_bytes;
            uint32_t dst = kv ? s_v : s_k, left = run;
            while (left) {  // split the run at page boundaries
                const long room = (1L << page_shift) - (off & pmask);
                const uint32_t n = uint32_t(long(left) < room ? long(left) : room);
                bulk_g2s(dst, pool + (long(pages[off >> page_shift]) << page_shift) + (off & pmask), n, b);
                off += n, dst += n, left -= n;
            }
        }
    }
    __syncthreads();
    {  // wait for both runs
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done)
                         : "r"(b)
                         : "memory");
    }
    const int vpr = kvdim >> 3, half = head_dim >> 1;
    if (hm_rows) {  // head-major K: rotate in registers and store each 16-byte vector straight to its head's block
        for (int i = threadIdx.x; i < ch.z * vpr; i += blockDim.x) {
            const int r = i / vpr, vi = i - r * vpr;
            const long pos = sg.pos0 + ch.y + r;
            uint4 w = *reinterpret_cast<const uint4*>(sm + long(r) * row_bytes + vi * 16);
            const int e0 = vi * 8, hh = e0 / head_dim, d0 = e0 - hh * head_dim;
            if (pos != 0) {
                const float4 c = *reinterpret_cast<const float4*>(cos_f + pos * half + (d0 >> 1));
                const float4 sn = *reinterpret_cast<const float4*>(sin_f + pos * half + (d0 >> 1));
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
                const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 ab = unpack_bf16x2(wp[e]);
                    wp[e] = pack_bf16x2(fmaf(ab.x, cc[e], -ab.y * ss[e]), fmaf(ab.x, ss[e], ab.y * cc[e]));
                }
            }
            *reinterpret_cast<uint4*>(out_k + ((long(hh) * hm_rows + sg.out_row0 + ch.y + r) * head_dim + d0) * 2) = w;
        }
        return;
    }
    for (int i = threadIdx.x; i < ch.z * vpr; i += blockDim.x) {
        const int r = i / vpr, vi = i - r * vpr;
        const long pos = sg.pos0 + ch.y + r;
        if (pos == 0) continue;
        uint4* p = reinterpret_cast<uint4*>(sm + long(r) * row_bytes + vi * 16);
        uint4 w = *p;
        const int k0 = ((vi * 8) % head_dim) >> 1;
        const float4 c = *reinterpret_cast<const float4*>(cos_f + pos * half + k0);
        const float4 sn = *reinterpret_cast<const float4*>(sin_f + pos * half + k0);
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
        const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 ab = unpack_bf16x2(wp[e]);
            wp[e] = pack_bf16x2(fmaf(ab.x, cc[e], -ab.y * ss[e]), fmaf(ab.x, ss[e], ab.y * cc[e]));
        }
        *p = w;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> bulk store reads
    __syncthreads();
    if (threadIdx.x == 0) {
        const long o = long(sg.out_row0 + ch.y) * row_bytes;
        bulk_s2g(out_k + o, s_k, run);
        if (out_v) bulk_s2g(out_v + o, s_v, run);
        asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
}

}  // namespace

bool gather_use_tma() {  // TKV_GATHER=lsu selects the 16-byte LSU kernel (A/B measurements)
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TKV_GATHER");
        v = (e && std::string(e) == "lsu") ? 0 : 1;
    }
    return v == 1;
}

int gather_chunks(const GatherSeg* segs, int n_segs, std::vector<int4>& out) {
    out.clear();
    const int rows = gather_use_tma() ? kTmaRows : kChunkRows;
    for (int s = 0; s < n_segs; ++s)
        for (int t = 0; t < segs[s].tokens; t += rows) out.push_back(make_int4(s, t, std::min(rows, segs[s].tokens - t), 0));
    return int(out.size());
}

void launch_gather_rope_bf16(const uint8_t* pool, size_t page_bytes, const int32_t* d_page_ids, const GatherSeg* d_segs,
                             const int4* d_chunks, int n_chunks, int L, int l, int kvdim, int head_dim, const float* cos_f,
                             const float* sin_f, void* out_k, void* out_v, long out_rows, cudaStream_t s, bool k_head_major) {
    if (n_chunks <= 0) return;
    if (k_head_major && (out_v || !gather_use_tma())) throw std::invalid_argument("gather: head-major K needs the TMA kernel, K only");
    if (kvdim % 8 || head_dim % 8) throw std::invalid_argument("gather: kv row must hold whole 16-byte vectors");
    if (page_bytes & (page_bytes - 1)) throw std::invalid_argument("gather fast path: page size must be a power of two");
    int shift = 0;
    while ((size_t(1) << shift) < page_bytes) ++shift;
    if (gather_use_tma()) {
        // K only (paged V) needs half the staging: twice the CTAs per SM, twice the bytes in flight
        const int smem = (out_v ? 2 : 1) * kTmaRows * kvdim * 2;
        ensure_smem_optin(reinterpret_cast<const void*>(gather_rope_tma_kernel), smem);
        gather_rope_tma_kernel<<<n_chunks, 256, smem, s>>>(pool, shift, d_page_ids, d_segs, d_chunks, L, l, kvdim, head_dim,
                                                           cos_f, sin_f, static_cast<uint8_t*>(out_k), static_cast<uint8_t*>(out_v),
                                                           k_head_major ? out_rows : 0L);
    } else {
        gather_rope_bf16_kernel<<<n_chunks, 32 * kChunkRows, 0, s>>>(pool, shift, d_page_ids, d_segs, d_chunks, L, l, kvdim,
                                                                     head_dim, cos_f, sin_f, static_cast<uint8_t*>(out_k),
                                                                     static_cast<uint8_t*>(out_v));
    }
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_gather_rope(const uint8_t* pool, size_t page_bytes, const int32_t* d_page_ids, const GatherSeg* d_segs,
                        int n_segs, int total_rows, int L, int kvdim, int head_dim, DType in_dt, DType out_dt,
                        const double* cos_d, const double* sin_d, const float* cos_f, const float* sin_f, void* out_k,
                        void* out_v, long out_rows, cudaStream_t s, int l0, int nl) {
    if (total_rows <= 0 || n_segs <= 0) return;
    if (nl < 0) nl = L - l0;
    if (l0 < 0 || l0 + nl > L) throw std::invalid_argument("gather: layer range outside the image");
    if ((long(kvdim) * dtype_size(in_dt)) % 16) throw std::invalid_argument("gather: kv row must be a multiple of 16 bytes");
    const int warps = 8;
    gather_rope_kernel<<<ceil_div(total_rows, warps), warps * 32, 0, s>>>(
        pool, long(page_bytes), d_page_ids, d_segs, n_segs, total_rows, L, kvdim, head_dim, in_dt, out_dt, cos_d, sin_d,
        cos_f, sin_f, static_cast<uint8_t*>(out_k), static_cast<uint8_t*>(out_v), out_rows, l0, nl);
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
