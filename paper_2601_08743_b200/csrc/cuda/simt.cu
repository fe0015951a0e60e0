// Reference-precision forward kernels (T = float | double storage, double accumulation).
//
// These reproduce the reference arithmetic of proj/include/tablekv/attention.hpp:84-203 and
// rotary.hpp:21-51 operation for operation: one thread owns one output and accumulates in
// the reference's sequential order with explicitly rounded double ops (no contraction), so
// for T = float the results are bit-identical up to the libm exp() in softmax. They back the
// f32/f64 "parity" model mode (tiny reference configs, drop-in prefill/query_attend
// wrappers); the bf16 tensor-core path (gemm_tc.cu, attn_tc.cu) is the performance path.
#include <algorithm>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace tkv {

namespace {

template <typename T>
__global__ void embed_kernel(const T* __restrict__ emb, const int32_t* __restrict__ tok, int n, int hidden, T* __restrict__ x) {
    const long total = long(n) * hidden;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const long t = i / hidden, c = i - t * hidden;
        x[i] = emb[long(tok[t]) * hidden + c];
    }
}

template <typename T>
__global__ void layer_norm_kernel(const T* __restrict__ x, T* __restrict__ out, int rows, int hidden, int rms, double eps) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const T* row = x + long(r) * hidden;
    T* orow = out + long(r) * hidden;
    if (rms) {
        double ss = 0.0;
        for (int i = 0; i < hidden; ++i) ss = __dadd_rn(ss, __dmul_rn(double(row[i]), double(row[i])));
        const double inv = 1.0 / sqrt(ss / hidden + eps);
        for (int i = 0; i < hidden; ++i) orow[i] = T(__dmul_rn(double(row[i]), inv));
        return;
    }
    double mean = 0.0;
    for (int i = 0; i < hidden; ++i) mean = __dadd_rn(mean, double(row[i]));
    mean /= hidden;
    double var = 0.0;
    for (int i = 0; i < hidden; ++i) {
        const double d = __dsub_rn(double(row[i]), mean);
        var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var /= hidden;
    const double inv = 1.0 / sqrt(var + eps);
    for (int i = 0; i < hidden; ++i) orow[i] = T(__dmul_rn(__dsub_rn(double(row[i]), mean), inv));
}

// y[t][r] = sum_c w[r][c] * x[t][c]  (matmul_rows, attention.hpp:107-122), optional SiLU
// applied to the stored value (ffn_block, attention.hpp:200).
template <typename T>
__global__ void matmul_kernel(const T* __restrict__ w, const T* __restrict__ x, T* __restrict__ y, int rows, int cols,
                              int tokens, int silu) {
    const long i = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (i >= long(tokens) * rows) return;
    const int t = int(i / rows), r = int(i - long(t) * rows);
    const T* wr = w + long(r) * cols;
    const T* xr = x + long(t) * cols;
    double acc = 0.0;
    for (int c = 0; c < cols; ++c) acc = __dadd_rn(acc, __dmul_rn(double(wr[c]), double(xr[c])));
    T v = T(acc);
    if (silu) {
        const double z = double(v);
        v = T(z / (1.0 + exp(-z)));
    }
    y[i] = v;
}

template <typename T>
__global__ void add_kernel(T* __restrict__ x, const T* __restrict__ y, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        x[i] = T(__dadd_rn(double(x[i]), double(y[i])));
}

template <typename T>
__global__ void mul_kernel(T* __restrict__ x, const T* __restrict__ y, long n) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
        x[i] = T(__dmul_rn(double(x[i]), double(y[i])));
}

template <typename T>
__global__ void rope_kernel(T* __restrict__ x, const int64_t* __restrict__ pos, int n, int heads, int d,
                            const double* __restrict__ cs, const double* __restrict__ sn, int table_pos) {
    const int half = d >> 1;
    const long total = long(n) * heads * half;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const long t = i / (long(heads) * half);
        const int rem = int(i - t * heads * half);
        const int h = rem / half, k = rem - h * half;
        const long p = pos[t];
        if (p == 0) continue;
        double c, s;
        if (p > 0 && p < table_pos) {
            c = cs[p * half + k];
            s = sn[p * half + k];
        } else {  // negative or out-of-table positions: recompute (rotary.hpp:36-38)
            const double invf = pow(10000.0, -2.0 * k / d);
            c = cos(double(p) * invf);
            s = sin(double(p) * invf);
        }
        T* e = x + t * long(heads) * d + long(h) * d + 2 * k;
        const double a = double(e[0]), b = double(e[1]);
        e[0] = T(__dsub_rn(__dmul_rn(a, c), __dmul_rn(b, s)));
        e[1] = T(__dadd_rn(__dmul_rn(a, s), __dmul_rn(b, c)));
    }
}

// detail::attend (attention.hpp:129-176): one thread per (own row, q head), sequential over
// keys in the combined [ctx ; own] index space, scores kept in a scratch row.
template <typename T>
__global__ void attend_kernel(const T* __restrict__ q, const T* __restrict__ k_own, const T* __restrict__ v_own,
                              const T* __restrict__ k_ctx, const T* __restrict__ v_ctx, const int32_t* __restrict__ group,
                              const AttnSeq* __restrict__ seqs, int n_seqs, int total_q, T* __restrict__ out, int H,
                              int Hkv, int d, int mode, double* __restrict__ scratch, int max_keys) {
    const long idx = blockIdx.x * long(blockDim.x) + threadIdx.x;
    if (idx >= long(total_q) * H) return;
    const int row = int(idx / H), h = int(idx - long(row) * H);
    int s = 0;
    while (s + 1 < n_seqs && seqs[s + 1].q_row0 <= row) ++s;
    const AttnSeq sq = seqs[s];
    const int i = row - sq.q_row0;
    const int kh = h / (H / Hkv);
    const int qw = H * d, kw = Hkv * d;
    const T* qv = q + long(row) * qw + long(h) * d;
    const double scale = 1.0 / sqrt(double(d));
    double* sc = scratch + idx * long(max_keys);
    const int limit = sq.n_ctx + i + 1;
    auto key = [&](int j) -> const T* {
        return j < sq.n_ctx ? k_ctx + long(sq.ctx_row0 + j) * kw + long(kh) * d
                            : k_own + long(sq.q_row0 + j - sq.n_ctx) * kw + long(kh) * d;
    };
    auto val = [&](int j) -> const T* {
        return j < sq.n_ctx ? v_ctx + long(sq.ctx_row0 + j) * kw + long(kh) * d
                            : v_own + long(sq.q_row0 + j - sq.n_ctx) * kw + long(kh) * d;
    };
    auto allowed = [&](int j) -> bool {
        if (mode == 0) return true;
        const int gi = group[sq.q_row0 + i];
        return gi == -1 || gi == group[sq.q_row0 + j - sq.n_ctx];
    };
    double mx = -1e300;
    bool any = false;
    for (int j = 0; j < limit; ++j) {
        if (!allowed(j)) continue;
        const T* kv = key(j);
        double dot = 0.0;
        for (int e = 0; e < d; ++e) dot = __dadd_rn(dot, __dmul_rn(double(qv[e]), double(kv[e])));
        sc[j] = __dmul_rn(dot, scale);
        mx = fmax(mx, sc[j]);
        any = true;
    }
    T* o = out + long(row) * qw + long(h) * d;
    if (!any) {
        for (int e = 0; e < d; ++e) o[e] = T(0);
        return;
    }
    double den = 0.0;
    for (int j = 0; j < limit; ++j) {
        if (!allowed(j)) continue;
        sc[j] = exp(__dsub_rn(sc[j], mx));
        den = __dadd_rn(den, sc[j]);
    }
    for (int e = 0; e < d; ++e) {
        double acc = 0.0;
        for (int j = 0; j < limit; ++j) {
            if (!allowed(j)) continue;
            acc = __dadd_rn(acc, __dmul_rn(sc[j], double(val(j)[e])));
        }
        o[e] = T(acc / den);
    }
}

inline int grid_for(long n, int threads) { return int(std::min<long>((n + threads - 1) / threads, 1L << 20)); }

}  // namespace

#define TKV_DISPATCH_REF(dt, ...)                                                  \
    do {                                                                           \
        if ((dt) == DType::f32) { using T = float; __VA_ARGS__; }                  \
        else if ((dt) == DType::f64) { using T = double; __VA_ARGS__; }            \
        else throw std::invalid_argument("reference-precision kernels need f32/f64"); \
    } while (0)

void launch_embed(const void* emb, DType dt, const int32_t* tokens, int n, int hidden, void* x, cudaStream_t s) {
    if (n == 0) return;
    TKV_DISPATCH_REF(dt, embed_kernel<T><<<grid_for(long(n) * hidden, 256), 256, 0, s>>>(
                             static_cast<const T*>(emb), tokens, n, hidden, static_cast<T*>(x)));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_layer_norm_ref(const void* x, void* out, DType dt, int rows, int hidden, int rms, double eps, cudaStream_t s) {
    if (rows == 0) return;
    TKV_DISPATCH_REF(dt, layer_norm_kernel<T><<<ceil_div(rows, 64), 64, 0, s>>>(
                             static_cast<const T*>(x), static_cast<T*>(out), rows, hidden, rms, eps));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_matmul_ref(const void* w, const void* x, void* y, DType dt, int rows_out, int cols_in, int tokens,
                       int act_silu, cudaStream_t s) {
    const long n = long(tokens) * rows_out;
    if (n == 0) return;
    TKV_DISPATCH_REF(dt, matmul_kernel<T><<<grid_for(n, 128), 128, 0, s>>>(
                             static_cast<const T*>(w), static_cast<const T*>(x), static_cast<T*>(y), rows_out, cols_in,
                             tokens, act_silu));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_add_ref(void* x, const void* y, DType dt, long n, cudaStream_t s) {
    if (n == 0) return;
    TKV_DISPATCH_REF(dt, add_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(static_cast<T*>(x), static_cast<const T*>(y), n));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_mul_ref(void* x, const void* y, DType dt, long n, cudaStream_t s) {
    if (n == 0) return;
    TKV_DISPATCH_REF(dt, mul_kernel<T><<<grid_for(n, 256), 256, 0, s>>>(static_cast<T*>(x), static_cast<const T*>(y), n));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_rope_ref(void* x, DType dt, const int64_t* positions, int n, int heads, int head_dim, const double* cos_d,
                     const double* sin_d, int table_pos, cudaStream_t s) {
    const long total = long(n) * heads * (head_dim / 2);
    if (total == 0) return;
    TKV_DISPATCH_REF(dt, rope_kernel<T><<<grid_for(total, 256), 256, 0, s>>>(
                             static_cast<T*>(x), positions, n, heads, head_dim, cos_d, sin_d, table_pos));
    TKV_CUDA_CHECK(cudaGetLastError());
}

void launch_attend_ref(const void* q, const void* k_own, const void* v_own, const void* k_ctx, const void* v_ctx,
                       const int32_t* group, const AttnSeq* seqs, int n_seqs, int total_q, void* out, DType dt,
                       int num_heads, int kv_heads, int head_dim, int mode, cudaStream_t s, const AttnSeq* seqs_host) {
    if (total_q == 0) return;
    // scratch for one score row per (row, head): bounded by the longest combined key range, taken
    // from the host copy of the sequence table (read back from the device only without one)
    int max_keys = 0;
    if (seqs_host) {
        for (int i = 0; i < n_seqs; ++i) max_keys = std::max(max_keys, seqs_host[i].n_ctx + seqs_host[i].n_own);
    } else {
        std::vector<AttnSeq> hs(static_cast<size_t>(n_seqs));
        TKV_CUDA_CHECK(cudaMemcpyAsync(hs.data(), seqs, sizeof(AttnSeq) * n_seqs, cudaMemcpyDeviceToHost, s));
        TKV_CUDA_CHECK(cudaStreamSynchronize(s));
        for (const auto& h : hs) max_keys = std::max(max_keys, h.n_ctx + h.n_own);
    }
    double* scratch = nullptr;
    const size_t bytes = size_t(total_q) * num_heads * std::max(1, max_keys) * sizeof(double);
    TKV_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes, s));
    const long n = long(total_q) * num_heads;
    TKV_DISPATCH_REF(dt, attend_kernel<T><<<grid_for(n, 64), 64, 0, s>>>(
                             static_cast<const T*>(q), static_cast<const T*>(k_own), static_cast<const T*>(v_own),
                             static_cast<const T*>(k_ctx), static_cast<const T*>(v_ctx), group, seqs, n_seqs, total_q,
                             static_cast<T*>(out), num_heads, kv_heads, head_dim, mode, scratch, std::max(1, max_keys)));
    TKV_CUDA_CHECK(cudaGetLastError());
    TKV_CUDA_CHECK(cudaFreeAsync(scratch, s));
}

}  // namespace tkv
