// Device weight init: bit-identical to ModelWeights<float>::fill
// (proj/include/tablekv/model.hpp:80-87): w[i] = float(signed_unit(mix3(seed, tag*131+layer, i)) * scale),
// then (bf16 mode) round-to-nearest-even to bf16. One thread per element, grid-stride.
#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace tkv {

namespace {

template <typename Out>
__global__ void fill_matrix_kernel(Out* __restrict__ dst, long rows, long cols, long dst_row0, uint64_t h0,
                                   double scale, int ib, int slot) {
    const long total = rows * cols;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < total; i += long(gridDim.x) * blockDim.x) {
        const uint64_t hv = splitmix64(h0 + uint64_t(i) * 0x9e3779b97f4a7c15ull);
        const float v = static_cast<float>(signed_unit(hv) * scale);
        const long r = i / cols, c = i - r * cols;
        const long dr = ib == 0 ? dst_row0 + r : dst_row0 + (r / ib) * 2 * ib + long(slot) * ib + (r % ib);
        if constexpr (sizeof(Out) == 2) {
            reinterpret_cast<uint16_t*>(dst)[dr * cols + c] = f32_to_bf16_bits(v);
        } else if constexpr (sizeof(Out) == 4) {
            dst[dr * cols + c] = v;
        } else {
            dst[dr * cols + c] = signed_unit(hv) * scale;  // Real = double: no float cast
        }
    }
}

}  // namespace

void launch_fill_matrix(void* dst, DType dt, long rows, long cols, long dst_row0, uint64_t seed, uint64_t tag_stream,
                        double scale, int interleave_block, int slot, cudaStream_t s) {
    const uint64_t h0 = mix3_prefix(seed, tag_stream);
    const long total = rows * cols;
    if (total == 0) return;
    const int threads = 256;
    const int blocks = int(std::min<long>((total + threads - 1) / threads, kNumSMs * 16L));
    switch (dt) {
        case DType::bf16:
            fill_matrix_kernel<uint16_t><<<blocks, threads, 0, s>>>(static_cast<uint16_t*>(dst), rows, cols, dst_row0,
                                                                    h0, scale, interleave_block, slot);
            break;
        case DType::f32:
            fill_matrix_kernel<float><<<blocks, threads, 0, s>>>(static_cast<float*>(dst), rows, cols, dst_row0, h0,
                                                                 scale, interleave_block, slot);
            break;
        case DType::f64:
            fill_matrix_kernel<double><<<blocks, threads, 0, s>>>(static_cast<double*>(dst), rows, cols, dst_row0, h0,
                                                                  scale, interleave_block, slot);
            break;
    }
    TKV_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tkv
