// tablekv B200 build — the non-template bridge from the C++ drop-in API (attention.hpp) to the
// CUDA model in libtkv.so. One device model per (ModelConfig, precision) is created lazily on the
// current device and reused; weights come from cfg.weight_seed (the reference's counter hash).
#pragma once

#include <cstdint>
#include <vector>

#include "tablekv/model.hpp"
#include "tablekv/table_kv.hpp"
#include "tablekv/types.hpp"

namespace tablekv::device {

// precision: 0 = Real float, 2 = Real double (reference-precision kernels, double accumulation)
struct Forward {
    const ModelConfig* cfg = nullptr;
    int precision = 0;
    const TokenId* tokens = nullptr;
    int n = 0;
    const int64_t* positions = nullptr;  // nullable: n_ctx + i
    const int* groups = nullptr;         // mode 1
    int mode = 0;                        // 0: own rows see all ctx rows + causal own; 1: block mask
    const void* ctx_k = nullptr;         // [L][n_ctx][kv_dim] Real, rotated
    const void* ctx_v = nullptr;
    int n_ctx = 0;
    void* hidden = nullptr;              // [n][hidden] Real
    void* kraw = nullptr;                // [L][n][kv_dim] Real (pre-rotation)
    void* krot = nullptr;                // [L][n][kv_dim] Real (rotated)
    void* v = nullptr;                   // [L][n][kv_dim] Real
};

void forward(const Forward& f);

// assemble() of f32 blocks on the GPU: blocks go through a pinned arena and pool pages, the
// gather kernel rotates K at cursor + t (bit-exact with the reference). Outputs [L][total][kv_dim].
void gather_f32(const ModelConfig& cfg, const std::vector<const TableKV<float>*>& tables, std::vector<std::vector<float>>& k,
                std::vector<std::vector<float>>& v);

// Throws BadConfig unless `probe` values equal the counter-hash weights of cfg (the device never
// takes host weights; it regenerates them).
void check_weights(const ModelConfig& cfg, const double* probe_embedding, const double* probe_wq, int n);

}  // namespace tablekv::device
