// tablekv B200 build — deterministic hashing / streams (drop-in for proj/include/tablekv/rng.hpp).
// Bit-for-bit the reference generator: the device weight-init kernel uses the same
// counter hash (paper_2601_08743_b200/csrc/cuda/common.cuh), so host and GPU agree.
#pragma once

#include <cstdint>

namespace tablekv {

namespace rng_detail {
constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr std::uint64_t scramble(std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
}  // namespace rng_detail

inline std::uint64_t splitmix64(std::uint64_t x) { return rng_detail::scramble(x + rng_detail::kGolden); }

// Counter-based: value depends only on (seed, tag, index), never on draw order.
inline std::uint64_t mix3(std::uint64_t seed, std::uint64_t tag, std::uint64_t index) {
    const std::uint64_t stream = splitmix64(splitmix64(seed ^ 0x243f6a8885a308d3ull) ^ splitmix64(tag));
    return splitmix64(stream + index * rng_detail::kGolden);
}

inline double u64_to_unit(std::uint64_t x) { return double(x >> 11) * 0x1.0p-53; }           // [0, 1)
inline double u64_to_signed_unit(std::uint64_t x) { return u64_to_unit(x) * 2.0 - 1.0; }    // [-1, 1)

class SeededRng {
   public:
    explicit SeededRng(std::uint64_t seed) : s_(splitmix64(seed ^ rng_detail::kGolden)) {}
    std::uint64_t next_u64() {
        s_ += rng_detail::kGolden;
        return rng_detail::scramble(s_);
    }
    std::uint64_t next_below(std::uint64_t n) { return n ? next_u64() % n : 0; }
    double next_unit() { return u64_to_unit(next_u64()); }

   private:
    std::uint64_t s_;
};

}  // namespace tablekv
