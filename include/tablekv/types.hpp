// tablekv B200 build — basic vocabulary types (drop-in for proj/include/tablekv/types.hpp).
#pragma once

#include <cstdint>

namespace tablekv {

using TokenId = std::int32_t;       // tokenizer output: bytes 0..255, corpus words 256+
using CacheHandle = std::uint64_t;  // opaque handle carried by trie terminals

}  // namespace tablekv
