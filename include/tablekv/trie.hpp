// tablekv B200 build — Table Trie (drop-in for proj/include/tablekv/trie.hpp:14-64).
//
// Flat layout: every edge (parent node, token) -> child lives in ONE open-addressing hash
// table of 64-bit keys; nodes are plain indices with a terminal record. Lookups touch one
// cache line per step instead of chasing per-node hash maps. Matching semantics are the
// reference's Algorithm 1: from a start, keep the LAST terminal passed on the walk
// (trie.cpp:38-50); match_all jumps past a match and advances by one on a miss.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "tablekv/errors.hpp"
#include "tablekv/types.hpp"

namespace tablekv {

struct MatchSpan {
    int table_id = -1;
    size_t start = 0;
    size_t end = 0;  // exclusive
};

struct TrieQueryResult {
    bool found = false;
    size_t next = 0;
    int table_id = -1;
    CacheHandle handle = 0;
};

struct MatchStats {
    size_t node_visits = 0;
};

class TableTrie {
   public:
    TableTrie();
    TableTrie(TableTrie&&) noexcept = default;
    TableTrie& operator=(TableTrie&&) noexcept = default;

    void insert(std::span<const TokenId> tokens, int table_id, CacheHandle handle);
    TrieQueryResult query(std::span<const TokenId> tokens, size_t start, MatchStats* stats = nullptr) const;
    std::vector<MatchSpan> match_all(std::span<const TokenId> tokens, MatchStats* stats = nullptr) const;
    size_t table_count() const { return tables_; }
    size_t node_count() const { return term_id_.size(); }

   private:
    int32_t child(int32_t node, TokenId tok) const;
    int32_t child_or_add(int32_t node, TokenId tok);
    void grow();

    std::vector<std::uint64_t> keys_;   // (node << 32 | uint32 token) + 1, 0 = empty slot
    std::vector<int32_t> vals_;         // child node index
    size_t used_ = 0;
    std::vector<int32_t> term_id_;      // per node: table id or -1
    std::vector<CacheHandle> term_handle_;
    std::vector<int32_t> seen_ids_;     // inserted table ids (sorted)
    size_t tables_ = 0;
};

}  // namespace tablekv
