// Table Trie over one flat open-addressing edge table (see include/tablekv/trie.hpp).
// Semantics: proj/src/trie.cpp:7-68 (insert errors, last-terminal-passed query, match_all).
#include <algorithm>

#include "tablekv/trie.hpp"

namespace tablekv {

namespace {
inline std::uint64_t edge_key(int32_t node, TokenId tok) {
    return ((std::uint64_t(std::uint32_t(node)) << 32) | std::uint32_t(tok)) + 1;  // never 0
}
inline size_t edge_hash(std::uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return size_t(k);
}
}  // namespace

TableTrie::TableTrie() : keys_(64, 0), vals_(64, -1), term_id_(1, -1), term_handle_(1, 0) {}

int32_t TableTrie::child(int32_t node, TokenId tok) const {
    const std::uint64_t k = edge_key(node, tok);
    const size_t mask = keys_.size() - 1;
    for (size_t i = edge_hash(k) & mask;; i = (i + 1) & mask) {
        if (keys_[i] == k) return vals_[i];
        if (keys_[i] == 0) return -1;
    }
}

void TableTrie::grow() {
    std::vector<std::uint64_t> ok;
    std::vector<int32_t> ov;
    ok.swap(keys_);
    ov.swap(vals_);
    keys_.assign(ok.size() * 2, 0);
    vals_.assign(ok.size() * 2, -1);
    const size_t mask = keys_.size() - 1;
    for (size_t j = 0; j < ok.size(); ++j) {
        if (!ok[j]) continue;
        size_t i = edge_hash(ok[j]) & mask;
        while (keys_[i]) i = (i + 1) & mask;
        keys_[i] = ok[j];
        vals_[i] = ov[j];
    }
}

int32_t TableTrie::child_or_add(int32_t node, TokenId tok) {
    if (2 * (used_ + 1) > keys_.size()) grow();  // load factor <= 1/2
    const std::uint64_t k = edge_key(node, tok);
    const size_t mask = keys_.size() - 1;
    size_t i = edge_hash(k) & mask;
    for (; keys_[i]; i = (i + 1) & mask)
        if (keys_[i] == k) return vals_[i];
    const int32_t fresh = int32_t(term_id_.size());
    term_id_.push_back(-1);
    term_handle_.push_back(0);
    keys_[i] = k;
    vals_[i] = fresh;
    ++used_;
    return fresh;
}

void TableTrie::insert(std::span<const TokenId> tokens, int table_id, CacheHandle handle) {
    if (tokens.empty())
        throw Error(Errc::empty_serialization, "table " + std::to_string(table_id) + " has an empty token serialization");
    const auto at = std::lower_bound(seen_ids_.begin(), seen_ids_.end(), table_id);
    if (at != seen_ids_.end() && *at == table_id)
        throw Error(Errc::duplicate_table, "table " + std::to_string(table_id) + " already inserted");
    int32_t node = 0;
    for (TokenId t : tokens) node = child_or_add(node, t);
    if (term_id_[size_t(node)] >= 0)
        throw Error(Errc::duplicate_serialization, "tables " + std::to_string(term_id_[size_t(node)]) + " and " +
                                                       std::to_string(table_id) + " share an identical serialization");
    term_id_[size_t(node)] = table_id;
    term_handle_[size_t(node)] = handle;
    seen_ids_.insert(std::lower_bound(seen_ids_.begin(), seen_ids_.end(), table_id), table_id);
    ++tables_;
}

TrieQueryResult TableTrie::query(std::span<const TokenId> tokens, size_t start, MatchStats* stats) const {
    TrieQueryResult r;
    int32_t node = 0;
    size_t steps = 0;
    for (size_t p = start; p < tokens.size(); ++p) {
        node = child(node, tokens[p]);
        if (node < 0) break;
        ++steps;
        if (term_id_[size_t(node)] >= 0) {  // remember the deepest terminal passed so far
            r.found = true;
            r.next = p + 1;
            r.table_id = term_id_[size_t(node)];
            r.handle = term_handle_[size_t(node)];
        }
    }
    if (stats) stats->node_visits += steps;
    return r;
}

std::vector<MatchSpan> TableTrie::match_all(std::span<const TokenId> tokens, MatchStats* stats) const {
    std::vector<MatchSpan> out;
    size_t p = 0;
    while (p < tokens.size()) {
        const TrieQueryResult q = query(tokens, p, stats);
        if (!q.found) {
            ++p;
            continue;
        }
        out.push_back({q.table_id, p, q.next});
        p = q.next;
    }
    return out;
}

}  // namespace tablekv
