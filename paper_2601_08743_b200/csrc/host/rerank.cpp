// Query reranking (paper §4.2, Eq. 1-2): semantics of proj/src/rerank.cpp:16-94.
// Bitsets are packed row-major [n][words]; the greedy chain's inner argmin is sharded across
// host threads for big batches, reduced by (distance, slot) so the permutation is identical to
// the single-threaded scan for any thread count.
#include <algorithm>
#include <atomic>
#include <barrier>
#include <bit>
#include <thread>
#include <unordered_map>

#include "tablekv/rerank.hpp"
#include "tablekv/rng.hpp"

namespace tablekv {

int IncidenceVector::popcount() const {
    int c = 0;
    for (std::uint64_t w : words) c += std::popcount(w);
    return c;
}

IncidenceVector incidence(const std::vector<int>& table_ids, int n_bits) {
    IncidenceVector v;
    v.n_bits = n_bits;
    v.words.assign((size_t(n_bits) + 63) / 64, 0);
    for (int id : table_ids) {
        if (id < 0 || id >= n_bits)
            throw Error(Errc::table_id_out_of_range,
                        "table id " + std::to_string(id) + " not below " + std::to_string(n_bits));
        v.words[size_t(id) >> 6] |= std::uint64_t(1) << (id & 63);
    }
    return v;
}

std::uint64_t hamming(const IncidenceVector& a, const IncidenceVector& b) {
    if (a.n_bits != b.n_bits) throw Error(Errc::length_mismatch, "incidence vectors cover different table counts");
    std::uint64_t d = 0;
    for (size_t i = 0; i < a.words.size(); ++i) d += std::uint64_t(std::popcount(a.words[i] ^ b.words[i]));
    return d;
}

QueryRecord make_query_record(std::string query_id, std::vector<TokenId> tokens, std::vector<int> matched_tables,
                              int table_count, int query_token_count) {
    std::sort(matched_tables.begin(), matched_tables.end());
    matched_tables.erase(std::unique(matched_tables.begin(), matched_tables.end()), matched_tables.end());
    QueryRecord r;
    r.query_id = std::move(query_id);
    r.inc = incidence(matched_tables, table_count);
    r.tables = std::move(matched_tables);
    r.query_token_count = query_token_count >= 0 ? query_token_count : int(tokens.size());
    r.tokens = std::move(tokens);
    return r;
}

namespace {

struct Best {
    std::uint64_t d = ~std::uint64_t(0);
    size_t slot = ~size_t(0);
    bool better(const Best& o) const { return o.d < d || (o.d == d && o.slot < slot); }
};

}  // namespace

RerankClasses rerank_classes(const std::uint64_t* inc, size_t n, size_t words, std::uint64_t seed, AnchorMode mode) {
    if (n == 0) throw Error(Errc::empty_batch, "rerank needs at least one query");
    RerankClasses rc;
    std::unordered_multimap<std::uint64_t, size_t> by_hash;  // row hash -> class
    size_t live = 0, anchor_slot = 0;
    std::vector<size_t> class_of;
    for (size_t i = 0; i < n; ++i) {
        const std::uint64_t* r = inc + i * words;
        std::uint64_t h = 0x9E3779B97F4A7C15ull;
        bool any = false;
        for (size_t w = 0; w < words; ++w) {
            any |= r[w] != 0;
            h = (h ^ r[w]) * 0xBF58476D1CE4E5B9ull;
            h ^= h >> 31;
        }
        if (!any) {
            rc.empty.push_back(i);
            continue;
        }
        size_t c = rc.members.size();
        for (auto [it, end] = by_hash.equal_range(h); it != end; ++it)
            if (std::equal(r, r + words, rc.rows.begin() + long(it->second * words))) {
                c = it->second;
                break;
            }
        if (c == rc.members.size()) {
            by_hash.emplace(h, c);
            rc.rows.insert(rc.rows.end(), r, r + words);
            rc.members.emplace_back();
        }
        rc.members[c].push_back(i);
        class_of.push_back(c);
        ++live;
    }
    if (live) {
        if (mode == AnchorMode::seeded) {  // rerank.cpp:68-71: the anchor slot among the live queries
            SeededRng r(seed);
            anchor_slot = size_t(r.next_below(live));
        }
        rc.anchor_class = class_of[anchor_slot];
        size_t k = 0;  // the anchor's original index: the anchor_slot-th live query
        for (size_t i = 0, seen = 0; i < n; ++i) {
            bool any = false;
            for (size_t w = 0; w < words && !any; ++w) any = inc[i * words + w] != 0;
            if (any && seen++ == anchor_slot) {
                k = i;
                break;
            }
        }
        rc.anchor_query = k;
    }
    return rc;
}

std::vector<size_t> expand_class_chain(const RerankClasses& rc, const std::vector<size_t>& class_order) {
    std::vector<size_t> out;
    size_t total = rc.empty.size();
    for (const auto& m : rc.members) total += m.size();
    out.reserve(total);
    for (size_t c : class_order) {
        if (c == rc.anchor_class) {  // the anchor first, then its class-mates ascending
            out.push_back(rc.anchor_query);
            for (size_t q : rc.members[c])
                if (q != rc.anchor_query) out.push_back(q);
        } else {
            out.insert(out.end(), rc.members[c].begin(), rc.members[c].end());
        }
    }
    out.insert(out.end(), rc.empty.begin(), rc.empty.end());  // rerank.cpp:92
    return out;
}

namespace {

// the greedy chain over m packed rows from `first` (rerank.cpp:72-89), the argmin sharded over
// host threads for big batches and reduced by (distance, slot)
std::vector<size_t> chain_rows(const std::uint64_t* inc, size_t m, size_t words, size_t first, int threads) {
    std::vector<size_t> out;
    out.reserve(m);
    // candidates kept compacted in slot order: remaining[] holds unused slots ascending
    std::vector<size_t> remaining(m);
    for (size_t s = 0; s < m; ++s) remaining[s] = s;
    size_t cur = first;
    out.push_back(cur);
    remaining.erase(remaining.begin() + long(first));
    if (threads <= 0) threads = int(std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency())));
    if (m < 4096) threads = 1;
    std::vector<Best> part(static_cast<size_t>(threads));
    const std::uint64_t* a = nullptr;
    auto scan = [&](size_t lo, size_t hi, Best& b) {
        for (size_t k = lo; k < hi; ++k) {
            const std::uint64_t* c = inc + remaining[k] * words;
            std::uint64_t d = 0;
            for (size_t w = 0; w < words; ++w) d += std::uint64_t(std::popcount(a[w] ^ c[w]));
            if (d < b.d) b = {d, k};  // k ascending => first minimum = lowest slot
        }
    };
    auto chunk_of = [&](int t, size_t& lo, size_t& hi) {
        const size_t chunk = (remaining.size() + size_t(threads) - 1) / size_t(threads);
        lo = std::min(remaining.size(), size_t(t) * chunk);
        hi = std::min(remaining.size(), lo + chunk);
    };
    // persistent workers, two barrier phases per chain step (scan, then the reduction on this thread)
    std::barrier sync(threads);
    bool done = false;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (;;) {
                sync.arrive_and_wait();
                if (done) return;
                size_t lo, hi;
                chunk_of(t, lo, hi);
                part[size_t(t)] = Best{};
                scan(lo, hi, part[size_t(t)]);
                sync.arrive_and_wait();
            }
        });
    while (!remaining.empty()) {
        a = inc + cur * words;
        Best best;
        if (threads == 1) {
            scan(0, remaining.size(), best);
        } else {
            sync.arrive_and_wait();
            size_t lo, hi;
            chunk_of(0, lo, hi);
            part[0] = Best{};
            scan(lo, hi, part[0]);
            sync.arrive_and_wait();
            for (const Best& b : part)
                if (best.better(b)) best = b;
        }
        cur = remaining[best.slot];
        out.push_back(cur);
        remaining.erase(remaining.begin() + long(best.slot));
    }
    if (threads > 1) {
        done = true;
        sync.arrive_and_wait();
        for (auto& th : pool) th.join();
    }
    return out;
}

}  // namespace

std::vector<size_t> rerank_packed(const std::uint64_t* inc, size_t n, size_t words, std::uint64_t seed, AnchorMode mode,
                                  int threads) {
    const RerankClasses rc = rerank_classes(inc, n, words, seed, mode);
    if (rc.n_classes() == 0) return rc.empty;
    return expand_class_chain(rc, chain_rows(rc.rows.data(), rc.n_classes(), words, rc.anchor_class, threads));
}

std::vector<size_t> rerank(const std::vector<QueryRecord>& queries, std::uint64_t seed, AnchorMode mode) {
    if (queries.empty()) throw Error(Errc::empty_batch, "rerank needs at least one query");
    const size_t words = queries.front().inc.words.size();
    std::vector<std::uint64_t> packed(queries.size() * words, 0);
    for (size_t i = 0; i < queries.size(); ++i) {
        if (queries[i].inc.words.size() != words)
            throw Error(Errc::length_mismatch, "incidence vectors cover different table counts");
        // a query's table list decides emptiness (rerank.cpp:62); the bitset mirrors it
        if (queries[i].tables.empty()) continue;
        std::copy(queries[i].inc.words.begin(), queries[i].inc.words.end(), packed.begin() + long(i * words));
    }
    // queries with tables but an all-zero bitset cannot occur (incidence() sets a bit per id)
    return rerank_packed(packed.data(), queries.size(), words, seed, mode);
}

}  // namespace tablekv
