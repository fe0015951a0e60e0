// Query reranking (paper §4.2, Eq. 1-2): semantics of proj/src/rerank.cpp:16-94.
// Bitsets are packed row-major [n][words]; the greedy chain's inner argmin is sharded across
// host threads for big batches, reduced by (distance, slot) so the permutation is identical to
// the single-threaded scan for any thread count.
#include <algorithm>
#include <atomic>
#include <barrier>
#include <bit>
#include <thread>

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

std::vector<size_t> rerank_packed(const std::uint64_t* inc, size_t n, size_t words, std::uint64_t seed, AnchorMode mode,
                                  int threads) {
    if (n == 0) throw Error(Errc::empty_batch, "rerank needs at least one query");
    std::vector<size_t> live, empty;
    for (size_t i = 0; i < n; ++i) {
        bool any = false;
        for (size_t w = 0; w < words && !any; ++w) any = inc[i * words + w] != 0;
        (any ? live : empty).push_back(i);
    }
    std::vector<size_t> out;
    out.reserve(n);
    if (!live.empty()) {
        const size_t m = live.size();
        // candidates kept compacted in slot order: remaining[] holds unused slots ascending
        std::vector<size_t> remaining(m);
        for (size_t s = 0; s < m; ++s) remaining[s] = s;
        size_t first = 0;
        if (mode == AnchorMode::seeded) {
            SeededRng r(seed);
            first = size_t(r.next_below(m));
        }
        size_t cur = live[first];
        out.push_back(cur);
        remaining.erase(remaining.begin() + long(first));
        if (threads <= 0) threads = int(std::min<unsigned>(8, std::max(1u, std::thread::hardware_concurrency())));
        if (m < 4096) threads = 1;
        std::vector<Best> part(static_cast<size_t>(threads));
        const std::uint64_t* a = nullptr;
        auto scan = [&](size_t lo, size_t hi, Best& b) {
            for (size_t k = lo; k < hi; ++k) {
                const std::uint64_t* c = inc + live[remaining[k]] * words;
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
            cur = live[remaining[best.slot]];
            out.push_back(cur);
            remaining.erase(remaining.begin() + long(best.slot));
        }
        if (threads > 1) {
            done = true;
            sync.arrive_and_wait();
            for (auto& th : pool) th.join();
        }
    }
    out.insert(out.end(), empty.begin(), empty.end());
    return out;
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
