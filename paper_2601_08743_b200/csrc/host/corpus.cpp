// Host corpus layer: error names, schema graph / topological order / encoding groups,
// corpus JSON IO, table serialization and the word/byte tokenizer.
// Semantics follow proj/src/{errors,schema,serialize,tokenizer}.cpp; implementation is new.
#include <algorithm>
#include <fstream>
#include <numeric>
#include <queue>
#include <set>
#include <sstream>

#include <json.hpp>

#include "tablekv/errors.hpp"
#include "tablekv/schema.hpp"
#include "tablekv/serialize.hpp"
#include "tablekv/tokenizer.hpp"

namespace tablekv {

// ------------------------------------------------------------------ errors (errors.cpp:5-27)
const char* errc_name(Errc c) {
    static const char* const names[] = {
        "DanglingForeignKey", "CycleDetected",   "DuplicateTable",      "EmptySerialization", "DuplicateSerialization",
        "UnknownTable",       "CacheNotFull",    "TableIdOutOfRange",   "LengthMismatch",     "DimensionMismatch",
        "EmptyGroup",         "MissingTableKV",  "GroupOrderViolation", "EmptyBatch",         "MissingCacheDir",
        "VerifyFailed",       "BadConfig",       "IoError"};
    const size_t i = size_t(c);
    return i < sizeof(names) / sizeof(names[0]) ? names[i] : "UnknownError";
}

// ------------------------------------------------------------------ graph (schema.cpp:53-226)
bool SchemaGraph::has_edge(int from, int to) const {
    if (from < 0 || from >= node_count) return false;
    const auto& e = out_edges[size_t(from)];
    return std::binary_search(e.begin(), e.end(), to);
}

size_t SchemaGraph::edge_count() const {
    size_t n = 0;
    for (const auto& e : out_edges) n += e.size();
    return n;
}

void validate_corpus(const std::vector<TableSchema>& schemas) {
    const int m = int(schemas.size());
    std::vector<bool> present(size_t(m), false);
    for (const auto& t : schemas) {
        if (t.table_id < 0 || t.table_id >= m || present[size_t(t.table_id)])
            throw Error(Errc::bad_config, "table_ids must be dense and unique in 0.." + std::to_string(m - 1) + " (got " +
                                              std::to_string(t.table_id) + ")");
        present[size_t(t.table_id)] = true;
        std::set<std::string> cols;
        for (const auto& c : t.columns) {
            if (c.name.empty()) throw Error(Errc::bad_config, "empty column name in table " + t.name);
            cols.insert(c.name);
        }
        for (const auto& fk : t.foreign_keys) {
            if (fk.ref_table < 0 || fk.ref_table >= m)
                throw Error(Errc::dangling_foreign_key,
                            "table " + t.name + " references unknown table_id " + std::to_string(fk.ref_table));
            if (!cols.count(fk.column))
                throw Error(Errc::dangling_foreign_key, "table " + t.name + " has no local column " + fk.column);
        }
    }
}

SchemaGraph build_graph(const std::vector<TableSchema>& schemas) {
    validate_corpus(schemas);
    SchemaGraph g;
    g.node_count = int(schemas.size());
    g.out_edges.resize(size_t(g.node_count));
    g.in_degree.assign(size_t(g.node_count), 0);
    for (const auto& t : schemas)
        for (const auto& fk : t.foreign_keys)
            if (fk.ref_table != t.table_id) g.out_edges[size_t(fk.ref_table)].push_back(t.table_id);
    for (auto& e : g.out_edges) {
        std::sort(e.begin(), e.end());
        e.erase(std::unique(e.begin(), e.end()), e.end());
        for (int v : e) ++g.in_degree[size_t(v)];
    }
    return g;
}

namespace {

// Kahn with a min-heap of ready nodes; returns the order and the leftover in-degrees.
std::vector<int> kahn_order(const std::vector<std::vector<int>>& adj, std::vector<int>& indeg) {
    const int n = int(adj.size());
    indeg.assign(size_t(n), 0);
    for (const auto& e : adj)
        for (int v : e) ++indeg[size_t(v)];
    std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
    for (int v = 0; v < n; ++v)
        if (indeg[size_t(v)] == 0) ready.push(v);
    std::vector<int> order;
    order.reserve(size_t(n));
    while (!ready.empty()) {
        const int v = ready.top();
        ready.pop();
        order.push_back(v);
        for (int w : adj[size_t(v)])
            if (--indeg[size_t(w)] == 0) ready.push(w);
    }
    return order;
}

// Walk from the lowest node left with in-degree > 0, following the first such successor,
// until a node repeats; the repeated suffix is a cycle (every leftover node leads into one).
std::vector<int> some_cycle(const SchemaGraph& g, const std::vector<int>& indeg) {
    int cur = -1;
    for (int v = 0; v < g.node_count && cur < 0; ++v)
        if (indeg[size_t(v)] > 0) cur = v;
    std::vector<int> seen_at(size_t(g.node_count), -1), path;
    while (seen_at[size_t(cur)] < 0) {
        seen_at[size_t(cur)] = int(path.size());
        path.push_back(cur);
        int nxt = -1;
        for (int w : g.out_edges[size_t(cur)])
            if (indeg[size_t(w)] > 0) {
                nxt = w;
                break;
            }
        cur = nxt;
    }
    return std::vector<int>(path.begin() + seen_at[size_t(cur)], path.end());
}

// Back edges in iterative-DFS discovery order (roots and children ascending).
std::vector<std::pair<int, int>> dfs_back_edges(const std::vector<std::vector<int>>& adj) {
    const int n = int(adj.size());
    std::vector<char> color(size_t(n), 0);  // 0 white, 1 grey, 2 black
    std::vector<std::pair<int, int>> back;
    std::vector<std::pair<int, size_t>> stack;
    for (int r = 0; r < n; ++r) {
        if (color[size_t(r)]) continue;
        color[size_t(r)] = 1;
        stack.assign(1, {r, 0});
        while (!stack.empty()) {
            auto& [u, i] = stack.back();
            if (i == adj[size_t(u)].size()) {
                color[size_t(u)] = 2;
                stack.pop_back();
                continue;
            }
            const int w = adj[size_t(u)][i++];
            if (color[size_t(w)] == 0) {
                color[size_t(w)] = 1;
                stack.push_back({w, 0});
            } else if (color[size_t(w)] == 1) {
                back.push_back({u, w});
            }
        }
    }
    return back;
}

}  // namespace

TopoResult topological_order(const SchemaGraph& graph, TopoMode mode) {
    TopoResult res;
    std::vector<int> indeg;
    if (mode == TopoMode::strict) {
        res.order = kahn_order(graph.out_edges, indeg);
        if (int(res.order.size()) != graph.node_count) {
            auto cyc = some_cycle(graph, indeg);
            throw CycleError(cyc, "schema graph contains a foreign-key cycle of " + std::to_string(cyc.size()) + " tables");
        }
        return res;
    }
    auto adj = graph.out_edges;
    for (;;) {
        const auto back = dfs_back_edges(adj);
        if (back.empty()) break;
        const auto [u, v] = back.back();  // drop the last-discovered back edge, retry
        auto& e = adj[size_t(u)];
        e.erase(std::find(e.begin(), e.end(), v));
        res.removed_edges.push_back({u, v});
    }
    res.order = kahn_order(adj, indeg);
    return res;
}

EncodingPlan encoding_groups(const SchemaGraph& graph, const std::vector<int>& order) {
    const int n = graph.node_count;
    std::vector<int> up(static_cast<size_t>(n));
    std::iota(up.begin(), up.end(), 0);
    auto root = [&](int x) {
        while (up[size_t(x)] != x) x = up[size_t(x)] = up[size_t(up[size_t(x)])];
        return x;
    };
    for (int u = 0; u < n; ++u)
        for (int v : graph.out_edges[size_t(u)]) up[size_t(root(u))] = root(v);
    EncodingPlan plan;
    plan.group_of.assign(size_t(n), -1);
    std::vector<int> gid(size_t(n), -1);
    for (int t : order) {
        const int r = root(t);
        if (gid[size_t(r)] < 0) {
            gid[size_t(r)] = int(plan.groups.size());
            plan.groups.emplace_back();
        }
        plan.group_of[size_t(t)] = gid[size_t(r)];
        plan.groups[size_t(gid[size_t(r)])].tables.push_back(t);
    }
    return plan;
}

void EncodingPlan::assign_offsets(const std::vector<int>& token_count_by_table) {
    for (auto& g : groups) {
        g.offsets.clear();
        int at = 0;
        for (int t : g.tables) {
            g.offsets.push_back(at);
            at += token_count_by_table.at(size_t(t));
        }
    }
}

// ------------------------------------------------------------------ corpus JSON (schema.cpp:230-314)
std::vector<TableSchema> parse_schema_corpus(const std::string& text) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw Error(Errc::io_error, std::string("schema corpus is not valid JSON: ") + e.what());
    }
    if (doc.is_object()) {
        if (doc.value("format_version", 0) != 1) throw Error(Errc::bad_config, "unsupported schema corpus format_version");
        if (!doc.contains("tables")) throw Error(Errc::bad_config, "schema corpus object lacks a tables array");
        doc = doc.at("tables");
    }
    if (!doc.is_array()) throw Error(Errc::bad_config, "schema corpus must be a JSON array of tables");
    std::vector<TableSchema> out;
    try {
        for (const auto& jt : doc) {
            TableSchema t;
            t.table_id = jt.at("table_id").get<int>();
            t.name = jt.at("name").get<std::string>();
            for (const auto& jc : jt.at("columns"))
                t.columns.push_back({jc.at("name").get<std::string>(), jc.value("description", std::string()),
                                     jc.value("is_primary_key", false)});
            if (jt.contains("foreign_keys"))
                for (const auto& jf : jt.at("foreign_keys"))
                    t.foreign_keys.push_back({jf.at("column").get<std::string>(), jf.at("ref_table").get<int>(),
                                              jf.at("ref_column").get<std::string>()});
            out.push_back(std::move(t));
        }
    } catch (const nlohmann::json::exception& e) {
        throw Error(Errc::bad_config, std::string("malformed table entry: ") + e.what());
    }
    std::sort(out.begin(), out.end(), [](const TableSchema& a, const TableSchema& b) { return a.table_id < b.table_id; });
    validate_corpus(out);
    return out;
}

std::vector<TableSchema> load_schema_corpus(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(Errc::io_error, "cannot open schema corpus: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_schema_corpus(ss.str());
}

std::string dump_schema_corpus(const std::vector<TableSchema>& schemas) {
    nlohmann::json tables = nlohmann::json::array();
    for (const auto& t : schemas) {
        nlohmann::json cols = nlohmann::json::array(), fks = nlohmann::json::array();
        for (const auto& c : t.columns)
            cols.push_back({{"name", c.name}, {"description", c.description}, {"is_primary_key", c.is_primary_key}});
        for (const auto& f : t.foreign_keys)
            fks.push_back({{"column", f.column}, {"ref_table", f.ref_table}, {"ref_column", f.ref_column}});
        tables.push_back({{"table_id", t.table_id}, {"name", t.name}, {"columns", cols}, {"foreign_keys", fks}});
    }
    nlohmann::json doc = {{"format_version", 1}, {"tables", tables}};
    return doc.dump(2) + "\n";
}

// ------------------------------------------------------------------ serialize (serialize.cpp:5-18)
std::string serialize_table(const TableSchema& schema) {
    std::string s;
    s.reserve(64 + 32 * schema.columns.size());
    s += "table ";
    s += schema.name;
    s += '\n';
    for (const auto& c : schema.columns) {
        s += "col ";
        s += c.name;
        if (!c.description.empty()) s += ": " + c.description;
        if (c.is_primary_key) s += " [pk]";
        for (const auto& fk : schema.foreign_keys)
            if (fk.column == c.name) s += " [fk #" + std::to_string(fk.ref_table) + "." + fk.ref_column + "]";
        s += '\n';
    }
    return s;
}

// ------------------------------------------------------------------ tokenizer (tokenizer.cpp:17-85)
namespace {
inline bool word_byte(unsigned char c) {
    return (c >= '0' && c <= '9') || (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_';
}

// visit(begin, end, is_word) for maximal word runs and single non-word bytes, in order
template <typename F>
void pieces(const std::string& s, F&& visit) {
    const size_t n = s.size();
    size_t i = 0;
    while (i < n) {
        if (!word_byte(static_cast<unsigned char>(s[i]))) {
            visit(i, i + 1, false);
            ++i;
            continue;
        }
        size_t j = i;
        while (j < n && word_byte(static_cast<unsigned char>(s[j]))) ++j;
        visit(i, j, true);
        i = j;
    }
}
}  // namespace

void Tokenizer::add_corpus_text(const std::string& text) {
    pieces(text, [&](size_t a, size_t b, bool word) {
        if (!word) return;  // only word runs (of any length) enter the vocabulary
        std::string w = text.substr(a, b - a);
        if (index_.count(w)) return;
        index_.emplace(w, TokenId(kByteVocab + int(vocab_.size())));
        vocab_.push_back(std::move(w));
    });
}

std::vector<TokenId> Tokenizer::encode(const std::string& text) const {
    std::vector<TokenId> ids;
    ids.reserve(text.size() / 2 + 1);
    pieces(text, [&](size_t a, size_t b, bool word) {
        if (word) {
            const auto it = index_.find(text.substr(a, b - a));
            if (it != index_.end()) {
                ids.push_back(it->second);
                return;
            }
        }
        for (size_t i = a; i < b; ++i) ids.push_back(TokenId(static_cast<unsigned char>(text[i])));
    });
    return ids;
}

std::string Tokenizer::decode(std::span<const TokenId> tokens) const {
    std::string out;
    for (TokenId t : tokens) {
        if (t >= 0 && t < kByteVocab)
            out.push_back(char(static_cast<unsigned char>(t)));
        else if (t >= kByteVocab && t < vocab_size())
            out += vocab_[size_t(t - kByteVocab)];
        else
            throw Error(Errc::bad_config, "token id " + std::to_string(t) + " outside vocabulary");
    }
    return out;
}

std::uint64_t Tokenizer::vocab_hash() const {
    // NB: the reference seeds with 1469598103934665603 (tokenizer.cpp:75), one digit short of the
    // textbook FNV offset basis; the manifest hash must match it, so we keep its constant.
    std::uint64_t h = 1469598103934665603ull;
    auto eat = [&h](unsigned char b) { h = (h ^ b) * 0x100000001b3ull; };
    for (const auto& w : vocab_) {
        for (unsigned char c : w) eat(c);
        eat(0xFF);
    }
    return h;
}

}  // namespace tablekv
