"""TableCache CPU oracle — TEST INFRASTRUCTURE ONLY.

A self-contained restatement of the reference algorithms on the online path
(/root/reference/proj, cited file:line throughout), used only by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline leg, as the CHECKER. The product
(paper_2601_08743_b200 + its CUDA library) never imports this module.

Pinned against the reference itself: tests/test_oracle.py checks every function here
against tests/golden/*, which oracle/_ref/golden_dump produced by running the unchanged
reference library (see tests/golden/make_goldens.py).

Host algorithms are plain Python (small cases); the model is numpy float64 with an
explicit storage-rounding policy:
  * storage="f32"  — the reference's own arithmetic (double accumulation, f32 storage),
  * storage="bf16" — the same algorithm rounding every stored activation/weight to bf16
    at the points the CUDA bf16 path stores them (used for the bf16 kernels' tolerance).
The model config extends the reference (G2/G3 in SURVEY.md): num_kv_heads (GQA),
ffn_dim, mlp in {silu, swiglu}, norm in {ln, rms}, and a documented head
(final LN/RMS + untied mix3 head, tag 8).
"""
from __future__ import annotations

import bisect
import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# ============================================================================ rng
# rng.hpp:9-53


def splitmix64(x):
    x = (x + GOLDEN) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix3(seed, tag, index):
    h = splitmix64((seed ^ 0x243F6A8885A308D3) & M64)
    h = splitmix64(h ^ splitmix64(tag & M64))
    return splitmix64((h + index * GOLDEN) & M64)


def u64_to_signed_unit(x):
    return float(x >> 11) * 2.0 ** -53 * 2.0 - 1.0


class SeededRng:
    def __init__(self, seed):
        self.state = splitmix64((seed ^ GOLDEN) & M64)

    def next_u64(self):
        self.state = (self.state + GOLDEN) & M64
        x = self.state
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
        return x ^ (x >> 31)

    def next_below(self, n):
        return 0 if n == 0 else self.next_u64() % n


def _np_splitmix(x):
    x = x + np.uint64(GOLDEN)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def mix3_unit_array(seed, tag, start, count):
    """Vectorised u64_to_signed_unit(mix3(seed, tag, i)) for i in [start, start+count)."""
    h = mix3(seed, tag, 0)  # h for index 0 = splitmix(h0); rebuild h0 below
    h0 = splitmix64((seed ^ 0x243F6A8885A308D3) & M64)
    h0 = splitmix64(h0 ^ splitmix64(tag & M64))
    with np.errstate(over="ignore"):
        idx = np.arange(start, start + count, dtype=np.uint64)
        x = _np_splitmix(np.uint64(h0) + idx * np.uint64(GOLDEN))
    del h
    return (x >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0


# ============================================================================ rounding


def round_bf16(x):
    """f64/f32 -> nearest bf16 (RNE through f32), returned as float64."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def round_f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def _identity(x):
    return np.asarray(x, dtype=np.float64)


def storage_round(storage):
    """bf16: the CUDA bf16 path; f32: the reference (Real=float); f64: the reference (Real=double)."""
    return {"bf16": round_bf16, "f32": round_f32, "f64": _identity}[storage]


def _ref_storage(storage):
    return storage in ("f32", "f64")


# ============================================================================ tokenizer
# tokenizer.cpp:17-85


def _is_word(c):
    return ("a" <= c <= "z") or ("A" <= c <= "Z") or ("0" <= c <= "9") or c == "_"


def _split(text):
    i, n = 0, len(text)
    while i < n:
        if _is_word(text[i]):
            j = i + 1
            while j < n and _is_word(text[j]):
                j += 1
            yield i, j
            i = j
        else:
            yield i, i + 1
            i += 1


class Tokenizer:
    BYTE_VOCAB = 256

    def __init__(self):
        self.word_ids, self.words = {}, []

    def add_corpus_text(self, text):  # :34-42 single non-word bytes are skipped
        for a, b in _split(text):
            if b - a < 2 and not _is_word(text[a]):
                continue
            w = text[a:b]
            if w not in self.word_ids:
                self.word_ids[w] = 256 + len(self.words)
                self.words.append(w)

    def encode(self, text):  # :44-58
        out = []
        for a, b in _split(text):
            if _is_word(text[a]) and text[a:b] in self.word_ids:
                out.append(self.word_ids[text[a:b]])
            else:
                out.extend(text[a:b].encode("utf-8"))
        return out

    def vocab_size(self):
        return 256 + len(self.words)

    def vocab_hash(self):  # :74-85 FNV-1a over words, 0xFF separators
        h = 1469598103934665603
        for w in self.words:
            for byte in w.encode("utf-8") + b"\xff":
                h = ((h ^ byte) * 1099511628211) & M64
        return h


def serialize_table(t):  # serialize.cpp:5-18
    out = "table " + t["name"] + "\n"
    for c in t["columns"]:
        out += "col " + c["name"]
        if c.get("description"):
            out += ": " + c["description"]
        if c.get("is_primary_key"):
            out += " [pk]"
        for fk in t.get("foreign_keys", []):
            if fk["column"] == c["name"]:
                out += " [fk #%d.%s]" % (fk["ref_table"], fk["ref_column"])
        out += "\n"
    return out


# ============================================================================ schema
# schema.cpp:53-226


def build_graph(tables):
    n = len(tables)
    pairs = set()
    for t in tables:
        for fk in t.get("foreign_keys", []):
            if fk["ref_table"] != t["table_id"]:
                pairs.add((fk["ref_table"], t["table_id"]))
    out = [[] for _ in range(n)]
    for a, b in sorted(pairs):
        out[a].append(b)
    return [sorted(v) for v in out]


def kahn(out_edges):  # :107-128 min-id ready queue
    import heapq
    n = len(out_edges)
    deg = [0] * n
    for u in range(n):
        for v in out_edges[u]:
            deg[v] += 1
    ready = [v for v in range(n) if deg[v] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        v = heapq.heappop(ready)
        order.append(v)
        for w in out_edges[v]:
            deg[w] -= 1
            if deg[w] == 0:
                heapq.heappush(ready, w)
    return order, len(order) == n


def encoding_groups(out_edges, order):  # :187-215 union-find components, first appearance
    n = len(out_edges)
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for u in range(n):
        for v in out_edges[u]:
            parent[find(u)] = find(v)
    groups, group_of, root_to_group = [], [-1] * n, {}
    for tid in order:
        r = find(tid)
        if r not in root_to_group:
            root_to_group[r] = len(groups)
            groups.append([])
        group_of[tid] = root_to_group[r]
        groups[root_to_group[r]].append(tid)
    return groups, group_of


@dataclass
class EnginePlan:
    table_tokens: list
    groups: list
    group_of: list
    local_offset: list
    tokenizer: Tokenizer
    trie: "Trie"


def build_engine(tables):  # engine.cpp:16-52
    edges = build_graph(tables)
    order, ok = kahn(edges)
    if not ok:
        raise ValueError("cycle")
    groups, group_of = encoding_groups(edges, order)
    tok = Tokenizer()
    ser = [serialize_table(t) for t in sorted(tables, key=lambda t: t["table_id"])]
    for s in ser:
        tok.add_corpus_text(s)
    table_tokens = [tok.encode(s) for s in ser]
    local = [0] * len(tables)
    for g in groups:
        off = 0
        for tid in g:
            local[tid] = off
            off += len(table_tokens[tid])
    trie = Trie()
    for i, t in enumerate(table_tokens):
        trie.insert(t, i)
    return EnginePlan(table_tokens, groups, group_of, local, tok, trie)


# ============================================================================ trie
# trie.cpp:7-68


class Trie:
    def __init__(self):
        self.root = {}

    def insert(self, tokens, table_id):
        node = self.root
        for t in tokens:
            node = node.setdefault(t, {})
        if "$" in node:
            raise ValueError("duplicate serialization")
        node["$"] = table_id

    def query(self, tokens, start):
        """Longest terminal passed on the walk from `start` (trie.cpp:38-50)."""
        found, nxt, tid = False, 0, -1
        node, pos = self.root, start
        while pos < len(tokens) and tokens[pos] in node:
            node = node[tokens[pos]]
            pos += 1
            if "$" in node:
                found, nxt, tid = True, pos, node["$"]
        return found, nxt, tid

    def match_all(self, tokens):
        spans, p = [], 0
        while p < len(tokens):
            found, nxt, tid = self.query(tokens, p)
            if found:
                spans.append((tid, p, nxt))
                p = nxt
            else:
                p += 1
        return spans


def analyze_query(plan: EnginePlan, text):  # engine.cpp:133-151
    tokens = plan.tokenizer.encode(text)
    spans = plan.trie.match_all(tokens)
    seen, match_order, remainder, cursor = set(), [], [], 0
    for tid, s, e in spans:
        if tid not in seen:
            seen.add(tid)
            match_order.append(tid)
        remainder.extend(tokens[cursor:s])
        cursor = e
    remainder.extend(tokens[cursor:])
    return tokens, spans, match_order, remainder


def assembly_order(plan: EnginePlan, match_order):  # engine.cpp:153-172
    seq, members = [], {}
    for tid in match_order:
        g = plan.group_of[tid]
        if g not in members:
            members[g] = []
            seq.append(g)
        members[g].append(tid)
    out = []
    for g in seq:
        out.extend(sorted(members[g], key=lambda t: plan.local_offset[t]))
    return out


# ============================================================================ rerank
# rerank.cpp:16-94


def incidence(tables, n_bits):
    words = [0] * ((n_bits + 63) // 64)
    for t in tables:
        if t < 0 or t >= n_bits:
            raise ValueError("table id out of range")
        words[t >> 6] |= 1 << (t & 63)
    return words


def hamming(a, b):
    return sum(bin(x ^ y).count("1") for x, y in zip(a, b))


def rerank(table_sets, n_bits, seed, mode="seeded"):
    """Greedy nearest-neighbour chain; strict < keeps the lowest slot; empties last."""
    if not table_sets:
        raise ValueError("empty batch")
    incs = [incidence(sorted(set(t)), n_bits) for t in table_sets]
    active = [i for i, t in enumerate(table_sets) if t]
    empties = [i for i, t in enumerate(table_sets) if not t]
    out = []
    if active:
        slot = SeededRng(seed).next_below(len(active)) if mode == "seeded" else 0
        used = [False] * len(active)
        cur = active[slot]
        used[slot] = True
        out.append(cur)
        for _ in range(1, len(active)):
            best, best_slot = None, None
            for s, q in enumerate(active):
                if used[s]:
                    continue
                d = hamming(incs[cur], incs[q])
                if best is None or d < best:
                    best, best_slot = d, s
            used[best_slot] = True
            cur = active[best_slot]
            out.append(cur)
    return out + empties


# ============================================================================ cache
# tiered_cache.cpp:61-155 (transcribed from the semantics; entry-count capacity)


class Cache:
    def __init__(self, capacity, policy, token_counts):
        self.cap, self.policy, self.tokens = capacity, policy, token_counts
        self.order = []  # LRU: [0] most recent; FIFO: [0] oldest
        self.freq, self.stamp = {}, {}
        self.clock = 0
        self.hits = self.misses = self.swaps = self.prefetch_loads = 0
        self.loads = []  # slow-tier load log (table ids in order)

    def resident(self, t):
        return t in self.freq

    def size(self):
        return len(self.freq)

    def _touch(self, t):
        if self.policy == "lru":
            self.order.remove(t)
            self.order.insert(0, t)
        elif self.policy == "lfu":
            self.freq[t] += 1
            self.stamp[t] = self.clock

    def evict_candidate(self):
        if self.cap == 0 or len(self.freq) < self.cap:
            raise ValueError("cache not full")
        if self.policy == "lru":
            return self.order[-1]
        if self.policy == "fifo":
            return self.order[0]
        return min(self.freq, key=lambda t: (self.freq[t], self.stamp[t]))

    def _admit(self, t):
        ev = -1
        if len(self.freq) == self.cap:
            ev = self.evict_candidate()
            if self.policy != "lfu":
                self.order.remove(ev)
            del self.freq[ev], self.stamp[ev]
            self.swaps += 1
        self.freq[t], self.stamp[t] = 1, self.clock
        if self.policy == "lru":
            self.order.insert(0, t)
        elif self.policy == "fifo":
            self.order.append(t)
        return ev

    def get(self, t):
        self.clock += 1
        if t in self.freq:
            self._touch(t)
            self.hits += 1
            return True, -1
        self.loads.append(t)
        self.misses += 1
        if self.cap == 0:
            return False, -1
        return False, self._admit(t)

    def prefetch(self, ids):
        admitted = []
        if self.cap == 0:
            return admitted
        for t in ids:
            self.clock += 1
            if t in self.freq:
                self._touch(t)
                continue
            self.loads.append(t)
            self.prefetch_loads += 1
            self._admit(t)
            admitted.append(t)
        return admitted

    def residents(self):
        return sorted(self.freq)

    def counters(self):
        return [self.hits, self.misses, self.swaps, self.prefetch_loads]


# ============================================================================ pipeline
# pipeline.cpp:44-116 (build_trace), 147-174 (schedule), 176-308 (simulate)


def _distinct(seq):
    seen, out = set(), []
    for t in seq:
        if t not in seen:
            seen.add(t)
            out.append(t)
    return out


def schedule(queries, b_c, b_m):
    """queries: list of (qid, tables_in_assembly_order, query_tokens)."""
    n = len(queries)
    last_use = {}
    for i, q in enumerate(queries):
        for t in q[1]:
            last_use[t] = i
    windows = []
    for b in range(0, n, b_c):
        e = min(n, b + b_c)
        demand = _distinct(t for q in queries[b:e] for t in q[1])
        pref = _distinct(t for q in queries[e:min(n, e + b_m)] for t in q[1])
        windows.append({"begin": b, "end": e, "demand": demand, "prefetch": pref})
    return {"queries": queries, "windows": windows, "last_use": last_use}


def build_trace(plan, cost, cache: Cache):
    cpt, lpt, sw = cost
    managed = cache.cap > 0
    tokens = {}
    pending = []
    windows, compute = [], [0.0] * len(plan["queries"])

    def lc(tok, swapped):
        return lpt * tok + (sw if swapped else 0.0)

    for w in plan["windows"]:
        wt = {"boundary": [], "prefetch": [], "emergency": [[] for _ in range(w["end"] - w["begin"])]}
        dset = set(w["demand"])
        if managed:
            for t in w["demand"]:
                hit, ev = cache.get(t)
                tokens[t] = cache.tokens[t]
                wt["boundary"].append((t, not hit, ev, 0.0 if hit else lc(cache.tokens[t], ev >= 0)))
            cands = _distinct(pending + w["prefetch"])
            pending = []
            for t in cands:
                lu = plan["last_use"].get(t)
                if lu is None or lu < w["begin"]:
                    continue
                if cache.resident(t):
                    cache.prefetch([t])
                    continue
                victim = -1
                if cache.size() == cache.cap:
                    victim = cache.evict_candidate()
                    if victim in dset:
                        pending.append(t)
                        continue
                cache.prefetch([t])
                tokens[t] = cache.tokens[t]
                wt["prefetch"].append((t, True, victim, lc(cache.tokens[t], victim >= 0)))
        for qi in range(w["begin"], w["end"]):
            q = plan["queries"][qi]
            em = wt["emergency"][qi - w["begin"]]
            for t in q[1]:
                if managed and cache.resident(t):
                    continue
                hit, ev = cache.get(t)
                tokens[t] = cache.tokens[t]
                em.append((t, True, ev, lc(cache.tokens[t], ev >= 0)))
            ctx = float(sum(tokens[t] for t in q[1]))
            compute[qi] = cpt * (ctx * q[2] + q[2] * q[2] / 2.0)
        windows.append(wt)
    return windows, compute


def simulate(plan, cost, cache: Cache, mode):
    """Two-timeline virtual clock (pipeline.cpp:176-308). Returns dict like SimReport."""
    INF = math.inf
    managed = cache.cap > 0
    windows, compute = build_trace(plan, cost, cache)
    d_clock, d_total, busy = 0.0, 0.0, []

    def dsched(issue, size):
        nonlocal d_clock, d_total
        start = max(issue, d_clock)
        d_clock = start + size
        if size > 0:
            busy.append((start, d_clock))
        d_total += size
        return d_clock

    jobs, ready, pending_job = [], {}, {}
    cc = 0.0
    st = {"next": 0, "busy": 0, "cursor": 0.0}

    def evaluate_through(target):
        while st["next"] <= target:
            j = jobs[st["next"]]
            cur = max(st["cursor"], j["issue"])
            rem = j["size"]
            while rem > 0:
                if cur >= j["cancel"]:
                    break
                s = e = INF
                if st["busy"] < len(busy):
                    s, e = busy[st["busy"]]
                if e <= cur:
                    st["busy"] += 1
                    continue
                if s > cur:
                    take = min(rem, min(s, j["cancel"]) - cur)
                    j["wire"] += take
                    rem -= take
                    cur += take
                    continue
                if j["cancel"] <= e:
                    cur = j["cancel"]
                    break
                cur = e
                st["busy"] += 1
            j["end"] = min(cur, j["cancel"])
            j["evaluated"] = True
            st["cursor"] = max(st["cursor"], cur)
            st["next"] += 1

    def evict_note(victim, when):
        if victim < 0:
            return
        ready.pop(victim, None)
        if victim in pending_job:
            j = jobs[pending_job.pop(victim)]
            if not j["evaluated"]:
                j["cancel"] = min(j["cancel"], when)

    rep = {"query_ids": [], "ttft": [], "total_compute": 0.0}
    for wi, w in enumerate(plan["windows"]):
        wt = windows[wi]
        boundary = cc
        for (t, miss, ev, size) in wt["boundary"]:
            if not miss:
                continue
            evict_note(ev, boundary)
            ready[t] = dsched(boundary, size)
        if mode == "overlapped":
            for (t, miss, ev, size) in wt["prefetch"]:
                evict_note(ev, boundary)
                jobs.append({"table": t, "size": size, "issue": boundary, "cancel": INF, "end": 0.0,
                             "wire": 0.0, "evaluated": False})
                pending_job[t] = len(jobs) - 1
        else:
            for (t, miss, ev, size) in wt["prefetch"]:
                evict_note(ev, boundary)
                ready[t] = dsched(boundary, size)
            cc = max(cc, d_clock)
        for qi in range(w["begin"], w["end"]):
            q = plan["queries"][qi]
            for (t, miss, ev, size) in wt["emergency"][qi - w["begin"]]:
                issue = cc if mode == "serial" else (cc if managed else boundary)
                evict_note(ev, issue)
                ready[t] = dsched(issue, size)
            ready_q = 0.0
            for t in q[1]:
                if t in pending_job:
                    idx = pending_job.pop(t)
                    evaluate_through(idx)
                    ready[t] = jobs[idx]["end"]
                if t in ready:
                    ready_q = max(ready_q, ready[t])
            start = max(cc, ready_q)
            cc = start + compute[qi]
            rep["total_compute"] += compute[qi]
            rep["query_ids"].append(q[0])
            rep["ttft"].append(cc)
    if jobs:
        evaluate_through(len(jobs) - 1)
    rep["total_ttft"] = sum(rep["ttft"])
    rep["makespan"] = cc
    rep["total_transfer"] = d_total + sum(j["wire"] for j in jobs)
    rep["hits"], rep["misses"], rep["swaps"], rep["prefetch_loads"] = cache.counters()
    return rep


def run_batch(records, token_counts, n_bits, opts, cost):
    """records: list of (qid, tables_in_assembly_order, query_tokens). pipeline.cpp:310-342."""
    if opts.get("rerank_on", True):
        order = rerank([r[1] for r in records], n_bits, opts.get("seed", 1), opts.get("anchor", "seeded"))
    else:
        order = list(range(len(records)))
    plan = schedule([records[i] for i in order], opts["b_c"], opts["b_m"])
    mode = "overlapped" if opts.get("pipeline_on", True) else "serial"
    rep = simulate(plan, cost, Cache(opts["capacity"], opts["policy"], token_counts), mode)
    if mode == "overlapped":
        base = simulate(plan, cost, Cache(opts["capacity"], opts["policy"], token_counts), "serial")
        rep["serial_baseline_ttft"] = base["total_ttft"]
    else:
        rep["serial_baseline_ttft"] = rep["total_ttft"]
    rep["order"] = order
    return rep


# ============================================================================ model
# model.hpp:15-87, attention.hpp:84-414, rotary.hpp:21-59


@dataclass
class ModelConfig:
    num_layers: int = 2
    num_heads: int = 4
    head_dim: int = 16
    vocab_size: int = 0
    rotary_base: float = 10000.0
    weight_seed: int = 1
    num_kv_heads: int = 0  # 0 => num_heads (MHA, reference)
    ffn_dim: int = 0  # 0 => 4*hidden (reference)
    mlp: str = "silu"  # "silu" (reference, W_out(silu(W_in x))) | "swiglu" (W_out(silu(W_gate x) * W_in x))
    norm: str = "ln"  # "ln" (reference LayerNorm, no affine) | "rms"
    eps: float = 1e-5

    @property
    def hidden(self):
        return self.num_heads * self.head_dim

    @property
    def kv_heads(self):
        return self.num_kv_heads or self.num_heads

    @property
    def ffn(self):
        return self.ffn_dim or 4 * self.hidden

    @property
    def kv_dim(self):
        return self.kv_heads * self.head_dim


TAG = {"embedding": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "ffn_in": 6, "ffn_out": 7, "head": 8, "ffn_gate": 9}


def weight(cfg: ModelConfig, name, layer, rows, cols, storage="f32", row_start=0, row_count=None):
    """model.hpp:80-87: u64_to_signed_unit(mix3(seed, tag*131+layer, i)) * scale, cast to float."""
    h, f = cfg.hidden, cfg.ffn
    scale = {"embedding": 0.5, "ffn_out": 1.0 / math.sqrt(f)}.get(name, 1.0 / math.sqrt(h))
    rc = rows if row_count is None else row_count
    u = mix3_unit_array(cfg.weight_seed, TAG[name] * 131 + layer, row_start * cols, rc * cols)
    w = u * scale
    if storage != "f64":
        w = np.asarray(w, dtype=np.float32).astype(np.float64)  # static_cast<float>(double)
    if storage == "bf16":
        w = round_bf16(w)
    return w.reshape(rc, cols)


class Weights:
    """Lazily materialised weights (embedding rows on demand)."""

    def __init__(self, cfg: ModelConfig, storage="f32"):
        self.cfg, self.storage = cfg, storage
        h, kv, f = cfg.hidden, cfg.kv_dim, cfg.ffn
        self.layers = []
        for l in range(cfg.num_layers):
            L = {"wq": weight(cfg, "wq", l, h, h, storage), "wk": weight(cfg, "wk", l, kv, h, storage),
                 "wv": weight(cfg, "wv", l, kv, h, storage), "wo": weight(cfg, "wo", l, h, h, storage),
                 "ffn_in": weight(cfg, "ffn_in", l, f, h, storage), "ffn_out": weight(cfg, "ffn_out", l, h, f, storage)}
            if cfg.mlp == "swiglu":
                L["ffn_gate"] = weight(cfg, "ffn_gate", l, f, h, storage)
            self.layers.append(L)
        self._emb = {}
        self._head = None

    def embed(self, tokens):
        cfg = self.cfg
        out = np.empty((len(tokens), cfg.hidden))
        for i, t in enumerate(tokens):
            if t < 0 or t >= cfg.vocab_size:
                raise ValueError("token id %d outside vocabulary" % t)
            if t not in self._emb:
                self._emb[t] = weight(cfg, "embedding", 0, cfg.vocab_size, cfg.hidden, self.storage, row_start=t, row_count=1)[0]
            out[i] = self._emb[t]
        return out

    def head(self):
        if self._head is None:
            self._head = weight(self.cfg, "head", 0, self.cfg.vocab_size, self.cfg.hidden, self.storage)
        return self._head


def inv_freq(cfg):
    d = cfg.head_dim
    return np.array([cfg.rotary_base ** (-2.0 * k / d) for k in range(d // 2)])


def rotate(x, positions, cfg, heads):
    """rotary.hpp:21-51 — interleaved pairs (2k, 2k+1), angle = pos * base^(-2k/d), double trig.
    x: [n, heads*d] float64 (values already at storage precision)."""
    n = x.shape[0]
    d = cfg.head_dim
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq(cfg)[None, :]
    c, s = np.cos(ang), np.sin(ang)
    v = x.reshape(n, heads, d // 2, 2)
    a, b = v[..., 0], v[..., 1]
    out = np.empty_like(v)
    out[..., 0] = a * c[:, None, :] - b * s[:, None, :]
    out[..., 1] = a * s[:, None, :] + b * c[:, None, :]
    return out.reshape(n, heads * d)


def norm_rows(x, cfg):
    """attention.hpp:84-104 (LN, no affine, eps 1e-5) or RMSNorm (gain 1)."""
    if cfg.norm == "rms":
        return x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + cfg.eps)
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    return (x - mu) / np.sqrt(var + cfg.eps)


def silu(z):
    return z / (1.0 + np.exp(-z))


def attend(q, k, v, cfg, allow):
    """attention.hpp:129-176 with GQA. q: [nq, Hq*d]; k, v: [nk, Hkv*d]; allow: bool [nq, nk].
    Rows with nothing allowed stay zero."""
    d, Hq, Hkv = cfg.head_dim, cfg.num_heads, cfg.kv_heads
    g = Hq // Hkv
    out = np.zeros_like(q)
    scale = 1.0 / math.sqrt(d)
    for h in range(Hq):
        kh = h // g
        qs = q[:, h * d:(h + 1) * d]
        ks = k[:, kh * d:(kh + 1) * d]
        vs = v[:, kh * d:(kh + 1) * d]
        s = (qs @ ks.T) * scale
        s = np.where(allow, s, -np.inf)
        m = s.max(axis=1, keepdims=True)
        any_ = np.isfinite(m[:, 0])
        m = np.where(np.isfinite(m), m, 0.0)
        p = np.where(allow, np.exp(s - m), 0.0)
        den = p.sum(axis=1, keepdims=True)
        den = np.where(den > 0, den, 1.0)
        o = (p @ vs) / den
        o[~any_] = 0.0
        out[:, h * d:(h + 1) * d] = o
    return out


def _norm_in(x, cfg, storage, first_layer):
    """The projection input norm(x). The bf16 mirror follows the CUDA path's RMSNorm fold
    (gemm_tc.cuh EpiParams, model.cu forward_bf16): for RMS models with hidden % 512 == 0 every
    projection after the embedding's reads bf16(x) and scales its accumulator rows by
    rsqrt(mean(x^2) + eps) of the f32 residual, i.e. norm(x) is bf16(x) * r, not bf16(x * r)."""
    if storage == "bf16" and cfg.norm == "rms" and cfg.hidden % 512 == 0 and not first_layer:
        r = 1.0 / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + cfg.eps)
        return round_bf16(x) * r
    return storage_round(storage)(norm_rows(x, cfg))


def _ffn(x, L, cfg, storage):
    """attention.hpp:192-203 (LN -> W_in -> SiLU -> W_out -> residual), + SwiGLU extension."""
    rnd = storage_round(storage)
    xn = _norm_in(x, cfg, storage, False)
    up = xn @ L["ffn_in"].T
    if _ref_storage(storage):
        up = rnd(up)
        mid = rnd(silu(rnd(xn @ L["ffn_gate"].T)) * up) if cfg.mlp == "swiglu" else rnd(silu(up))
        return rnd(x + rnd(mid @ L["ffn_out"].T))
    # bf16 mirror: the up/gate GEMM epilogue applies the activation to the f32 accumulator
    mid = rnd(silu(xn @ L["ffn_gate"].T) * up) if cfg.mlp == "swiglu" else rnd(silu(up))
    return round_f32(x + mid @ L["ffn_out"].T)


def forward(cfg, W: Weights, own_tokens, own_pos, ctx_k=None, ctx_v=None, allow=None,
            storage="f32", keep_kv=False):
    """Shared core of prefill (attention.hpp:210-247) and query_attend (:368-414).

    own rows attend [ctx ; own] with `allow` [n_own, n_ctx + n_own]. ctx_k is already
    rotated (per layer list). Returns (hidden, k_raw, k_rot, v) per layer.
    f32 storage rounds exactly where the reference stores Real; bf16 storage mirrors the
    CUDA bf16 path (bf16 GEMM inputs/outputs, f32 residual stream).
    """
    rnd = storage_round(storage)
    x = W.embed(own_tokens)
    n_ctx = 0 if ctx_k is None else ctx_k[0].shape[0]
    k_raw_l, k_rot_l, v_l = [], [], []
    for l, L in enumerate(W.layers):
        xn = _norm_in(x, cfg, storage, l == 0)
        q = xn @ L["wq"].T
        k = xn @ L["wk"].T
        v = rnd(xn @ L["wv"].T)
        if _ref_storage(storage):
            q, k = rnd(q), rnd(k)
            q_rot = rnd(rotate(q, own_pos, cfg, cfg.num_heads))
            k_rot = rnd(rotate(k, own_pos, cfg, cfg.kv_heads))
        else:  # GEMM epilogue rotates the f32 accumulator, then stores bf16
            q_rot = rnd(rotate(q, own_pos, cfg, cfg.num_heads))
            k_rot = rnd(rotate(k, own_pos, cfg, cfg.kv_heads))
            k = rnd(k)
        if keep_kv:
            k_raw_l.append(k)
            k_rot_l.append(k_rot)
            v_l.append(v)
        kk = k_rot if n_ctx == 0 else np.concatenate([ctx_k[l], k_rot])
        vv = v if n_ctx == 0 else np.concatenate([ctx_v[l], v])
        att = rnd(attend(q_rot, kk, vv, cfg, allow))
        if _ref_storage(storage):
            x = rnd(x + rnd(att @ L["wo"].T))
        else:  # f32 residual stream, O-GEMM epilogue adds the accumulator
            x = round_f32(x + att @ L["wo"].T)
        x = _ffn(x, L, cfg, storage)
    return x, k_raw_l, k_rot_l, v_l


def block_allow(groups_own, n_ctx=0):
    """BlockMask::allows (attention.hpp:37-39) over own rows; ctx rows (if any) are
    always visible to query rows (group -1)."""
    g = np.asarray(groups_own)
    n = len(g)
    j = np.arange(n)
    causal = j[None, :] <= j[:, None]
    same = (g[:, None] == -1) | (g[:, None] == g[None, :])
    own = causal & same
    if n_ctx:
        return np.concatenate([np.ones((n, n_ctx), bool), own], axis=1)
    return own


def prefill(cfg, W, tokens, groups, storage="f32"):
    """attention.hpp:210-247. positions are 0..n-1 (BlockMask::append_block)."""
    h, kr, kro, v = forward(cfg, W, tokens, np.arange(len(tokens)), allow=block_allow(groups),
                            storage=storage, keep_kv=True)
    return {"hidden": h, "k_raw": kr, "k_rot": kro, "v": v}


def encode_group(cfg, W, tables_tokens, storage="f32"):
    """attention.hpp:254-294: single causal block at local positions; returns per table
    (local_offset, k_raw[l], v[l]) — stored K is the PRE-rotation projection."""
    concat = [t for tt in tables_tokens for t in tt]
    r = prefill(cfg, W, concat, [0] * len(concat), storage)
    out, off = [], 0
    for tt in tables_tokens:
        n = len(tt)
        out.append({"local_offset": off, "k": [k[off:off + n] for k in r["k_raw"]],
                    "v": [v[off:off + n] for v in r["v"]]})
        off += n
    return out


def assemble(cfg, kvs, storage="f32"):
    """attention.hpp:300-362: concat in order; K rotated at cursor+t (global from 0), V copied."""
    rnd = storage_round(storage)
    L = len(kvs[0]["k"]) if kvs else cfg.num_layers
    ks, vs, spans, cursor = [[] for _ in range(L)], [[] for _ in range(L)], [], 0
    for kv in kvs:
        n = kv["k"][0].shape[0]
        pos = np.arange(cursor, cursor + n)
        for l in range(L):
            ks[l].append(rnd(rotate(kv["k"][l], pos, cfg, cfg.kv_heads)))
            vs[l].append(rnd(kv["v"][l]) if storage == "bf16" else kv["v"][l])  # bf16 prefix slab
        spans.append((cursor, cursor + n))
        cursor += n
    ks = [np.concatenate(k) if k else np.zeros((0, cfg.kv_dim)) for k in ks]
    vs = [np.concatenate(v) if v else np.zeros((0, cfg.kv_dim)) for v in vs]
    return ks, vs, cursor


def query_attend(cfg, W, ctx_k, ctx_v, n_ctx, query_tokens, storage="f32"):
    """attention.hpp:368-414: positions nctx+i; own rows see all ctx + causal own."""
    nq = len(query_tokens)
    allow = block_allow([-1] * nq, n_ctx)
    h, *_ = forward(cfg, W, query_tokens, np.arange(n_ctx, n_ctx + nq),
                    ctx_k if n_ctx else None, ctx_v if n_ctx else None, allow, storage)
    return h


def head_logits(cfg, W, last_row, storage="f32"):
    """Documented extension: final norm + untied mix3 head (tag 8), double."""
    xn = norm_rows(np.asarray(last_row, dtype=np.float64)[None, :], cfg)
    if storage == "bf16":
        xn = round_bf16(xn)
    return (xn @ W.head().T)[0]


def head_logits_rows(cfg, W, rows, storage="f32", chunk=8192):
    """head_logits for several final rows at once, the head generated chunk by chunk (a
    128256 x 4096 head is 4.2 GB in f64): same definition and rounding as head_logits."""
    xn = norm_rows(np.asarray(rows, dtype=np.float64).reshape(-1, cfg.hidden), cfg)
    if storage == "bf16":
        xn = round_bf16(xn)
    out = np.empty((xn.shape[0], cfg.vocab_size))
    for r0 in range(0, cfg.vocab_size, chunk):
        n = min(chunk, cfg.vocab_size - r0)
        w = weight(cfg, "head", 0, cfg.vocab_size, cfg.hidden, storage, row_start=r0, row_count=n)
        out[:, r0:r0 + n] = xn @ w.T
    return out


def groups_prefix_complete(plan_groups, group_of, assembly):
    """True when every encoding group the assembly touches contributes a PREFIX of its encode
    order (engine.cpp:83-112): then each cached table saw exactly the same predecessors at encode
    time as in the no-cache block-masked prefill, and (RoPE being relative) the cached path equals
    the no-cache one in exact arithmetic. Otherwise a table was encoded against group members the
    query does not contain — the reference's by-design approximation (engine_test.cpp:264-269)."""
    used = {}
    for t in assembly:
        used.setdefault(group_of[t], []).append(t)
    return all(plan_groups[g][:len(ts)] == ts for g, ts in used.items())


# ============================================================================ .kv format
# table_kv.hpp:45-118


def decode_kv(raw: bytes):
    hdr = np.frombuffer(raw[:24], dtype="<u4")
    tid, ntok, nl, nh, hd, off = (int(x) for x in hdr)
    per = ntok * nh * hd
    if len(raw) != 24 + 8 * per * nl:
        raise ValueError("KV file size mismatch")
    body = np.frombuffer(raw[24:], dtype="<f4").astype(np.float64)
    k = [body[l * per:(l + 1) * per].reshape(ntok, nh * hd) for l in range(nl)]
    v = [body[(nl + l) * per:(nl + l + 1) * per].reshape(ntok, nh * hd) for l in range(nl)]
    return {"table_id": tid, "token_count": ntok, "num_layers": nl, "num_heads": nh, "head_dim": hd,
            "local_offset": off, "k": k, "v": v}
