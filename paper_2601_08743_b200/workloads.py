"""Synthetic schema corpora and query workloads for the BASELINE.json configs.

* ``demo`` (C1): the reference's demo generator semantics (proj/tools/gen_demo.cpp:30-178):
  12-table schema (a 4-table PFK chain, a 4-table ledger cluster, 4 cold tables), prompts
  = the matched tables' serializations in a SeededRng-shuffled order + a question line;
  two hot clusters alternate and every 50th query touches a cold table. The first 64
  queries of the 200-query file are the C1 workload (generation is sequential, so the
  64-query run is a prefix). Output is byte-identical to proj/data/*.
* ``spider_like`` (C2/C3/C5): many small databases, per-database random PFK DAGs
  (FK only to lower ids, p = fk_p), text serializations sized to a token range, queries
  drawn Zipf over databases and Zipf over tables inside a database, shuffled table order,
  a question suffix of a given token range.

Everything is deterministic in the seed. Files are written in the reference's own
formats (schema corpus JSON, proj/src/schema.cpp:373-396; workload JSONL,
proj/src/engine.cpp:329-334), so the same files feed the reference and this repo.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

from .rng import SeededRng


# ----------------------------------------------------------------------------- corpus IO

def _col(name, desc="", pk=False):
    return {"name": name, "description": desc, "is_primary_key": pk}


def _table(tid, name, cols, fks=()):
    return {"table_id": tid, "name": name, "columns": list(cols),
            "foreign_keys": [{"column": c, "ref_table": t, "ref_column": rc} for (c, t, rc) in fks]}


def dump_schema_corpus(tables) -> str:
    """Same bytes as the reference's dump_schema_corpus (nlohmann dump(2), sorted keys)."""
    doc = {"format_version": 1, "tables": tables}
    return json.dumps(doc, indent=2, sort_keys=True, ensure_ascii=False) + "\n"


def dump_workload(entries) -> str:
    out = json.dumps({"format_version": 1}, separators=(",", ":")) + "\n"
    for qid, text in entries:
        out += json.dumps({"query_id": qid, "text": text}, separators=(",", ":"),
                          sort_keys=True, ensure_ascii=False) + "\n"
    return out


def serialize_table(t) -> str:
    """proj/src/serialize.cpp:5-18 — one name line, one line per column."""
    out = "table " + t["name"] + "\n"
    for c in t["columns"]:
        out += "col " + c["name"]
        if c["description"]:
            out += ": " + c["description"]
        if c["is_primary_key"]:
            out += " [pk]"
        for fk in t["foreign_keys"]:
            if fk["column"] == c["name"]:
                out += " [fk #%d.%s]" % (fk["ref_table"], fk["ref_column"])
        out += "\n"
    return out


# ----------------------------------------------------------------------------- C1 demo

def demo_schema():
    return [
        _table(0, "districts", [_col("id", "district identifier", True), _col("name"),
                                _col("county", "county the district serves")]),
        _table(1, "schools", [_col("id", "", True), _col("district_id"), _col("name", "school name"),
                              _col("charter", "1 if charter funded")], [("district_id", 0, "id")]),
        _table(2, "classes", [_col("id", "", True), _col("school_id"), _col("subject", "course subject code"),
                              _col("room")], [("school_id", 1, "id")]),
        _table(3, "enrollments", [_col("id", "", True), _col("class_id"), _col("student_name"),
                                  _col("grade", "final letter grade")], [("class_id", 2, "id")]),
        _table(4, "vendors", [_col("id", "", True), _col("name", "legal entity name"), _col("city")]),
        _table(5, "invoices", [_col("id", "", True), _col("vendor_name"), _col("total", "amount in dollars"),
                               _col("issued", "issue date")]),
        _table(6, "audits", [_col("id", "", True), _col("subject"), _col("status", "open, closed, or escalated")]),
        _table(7, "payments", [_col("id", "", True), _col("invoice_ref", "free-form invoice reference"),
                               _col("amount"), _col("method")]),
        _table(8, "budgets", [_col("id", "", True), _col("year"), _col("allocation", "planned spend in dollars")]),
        _table(9, "grants", [_col("id", "", True), _col("sponsor"), _col("awarded")]),
        _table(10, "assets", [_col("id", "", True), _col("description"), _col("purchased", "purchase date")]),
        _table(11, "permits", [_col("id", "", True), _col("holder"), _col("expires")]),
    ]


_CHAIN_Q = ["question: how many students enrolled in charter schools\n",
            "question: which county has the most classes per school\n",
            "question: list schools whose enrollments dropped\n",
            "question: average grade by district\n"]
_LEDGER_Q = ["question: total invoice amount per vendor\n",
             "question: which payments lack an audit\n",
             "question: vendors with escalated audits\n",
             "question: largest payment method by volume\n"]
_COLD_Q = ["question: budget allocation for the current year\n",
           "question: sponsors with more than one grant\n",
           "question: assets purchased this quarter\n",
           "question: permits expiring soon\n"]


def demo_workload(n_queries=200, seed=1, shuffle_tables=True):
    """gen_demo.cpp:149-178 semantics."""
    corpus = demo_schema()
    rendered = [serialize_table(t) for t in corpus]
    rng = SeededRng(seed)

    def prompt(tables, question):
        tables = list(tables)
        if shuffle_tables:
            for i in range(len(tables), 1, -1):
                j = rng.next_below(i)
                tables[i - 1], tables[j] = tables[j], tables[i - 1]
        return "".join(rendered[t] for t in tables) + question

    out = []
    for i in range(n_queries):
        qid = "q%d" % i
        if i % 50 == 49:
            cold = 8 + (i // 50) % 4
            out.append((qid, prompt([cold], _COLD_Q[cold - 8])))
        elif i % 2 == 0:
            out.append((qid, prompt([0, 1, 2, 3], _CHAIN_Q[(i // 2) % 4])))
        else:
            out.append((qid, prompt([4, 5, 6, 7], _LEDGER_Q[(i // 2) % 4])))
    return out


DEMO_CONFIG = {"format_version": 1, "capacity_C": 6, "policy": "lru", "b_c": 1, "b_m": 1,
               "compute_per_token": 0.01, "load_per_token": 1.0, "switch_overhead": 5.0,
               "rerank_on": True, "pipeline_on": True, "seed": 1}


# ----------------------------------------------------------------------------- Spider-like

_SYL = ["ka", "lo", "mi", "ne", "ru", "ta", "vo", "si", "de", "pa", "gu", "ze", "bo", "fi", "ho", "ja"]


def _word(i: int) -> str:
    """Deterministic pseudo-word (3 syllables, base-16 digits of i)."""
    s = ""
    for _ in range(3):
        s += _SYL[i % 16]
        i //= 16
    return s + ("" if i == 0 else str(i))


def _zipf_pick(rng: SeededRng, weights_cdf):
    u = rng.next_unit() * weights_cdf[-1]
    lo, hi = 0, len(weights_cdf) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if weights_cdf[mid] > u:
            hi = mid
        else:
            lo = mid + 1
    return lo


def _zipf_cdf(n, s):
    acc, out = 0.0, []
    for r in range(1, n + 1):
        acc += 1.0 / (r ** s)
        out.append(acc)
    return out


def _approx_tokens(cols, fks_by_col):
    # tokens: "table", " ", name, "\n" = 4; per column "col"," ",name = 3, desc words w: 2 + 2w - 1,
    # pk " [pk]" = 4, fk " [fk #t.c]" = 9 (+digits), newline 1.
    n = 4
    for c in cols:
        n += 3 + 1
        if c["description"]:
            n += 2 + 2 * len(c["description"].split(" ")) - 1
        if c["is_primary_key"]:
            n += 4
        if c["name"] in fks_by_col:
            n += 9
    return n


@dataclass
class SpiderSpec:
    n_db: int = 40
    tables_per_db: int = 5
    table_tokens: tuple = (40, 160)
    query_tables: tuple = (2, 5)
    query_tokens: tuple = (16, 64)
    n_queries: int = 1000
    zipf_s: float = 1.1
    fk_p: float = 0.3
    seed: int = 1


def spider_like(spec: SpiderSpec):
    """Returns (tables, workload entries, per-query db ids)."""
    rng = SeededRng(spec.seed)
    tables = []
    word_base = 0
    for db in range(spec.n_db):
        dbw = "db" + _word(db)
        for k in range(spec.tables_per_db):
            tid = db * spec.tables_per_db + k
            target = spec.table_tokens[0] + rng.next_below(spec.table_tokens[1] - spec.table_tokens[0] + 1)
            fks = []
            cols = [_col("id", "row identifier", True)]
            for j in range(k):
                if rng.next_unit() < spec.fk_p:
                    cname = "t%d_id" % j
                    cols.append(_col(cname))
                    fks.append((cname, db * spec.tables_per_db + j, "id"))
            fk_cols = {c for (c, _, _) in fks}
            ci = 0
            while True:
                nw = rng.next_below(4)
                desc = " ".join(_word(word_base + rng.next_below(600)) for _ in range(nw))
                cand = cols + [_col("c%d_%s" % (ci, _word(rng.next_below(300))), desc)]
                if _approx_tokens(cand, fk_cols) > target and len(cols) > 1:
                    break
                cols = cand
                ci += 1
            tables.append(_table(tid, "%s_t%d_%s" % (dbw, k, _word(tid)), cols, fks))
    db_cdf = _zipf_cdf(spec.n_db, spec.zipf_s)
    tb_cdf = _zipf_cdf(spec.tables_per_db, spec.zipf_s)
    rendered = [serialize_table(t) for t in tables]
    entries, dbs = [], []
    for i in range(spec.n_queries):
        db = _zipf_pick(rng, db_cdf)
        lo, hi = spec.query_tables
        want = min(spec.tables_per_db, lo + rng.next_below(hi - lo + 1))
        picked = []
        while len(picked) < want:
            t = _zipf_pick(rng, tb_cdf)
            if t not in picked:
                picked.append(t)
        for a in range(len(picked), 1, -1):
            b = rng.next_below(a)
            picked[a - 1], picked[b] = picked[b], picked[a - 1]
        ids = [db * spec.tables_per_db + t for t in picked]
        qlo, qhi = spec.query_tokens
        qt = qlo + rng.next_below(qhi - qlo + 1)
        # "question" ":" " " + words separated by spaces + "\n": 3 + 2w tokens
        nw = max(1, (qt - 3) // 2)
        q = "question: " + " ".join(_word(rng.next_below(600)) for _ in range(nw)) + "\n"
        entries.append(("q%d" % i, "".join(rendered[t] for t in ids) + q))
        dbs.append(db)
    return tables, entries, dbs


CONFIGS = {
    # BASELINE.json configs[1]: 40 DBs / 200 tables, Zipf, 1k queries (FIFO vs LRU, C=32,
    # b_c=100, b_m=10); TTFT measured with the Llama-3-8B-shaped model.
    "c2": SpiderSpec(),
    # configs[2]: ~4k-token prefixes, 8-16 tables x 256-512 tokens, 32-128 suffix tokens.
    "c3": SpiderSpec(n_db=16, tables_per_db=16, table_tokens=(256, 512), query_tables=(8, 16),
                     query_tokens=(32, 128), n_queries=256),
    # configs[4]: BIRD-like wide schemas (~60 tables per DB), prefixes up to 16k tokens.
    "c5": SpiderSpec(n_db=11, tables_per_db=60, table_tokens=(180, 360), query_tables=(10, 50),
                     query_tokens=(32, 128), n_queries=10000),
}


def write_corpus(dirpath, tables, entries):
    os.makedirs(dirpath, exist_ok=True)
    sp = os.path.join(dirpath, "schema.json")
    wp = os.path.join(dirpath, "workload.jsonl")
    with open(sp, "w") as f:
        f.write(dump_schema_corpus(tables))
    with open(wp, "w") as f:
        f.write(dump_workload(entries))
    return sp, wp
