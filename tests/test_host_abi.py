"""CPU tests of the product's host side through the C ABI (no GPU work is launched).

The C++ implementations behind libtkv.so (trie, rerank, TieredCache, schedule/build_trace/
simulate, engine) must reproduce the reference's goldens exactly — the same fixtures the
oracle is pinned to (tests/golden, written by the unchanged reference).
"""
import json
import os

import numpy as np
import pytest

import golden_inputs as GI
import tkv_oracle as O
from golden_util import demo_path, load

N = pytest.importorskip("paper_2601_08743_b200.native")


def test_library_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(N.LIB_PATH)
    assert len(N.EXPORTED) >= 40
    for name in N.EXPORTED:
        assert hasattr(lib, name), name


def test_status_names_match_reference_taxonomy():
    names = ["DanglingForeignKey", "CycleDetected", "DuplicateTable", "EmptySerialization", "DuplicateSerialization",
             "UnknownTable", "CacheNotFull", "TableIdOutOfRange", "LengthMismatch", "DimensionMismatch", "EmptyGroup",
             "MissingTableKV", "GroupOrderViolation", "EmptyBatch", "MissingCacheDir", "VerifyFailed", "BadConfig",
             "IoError"]
    assert [N.status_name(i + 1) for i in range(18)] == names
    assert N.status_name(0) == "ok"


@pytest.fixture(scope="module")
def demo_engine():
    return N.Engine(demo_path("demo_schema.json"))


def test_engine_build_matches_reference(demo_engine):
    g = load("demo64")["result"]
    info = demo_engine.info
    assert info["vocab_size"] == g["vocab_size"]
    assert info["vocab_hash"] == g["vocab_hash"]
    assert info["table_tokens"] == g["table_tokens"]
    assert info["groups"] == g["groups"]
    assert info["group_of"] == g["group_of"]
    assert info["local_offset"] == g["local_offset"]
    assert info["topo_order"] == g["topo_order"]
    assert info["serialized"] == g["serialized"]
    assert info["edges"] == g["edges"]


def _workload(path, n):
    lines = [json.loads(l) for l in open(path) if l.strip()]
    return [(l["query_id"], l["text"]) for l in lines if "query_id" in l][:n]


def test_prompt_analysis_matches_reference(demo_engine):
    g = load("demo64")["result"]
    for (qid, text), gq in zip(_workload(demo_path("demo_workload.jsonl"), 64), g["queries"]):
        a = demo_engine.analyze(text, qid)
        assert a["tokens"] == gq["tokens"]
        assert a["spans"] == gq["spans"]
        assert a["match_order"] == gq["match_order"]
        assert a["remainder"] == gq["remainder"]
        assert a["assembly_order"] == gq["assembly_order"]
        assert a["record_tables"] == gq["record_tables_sorted"]


def test_c2_engine_and_analysis():
    from paper_2601_08743_b200 import workloads as W
    g = load("c2")["result"]
    tabs, ents, _ = W.spider_like(W.CONFIGS["c2"])
    e = N.Engine(corpus_json=W.dump_schema_corpus(tabs))
    assert e.info["vocab_hash"] == g["vocab_hash"]
    for (qid, text), gq in list(zip(ents, g["queries"]))[:300]:
        a = e.analyze(text, qid)
        assert a["spans"] == gq["spans"] and a["assembly_order"] == gq["assembly_order"]


def test_engine_errors_carry_reference_codes(tmp_path):
    bad = {"format_version": 1, "tables": [
        {"table_id": 0, "name": "a", "columns": [{"name": "id"}], "foreign_keys": [{"column": "id", "ref_table": 1, "ref_column": "id"}]},
        {"table_id": 1, "name": "b", "columns": [{"name": "id"}], "foreign_keys": [{"column": "id", "ref_table": 0, "ref_column": "id"}]}]}
    with pytest.raises(N.TkvError) as ei:
        N.Engine(corpus_json=json.dumps(bad))
    assert ei.value.name == "CycleDetected"
    e = N.Engine(corpus_json=json.dumps(bad), break_cycles=True)
    assert e.info["removed_edges"] and len(e.info["topo_order"]) == 2
    dangling = {"format_version": 1, "tables": [
        {"table_id": 0, "name": "a", "columns": [{"name": "id"}], "foreign_keys": [{"column": "id", "ref_table": 5, "ref_column": "id"}]}]}
    with pytest.raises(N.TkvError) as ei:
        N.Engine(corpus_json=json.dumps(dangling))
    assert ei.value.name == "DanglingForeignKey"
    with pytest.raises(N.TkvError) as ei:
        N.Engine(schema_path=str(tmp_path / "missing.json"))
    assert ei.value.name == "IoError"


def test_trie_goldens_and_errors():
    g = load("trie")["result"]
    pats, inputs = GI.trie_inputs()
    t = N.Trie()
    for i, p in enumerate(pats):
        t.insert(p, i)
    for x, gg in zip(inputs, g):
        spans, visits = t.match_all(x)
        assert [list(s) for s in spans] == gg["spans"]
        assert visits == gg["node_visits"]
        for s, q in enumerate(gg["query_first32"]):
            f, n, tid = t.query(x, s)
            assert f == q[0] and tid == q[2] and (not f or n == q[1])
    with pytest.raises(N.TkvError) as ei:
        t.insert([], 99)
    assert ei.value.name == "EmptySerialization"
    with pytest.raises(N.TkvError) as ei:
        t.insert([1, 2, 3, 4, 5], 0)
    assert ei.value.name == "DuplicateTable"
    with pytest.raises(N.TkvError) as ei:
        t.insert(pats[1], 1000)
    assert ei.value.name == "DuplicateSerialization"


def test_trie_nested_fallback_pinned_by_reference_test():
    # trie_test.cpp:81-92: [5,7] and [5,7,9] inserted; input {5,7,8} matches t1, next 2
    t = N.Trie()
    t.insert([5, 7], 1)
    t.insert([5, 7, 9], 3)
    assert t.query([5, 7, 8], 0) == (True, 2, 1)
    assert t.query([5, 7, 9], 0) == (True, 3, 3)


def test_rerank_goldens_single_and_multithreaded():
    g = load("rerank")["result"]
    for b, gg in zip(GI.rerank_batches(), g):
        assert N.rerank(b["queries"], b["n_bits"], b["seed"], b["mode"]) == gg["order"]
    # threaded argmin must give the same chain as the serial scan on a big batch
    rng = np.random.default_rng(3)
    sets = [list(rng.choice(300, size=rng.integers(0, 6), replace=False)) for _ in range(5000)]
    a = N.rerank(sets, 300, 7, threads=1)
    b = N.rerank(sets, 300, 7, threads=8)
    assert a == b and sorted(a) == list(range(5000))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_rerank_class_reduction_equals_row_chain(seed):
    """rerank_packed chains distinct table sets and expands each class in ascending slot order
    (rerank_classes): on batches full of duplicate sets, empty sets and anchors landing inside a
    class, the order equals the oracle's row-by-row restatement of rerank.cpp:55-94."""
    rng = np.random.default_rng(seed)
    base = [sorted(set(rng.integers(0, 20, rng.integers(0, 4)).tolist())) for _ in range(12)]
    sets = [base[int(rng.integers(0, len(base)))] for _ in range(300)]
    for mode in ("seeded", "fixed_first"):
        for s in (seed, seed + 10, seed + 20):
            assert N.rerank(sets, 20, s, mode) == O.rerank(sets, 20, s, mode)


def test_cache_goldens():
    g = load("cache_ops")["result"]
    for case, gg in zip(GI.cache_cases(), g):
        c = N.Cache(case["capacity"], case["policy"], GI.CACHE_TOKEN_COUNTS)
        for op, st in zip(case["ops"], gg["steps"]):
            if "candidate" in st:
                assert c.evict_candidate() == st["candidate"]
            if "get" in op:
                assert c.get(op["get"]) == (st["hit"], st["evicted"])
            else:
                assert c.prefetch(op["prefetch"]) == st["admitted"]
            cnt, res = c.state()
            assert res == st["residents"] and cnt == st["counters"]
    c = N.Cache(2, "lru", [5, 5, 5])
    with pytest.raises(N.TkvError) as ei:
        c.evict_candidate()
    assert ei.value.name == "CacheNotFull"


def test_cache_unbounded_capacity():
    """The reference cache is map-based: any size_t capacity, SIZE_MAX included, costs nothing
    up front (slots are allocated as entries are admitted)."""
    c = N.Cache(2**64 - 1, "lfu", [5] * 100)
    for t in range(100):
        assert c.get(t) == (False, -1)
    assert c.get(7) == (True, -1)
    cnt, res = c.state()
    assert res == list(range(100)) and cnt[:3] == [1, 100, 0]


def _cmp_run(mine, ref):
    assert mine["order"] == ref["order"]
    assert [[w["begin"], w["end"], w["demand"], w["prefetch"]] for w in mine["plan"]["windows"]] == \
           [[w["begin"], w["end"], w["demand"], w["prefetch"]] for w in ref["plan"]["windows"]]
    assert mine["trace"]["windows"] == ref["trace"]["windows"]
    assert np.allclose(mine["trace"]["compute"], ref["trace"]["compute"], rtol=1e-12)
    assert mine["final_residents"] == ref["final_residents"]
    for rk in ("report", "report_overlapped", "report_serial"):
        a, b = mine[rk], ref[rk]
        for k in ("hits", "misses", "swaps", "prefetch_loads"):
            assert a[k] == b[k], (rk, k)
        for k in ("total_ttft", "makespan", "total_compute", "total_transfer", "serial_baseline_ttft"):
            assert a[k] == pytest.approx(b[k], rel=1e-12, abs=1e-12), (rk, k)
        assert a["queries"] == b["queries"]


def test_run_batch_matches_reference_traces():
    for sc in load("run_batch"):
        out = N.run_batch_json(sc["input"])
        for r in sc["input"]["runs"]:
            _cmp_run(out[r["name"]], sc["output"][r["name"]])


@pytest.mark.parametrize("name,runs", [("demo64", "demo"), ("demo200", "demo"), ("c2", "c2")])
def test_serving_traces_match_reference(name, runs):
    g = load(name)["result"]
    counts = [len(t) for t in g["table_tokens"]]
    qs = [{"id": q["query_id"], "tables": q["assembly_order"], "query_tokens": q["query_token_count"]} for q in g["queries"]]
    run_list = [r for r in (GI.demo_runs() if runs == "demo" else GI.c2_runs()) if r["name"] in g["runs"]]
    out = N.run_batch_json({"token_counts": counts, "queries": qs, "runs": run_list})
    for r in run_list:
        _cmp_run(out[r["name"]], g["runs"][r["name"]])


def test_run_workload_simulated_report(demo_engine, tmp_path):
    g = load("demo64")["result"]
    wl = tmp_path / "w.jsonl"
    lines = open(demo_path("demo_workload.jsonl")).read().splitlines()[:65]
    wl.write_text("\n".join(lines) + "\n")
    for r in GI.demo_runs():
        rep = demo_engine.run_workload(str(wl), r)
        ref = g["runs"][r["name"]]["run_workload"]
        assert rep["queries"] == ref["queries"]
        assert [rep[k] for k in ("hits", "misses", "swaps", "prefetch_loads")] == \
               [ref[k] for k in ("hits", "misses", "swaps", "prefetch_loads")]
        assert rep["total_ttft"] == pytest.approx(ref["total_ttft"], rel=1e-12)


def test_run_workload_reads_reference_kv_files(demo_engine):
    rep = demo_engine.run_workload(demo_path("demo_workload.jsonl"), GI.demo_runs()[0], kv_dir=demo_path("kv"))
    assert [rep[k] for k in ("hits", "misses", "swaps", "prefetch_loads")] == [784, 4, 6, 8]


def test_check_manifest_detects_missing_dir(demo_engine, tmp_path):
    with pytest.raises(N.TkvError) as ei:
        demo_engine.check_manifest(str(tmp_path / "nope"))
    assert ei.value.name == "MissingCacheDir"
