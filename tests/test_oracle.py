"""Pins the CPU oracle (oracle/tkv_oracle.py) to the unchanged reference's own outputs.

Every golden here was produced by running /root/reference/proj (compiled by oracle/Makefile)
through oracle/_ref/golden_dump — see tests/golden/make_goldens.py. Integer/trace work
must match exactly; floating point within the reference's own tolerances
(f32 1e-5 / f64 1e-10, proj/tests/acceptance/acceptance.cpp:131).
"""
import json

import numpy as np
import pytest

import golden_inputs as GI
import tkv_oracle as O
from golden_util import Tensors, demo_path, load


def test_rng_mix3_and_stream():
    g = load("rng")["result"]
    assert [str(O.mix3(*t)) for t in GI.RNG_TRIPLES] == g["mix3"]
    for seed, seq in zip(GI.RNG_SEEDS, g["seeded"]):
        r = O.SeededRng(seed)
        assert [str(r.next_u64()) for _ in range(8)] == seq
    assert [O.u64_to_signed_unit(O.mix3(*t)) for t in GI.RNG_TRIPLES] == g["signed_unit"]
    for t in GI.RNG_TRIPLES:  # vectorised form used for weights
        assert O.mix3_unit_array(t[0], t[1], t[2], 1)[0] == O.u64_to_signed_unit(O.mix3(*t))


def test_rotary_matches_reference():
    T = Tensors("rotary")
    for i, c in enumerate(GI.ROTARY_CASES):
        cfg = O.ModelConfig(num_heads=c["heads"], head_dim=c["head_dim"], rotary_base=c["base"])
        got = O.round_f32(O.rotate(T["r%d.in" % i].astype(np.float64), c["positions"], cfg, c["heads"]))
        assert np.abs(got - T["r%d.out" % i]).max() <= 1e-7


@pytest.fixture(scope="module")
def demo_plan():
    return O.build_engine(json.load(open(demo_path("demo_schema.json")))["tables"])


def _workload(path, n):
    lines = [json.loads(l) for l in open(path) if l.strip()]
    return [(l["query_id"], l["text"]) for l in lines if "query_id" in l][:n]


def test_demo_engine_and_prompt_analysis(demo_plan):
    g = load("demo64")["result"]
    p = demo_plan
    assert p.tokenizer.vocab_size() == g["vocab_size"]
    assert p.tokenizer.vocab_hash() == g["vocab_hash"]
    assert p.table_tokens == g["table_tokens"]
    assert [grp["tables"] for grp in g["groups"]] == p.groups
    assert p.group_of == g["group_of"]
    assert p.local_offset == g["local_offset"]
    for (qid, text), gq in zip(_workload(demo_path("demo_workload.jsonl"), 64), g["queries"]):
        tokens, spans, mo, rem = O.analyze_query(p, text)
        assert tokens == gq["tokens"]
        assert [list(s) for s in spans] == gq["spans"]
        assert mo == gq["match_order"]
        assert rem == gq["remainder"]
        assert O.assembly_order(p, mo) == gq["assembly_order"]


def test_trie_goldens():
    g = load("trie")["result"]
    pats, inputs = GI.trie_inputs()
    t = O.Trie()
    for i, pt in enumerate(pats):
        t.insert(pt, i)
    for x, gg in zip(inputs, g):
        assert [list(s) for s in t.match_all(x)] == gg["spans"]
        for s, q in enumerate(gg["query_first32"]):
            f, n, tid = t.query(x, s)
            assert f == q[0] and tid == q[2] and (not f or n == q[1])


def test_rerank_goldens():
    g = load("rerank")["result"]
    for b, gg in zip(GI.rerank_batches(), g):
        assert O.rerank(b["queries"], b["n_bits"], b["seed"], b["mode"]) == gg["order"]


def test_cache_ops_goldens():
    g = load("cache_ops")["result"]
    for case, gg in zip(GI.cache_cases(), g):
        c = O.Cache(case["capacity"], case["policy"], GI.CACHE_TOKEN_COUNTS)
        for op, st in zip(case["ops"], gg["steps"]):
            if "candidate" in st:
                assert c.evict_candidate() == st["candidate"]
            if "get" in op:
                assert c.get(op["get"]) == (st["hit"], st["evicted"])
            else:
                assert c.prefetch(op["prefetch"]) == st["admitted"]
            assert c.residents() == st["residents"]
            assert c.counters() == st["counters"]


def cmp_trace(windows, compute, gt):
    assert len(windows) == len(gt["windows"])
    for w, gw in zip(windows, gt["windows"]):
        for kind in ("boundary", "prefetch"):
            assert [(r[0], r[1], r[2]) for r in w[kind]] == [(x["table"], x["miss"], x["evicted"]) for x in gw[kind]]
            assert np.allclose([r[3] for r in w[kind]], [x["size"] for x in gw[kind]])
        assert [[(r[0], r[2]) for r in q] for q in w["emergency"]] == \
               [[(x["table"], x["evicted"]) for x in q] for q in gw["emergency"]]
    assert np.allclose(compute, gt["compute"], rtol=1e-12, atol=1e-12)


def cmp_report(rep, gr):
    for k in ("hits", "misses", "swaps", "prefetch_loads"):
        assert rep[k] == gr[k], k
    for k in ("total_ttft", "makespan", "total_compute", "total_transfer", "serial_baseline_ttft"):
        if k in rep:
            assert rep[k] == pytest.approx(gr[k], rel=1e-9, abs=1e-9), k
    assert rep["query_ids"] == [q["query_id"] for q in gr["queries"]]
    assert np.allclose(rep["ttft"], [q["ttft"] for q in gr["queries"]], rtol=1e-9, atol=1e-9)


def check_runs(records, counts, n_bits, runs_in, runs_out):
    for r in runs_in:
        go = runs_out[r["name"]]
        cost = (r["cost"]["compute_per_token"], r["cost"]["load_per_token"], r["cost"]["switch_overhead"])
        rep = O.run_batch(records, counts, n_bits, r, cost)
        assert rep["order"] == go["order"]
        plan = O.schedule([records[i] for i in rep["order"]], r["b_c"], r["b_m"])
        assert [[w["begin"], w["end"], w["demand"], w["prefetch"]] for w in plan["windows"]] == \
               [[w["begin"], w["end"], w["demand"], w["prefetch"]] for w in go["plan"]["windows"]]
        c = O.Cache(r["capacity"], r["policy"], counts)
        windows, compute = O.build_trace(plan, cost, c)
        cmp_trace(windows, compute, go["trace"])
        assert c.residents() == go["final_residents"]
        cmp_report(rep, go["report"])


def test_run_batch_random_scenarios():
    for sc in load("run_batch"):
        inp = sc["input"]
        recs = [(q["id"], q["tables"], q["query_tokens"]) for q in inp["queries"]]
        check_runs(recs, inp["token_counts"], len(inp["token_counts"]), inp["runs"], sc["output"])


@pytest.mark.parametrize("name", ["demo64", "demo200"])
def test_demo_serving_runs(demo_plan, name):
    g = load(name)["result"]
    counts = [len(t) for t in demo_plan.table_tokens]
    recs = [(q["query_id"], q["assembly_order"], q["query_token_count"]) for q in g["queries"]]
    runs = [r for r in GI.demo_runs() if r["name"] in g["runs"]]
    check_runs(recs, counts, len(counts), runs, g["runs"])
    if name == "demo64":  # survey-recorded C1 counters
        rep = g["runs"]["config"]["report"]
        assert [rep[k] for k in ("hits", "misses", "swaps", "prefetch_loads")] == [249, 4, 3, 5]


def test_c2_spider_like_trace():
    g = load("c2")["result"]
    from paper_2601_08743_b200 import workloads as W
    tabs, ents, _ = W.spider_like(W.CONFIGS["c2"])
    p = O.build_engine(tabs)
    assert p.tokenizer.vocab_hash() == g["vocab_hash"]
    counts = [len(t) for t in p.table_tokens]
    recs = []
    for (qid, text), gq in zip(ents, g["queries"]):
        _, spans, mo, rem = O.analyze_query(p, text)
        assert [list(s) for s in spans] == gq["spans"]
        ao = O.assembly_order(p, mo)
        assert ao == gq["assembly_order"]
        recs.append((qid, ao, len(rem)))
    check_runs(recs, counts, len(counts), GI.c2_runs(), g["runs"])


def test_attention_random_corpora():
    """encode_group / assemble / query_attend / prefill vs the reference on random token
    corpora, in both of the reference's precisions (Real=float and Real=double)."""
    T = Tensors("attention")
    for case, info in zip(GI.attention_cases(), T.result):
        tag = info["tag"]
        st = "f64" if case["double"] else "f32"
        tol = 1e-10 if case["double"] else 2e-6
        cfg = O.ModelConfig(num_layers=case.get("num_layers", 2), num_heads=case.get("num_heads", 4),
                            head_dim=case.get("head_dim", 16), vocab_size=case["vocab"], weight_seed=case["weight_seed"])
        W = O.Weights(cfg, st)
        tt = info["table_tokens"]
        for grp in info["groups"]:
            for t, e in zip(grp["tables"], O.encode_group(cfg, W, [tt[t] for t in grp["tables"]], st)):
                for l in range(cfg.num_layers):
                    assert np.abs(e["k"][l] - T["%skv%d.k%d" % (tag, t, l)]).max() <= tol
                    assert np.abs(e["v"][l] - T["%skv%d.v%d" % (tag, t, l)]).max() <= tol
        # assemble from the REFERENCE's stored blocks (isolates assemble from encode rounding)
        ref_kvs = [{"k": [T["%skv%d.k%d" % (tag, t, l)].astype(np.float64) for l in range(cfg.num_layers)],
                    "v": [T["%skv%d.v%d" % (tag, t, l)].astype(np.float64) for l in range(cfg.num_layers)]}
                   for t in range(len(tt))]
        ks, vs, n = O.assemble(cfg, [ref_kvs[t] for t in info["order"]], st)
        for l in range(cfg.num_layers):
            assert np.abs(ks[l] - T["%sctx_k%d" % (tag, l)]).max() <= (1e-13 if case["double"] else 1e-7)
            assert np.array_equal(vs[l], T["%sctx_v%d" % (tag, l)].astype(np.float64))
        served = O.query_attend(cfg, W, ks, vs, n, case["query_tokens"], st)
        assert np.abs(served - T[tag + "served"]).max() <= tol * 5
        assert np.abs(served - T[tag + "served_oracle"]).max() <= (1e-10 if case["double"] else 1e-5)
        toks = [x for t in info["order"] for x in tt[t]]
        groups = [info["group_of"][t] for t in info["order"] for _ in tt[t]]
        pre = O.prefill(cfg, W, toks, groups, st)  # block-masked no-cache oracle
        assert np.abs(pre["hidden"] - T[tag + "pre_hidden"]).max() <= tol * 5
        for l in range(cfg.num_layers):
            assert np.abs(pre["k_rot"][l] - T["%spre_krot%d" % (tag, l)]).max() <= tol * 5


def test_demo_kv_files_and_numerics(demo_plan):
    """Oracle encode == reference .kv payloads; oracle serving == reference hidden rows;
    documented head logits/argmax == the golden tool's double-precision head."""
    T = Tensors("demo64")
    cfg = O.ModelConfig(vocab_size=T.result["vocab_size"])
    W = O.Weights(cfg, "f32")
    kvs = {}
    for grp in demo_plan.groups:
        enc = O.encode_group(cfg, W, [demo_plan.table_tokens[t] for t in grp], "f32")
        for t, e in zip(grp, enc):
            ref = O.decode_kv(open(demo_path("kv", "%d.kv" % t), "rb").read())
            assert ref["local_offset"] == e["local_offset"] == demo_plan.local_offset[t]
            for l in range(cfg.num_layers):
                assert np.abs(ref["k"][l] - e["k"][l]).max() <= 2e-6
                assert np.abs(ref["v"][l] - e["v"][l]).max() <= 2e-6
            kvs[t] = ref  # serve from the reference bytes, as the product does
    for info, gq in zip(T.result["numerics"], T.result["queries"]):
        qi = info["query"]
        ks, vs, n = O.assemble(cfg, [kvs[t] for t in gq["assembly_order"]], "f32")
        assert n == info["nctx"]
        if "q%d.ctx_k0" % qi in T:
            for l in range(cfg.num_layers):
                assert np.abs(ks[l] - T["q%d.ctx_k%d" % (qi, l)]).max() <= 1e-7
                assert np.array_equal(vs[l], T["q%d.ctx_v%d" % (qi, l)].astype(np.float64))
        h = O.query_attend(cfg, W, ks, vs, n, gq["remainder"], "f32")
        assert np.abs(h - T["q%d.hidden" % qi]).max() <= 1e-5
        if "argmax" in info:
            lg = O.head_logits(cfg, W, T["q%d.hidden" % qi][-1])
            assert np.abs(lg - T["q%d.logits" % qi]).max() <= 1e-9
            assert int(np.argmax(lg)) == info["argmax"]
