"""Deterministic inputs behind every golden fixture (shared by make_goldens.py and tests)."""
from paper_2601_08743_b200.rng import SeededRng

COST = {"compute_per_token": 0.01, "load_per_token": 1.0, "switch_overhead": 5.0}


def run(name, **kw):
    r = {"name": name, "rerank_on": True, "pipeline_on": True, "capacity": 6, "policy": "lru",
         "b_c": 1, "b_m": 1, "seed": 1, "anchor": "seeded", "cost": dict(COST)}
    r.update(kw)
    return r


def demo_runs():
    return [run("config"), run("no_pipeline", pipeline_on=False), run("no_rerank", rerank_on=False),
            run("no_mgmt", pipeline_on=False, capacity=0), run("fifo", policy="fifo"),
            run("lfu", policy="lfu"), run("bc4_bm2", b_c=4, b_m=2),
            run("cap2_lfu_bc3", capacity=2, policy="lfu", b_c=3, b_m=5),
            run("fixed_anchor", anchor="fixed_first")]


def c2_runs():
    return [run("lru", capacity=32, b_c=100, b_m=10), run("fifo", capacity=32, policy="fifo", b_c=100, b_m=10),
            run("lfu", capacity=32, policy="lfu", b_c=100, b_m=10),
            run("lru_nopipe", capacity=32, b_c=100, b_m=10, pipeline_on=False),
            run("lru_small", capacity=8, b_c=10, b_m=4)]


CACHE_TOKEN_COUNTS = [10 + 3 * i for i in range(16)]


def cache_cases():
    rng = SeededRng(0xCAC4E)
    cases = []
    for pol in ("lru", "fifo", "lfu"):
        for cap in (0, 1, 2, 3, 5, 8):
            ops = []
            for _ in range(600):
                if rng.next_below(5) == 0:
                    ops.append({"prefetch": [int(rng.next_below(12)) for _ in range(1 + rng.next_below(3))]})
                else:
                    ops.append({"get": int(rng.next_below(4) if rng.next_below(3) == 0 else rng.next_below(16))})
            cases.append({"capacity": cap, "policy": pol, "ops": ops})
    return cases


def run_batch_scenarios():
    rng = SeededRng(0x51AA)
    scen = []
    for _ in range(24):
        universe = 4 + rng.next_below(20)
        counts = [5 + int(rng.next_below(120)) for _ in range(universe)]
        qs = []
        for i in range(1 + rng.next_below(60)):
            ts = []
            for _ in range(rng.next_below(6)):
                t = int(rng.next_below(universe))
                if t not in ts:
                    ts.append(t)
            qs.append({"id": "q%d" % i, "tables": ts, "query_tokens": 1 + int(rng.next_below(50))})
        runs = []
        for k in range(3):
            runs.append({"name": "r%d" % k, "rerank_on": bool(rng.next_below(2)), "pipeline_on": bool(rng.next_below(2)),
                         "capacity": int(rng.next_below(10)) if rng.next_below(4) else 0,
                         "policy": ["lru", "fifo", "lfu"][rng.next_below(3)],
                         "b_c": 1 + int(rng.next_below(8)), "b_m": 1 + int(rng.next_below(8)),
                         "seed": int(rng.next_below(100)), "anchor": "seeded",
                         "cost": {"compute_per_token": 0.001 * rng.next_below(50),
                                  "load_per_token": 0.1 * rng.next_below(30),
                                  "switch_overhead": float(rng.next_below(10))}})
        scen.append({"token_counts": counts, "queries": qs, "runs": runs})
    return scen


def rerank_batches():
    rng = SeededRng(0x12E1)
    batches = []
    for b in range(200):
        n = 1 + rng.next_below(60)
        nb = 1 + rng.next_below(150)
        qs = [[int(rng.next_below(nb)) for _ in range(rng.next_below(6))] for _ in range(n)]
        batches.append({"n_bits": nb, "seed": b, "queries": qs, "mode": "seeded" if b % 3 else "fixed_first"})
    batches.append({"n_bits": 32, "seed": 0, "mode": "fixed_first",
                    "queries": [[0, 1, 2] if i % 2 == 0 else [20, 21] for i in range(20)]})
    return batches


def trie_inputs():
    rng = SeededRng(0x7121E)
    pats, used = [], set()
    while len(pats) < 40:
        seq = tuple(int(rng.next_below(6)) for _ in range(2 + rng.next_below(10)))
        if seq not in used:
            used.add(seq)
            pats.append(list(seq))
    pats.append(pats[0] + [5, 5, 5])  # nested longer serialization
    inputs = []
    for _ in range(60):
        n = 20 + rng.next_below(400)
        x = []
        while len(x) < n:
            if rng.next_below(6) == 0:
                x += pats[rng.next_below(len(pats))]
            else:
                x.append(int(rng.next_below(6)))
        inputs.append(x[:n])
    inputs += [[], [5], pats[0], pats[0] + [5, 5], pats[-1]]
    return pats, inputs


def attention_cases():
    cases = []
    for k in range(4):
        cases.append({"corpus_seed": 100 + k, "n_tables": 6, "max_group": 4, "min_tokens": 8, "max_tokens": 30,
                      "vocab": 64, "weight_seed": 1 + k, "order_seed": 7 + 31 * k, "double": k >= 2,
                      "query_tokens": list(range(3, 3 + 5 + k))})
    cases.append({"corpus_seed": 555, "n_tables": 5, "max_group": 3, "min_tokens": 8, "max_tokens": 20,
                  "vocab": 64, "weight_seed": 9, "order_seed": 3, "num_layers": 1, "num_heads": 2, "head_dim": 32,
                  "double": True, "query_tokens": [1, 2, 3]})
    return cases


RNG_TRIPLES = [[1, 2, 3], [0, 0, 0], [1, 8 * 131, 7], [42, 6 * 131 + 1, 123456789], [2**63 + 5, 2**40, 2**33 + 1]]
RNG_SEEDS = [0, 1, 7, 0x12E1, 2**64 - 1]
ROTARY_CASES = [{"heads": 4, "head_dim": 16, "positions": [0, 1, 2, 5, 100, 4097, -3], "seed": 3, "base": 10000.0},
                {"heads": 2, "head_dim": 8, "positions": list(range(20)), "seed": 4, "base": 500.0}]
