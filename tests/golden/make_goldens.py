#!/usr/bin/env python3
"""Regenerates every golden fixture in tests/golden/ from the UNCHANGED reference.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/make_goldens.py
The reference library is driven through oracle/_ref/golden_dump (oracle/tools/golden_dump.cpp).
Inputs come from tests/golden_inputs.py (deterministic SeededRng streams), so rerunning
reproduces the committed files and the tests rebuild the very same inputs.
"""
import gzip
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import golden_inputs as GI  # noqa: E402
from paper_2601_08743_b200 import workloads as W  # noqa: E402

TOOL = os.path.join(ROOT, "oracle", "_ref", "golden_dump")
REF_DATA = "/root/reference/proj/data"
TMP = "/tmp/tkv_goldens"


def dump(cmd, inp, name, blob=False):
    os.makedirs(TMP, exist_ok=True)
    ip = os.path.join(TMP, name + ".in.json")
    with open(ip, "w") as f:
        json.dump(inp, f)
    args = [TOOL, cmd, ip, os.path.join(HERE, name + ".json")]
    if blob:
        args.append(os.path.join(HERE, name + ".bin"))
    subprocess.run(args, check=True)
    print("wrote", name)


def demo_files():
    d = os.path.join(HERE, "demo")
    os.makedirs(d, exist_ok=True)
    schema = W.dump_schema_corpus(W.demo_schema())
    workload = W.dump_workload(W.demo_workload(200))
    if os.path.isdir(REF_DATA):  # pin our generator to the reference's committed demo data
        assert schema == open(os.path.join(REF_DATA, "demo_schema.json")).read()
        assert workload == open(os.path.join(REF_DATA, "demo_workload.jsonl")).read()
    open(os.path.join(d, "demo_schema.json"), "w").write(schema)
    open(os.path.join(d, "demo_workload.jsonl"), "w").write(workload)
    open(os.path.join(d, "demo_config.json"), "w").write(json.dumps(W.DEMO_CONFIG, indent=2) + "\n")
    return os.path.join(d, "demo_schema.json"), os.path.join(d, "demo_workload.jsonl")


def main():
    sp, wp = demo_files()
    kv_dir = os.path.join(TMP, "demo_kv")
    shutil.rmtree(kv_dir, ignore_errors=True)
    dump("engine", {"schema_path": sp, "workload_path": wp, "n_queries": 64, "kv_dir": kv_dir,
                    "runs": GI.demo_runs(), "tensors": {"assemble_queries": 6, "hidden_queries": 64}},
         "demo64", blob=True)
    # the reference .kv payloads themselves: ground truth for "loaded KV bytes"
    out_kv = os.path.join(HERE, "demo", "kv")
    shutil.rmtree(out_kv, ignore_errors=True)
    shutil.copytree(kv_dir, out_kv)
    dump("engine", {"schema_path": sp, "workload_path": wp, "n_queries": 200, "runs": GI.demo_runs()[:5]}, "demo200")

    tabs, ents, _ = W.spider_like(W.CONFIGS["c2"])
    csp, cwp = W.write_corpus(os.path.join(TMP, "c2"), tabs, ents)
    dump("engine", {"schema_path": csp, "workload_path": cwp, "n_queries": 1000, "runs": GI.c2_runs()}, "c2")

    dump("cache_ops", {"token_counts": GI.CACHE_TOKEN_COUNTS, "cases": GI.cache_cases()}, "cache_ops")

    merged = []
    for sc in GI.run_batch_scenarios():
        dump("run_batch", sc, "run_batch_tmp")
        p = os.path.join(HERE, "run_batch_tmp.json")
        merged.append({"input": sc, "output": json.load(open(p))["result"]})
        os.remove(p)
    json.dump(merged, open(os.path.join(HERE, "run_batch.json"), "w"), indent=0)

    dump("rerank", {"batches": GI.rerank_batches()}, "rerank")
    pats, inputs = GI.trie_inputs()
    dump("trie", {"patterns": pats, "inputs": inputs}, "trie")
    dump("attention", {"cases": GI.attention_cases()}, "attention", blob=True)
    dump("rng", {"mix3": GI.RNG_TRIPLES, "seeded": GI.RNG_SEEDS}, "rng")
    dump("rotary", {"cases": GI.ROTARY_CASES}, "rotary", blob=True)


def compress_large(limit=256 * 1024):
    for name in os.listdir(HERE):
        path = os.path.join(HERE, name)
        if name.endswith(".json") and os.path.getsize(path) > limit:
            with open(path, "rb") as f, open(path + ".gz", "wb") as raw:
                with gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as g:
                    g.write(f.read())
            os.remove(path)


if __name__ == "__main__":
    main()
    compress_large()
