"""Multi-process (gloo, world size 2) check of the N>1 request partitioning on CPU: both ranks
derive the same global chain, their slices are disjoint, cover every query, keep chain order,
and each rank's cache trace is the reference trace of its own slice (rerank off)."""
import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import load


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_08743_b200 import native as N
    from paper_2601_08743_b200 import sharding as S
    g = load("c2")["result"]
    sets = [q["assembly_order"] for q in g["queries"]]
    order = S.global_order(sets, len(g["table_tokens"]), seed=1)
    mine = S.rank_slice(order, rank, world)
    counts = [len(t) for t in g["table_tokens"]]
    qs = [{"id": g["queries"][i]["query_id"], "tables": sets[i], "query_tokens": g["queries"][i]["query_token_count"]}
          for i in mine]
    run = {"name": "r", "rerank_on": False, "pipeline_on": True, "capacity": 32, "policy": "lru", "b_c": 100, "b_m": 10,
           "seed": 1, "cost": {"compute_per_token": 0.01, "load_per_token": 1.0, "switch_overhead": 5.0}}
    res = N.run_batch_json({"token_counts": counts, "queries": qs, "runs": [run]})["r"]
    gathered = [None] * world
    dist.all_gather_object(gathered, {"order": order, "slice": mine, "counters": res["report"]["hits"]})
    if rank == 0:
        json.dump({"gathered": gathered}, open(os.path.join(out_dir, "out.json"), "w"))
    json.dump({"slice": mine, "trace": res["trace"], "report": res["report"]},
              open(os.path.join(out_dir, "rank%d.json" % rank), "w"))
    dist.destroy_process_group()


def test_two_rank_request_partition(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    gathered = json.load(open(tmp_path / "out.json"))["gathered"]
    assert gathered[0]["order"] == gathered[1]["order"]  # same chain on every rank
    order = gathered[0]["order"]
    s0, s1 = gathered[0]["slice"], gathered[1]["slice"]
    assert s0 + s1 == order and not set(s0) & set(s1) and sorted(order) == list(range(len(order)))
    # each rank's trace == the oracle's run_batch of that slice with rerank off
    import tkv_oracle as O
    g = load("c2")["result"]
    counts = [len(t) for t in g["table_tokens"]]
    for r in range(world):
        mine = json.load(open(tmp_path / ("rank%d.json" % r)))
        recs = [(g["queries"][i]["query_id"], g["queries"][i]["assembly_order"], g["queries"][i]["query_token_count"])
                for i in mine["slice"]]
        rep = O.run_batch(recs, counts, len(counts), {"rerank_on": False, "capacity": 32, "policy": "lru",
                                                      "b_c": 100, "b_m": 10}, (0.01, 1.0, 5.0))
        assert [rep[k] for k in ("hits", "misses", "swaps", "prefetch_loads")] == \
               [mine["report"][k] for k in ("hits", "misses", "swaps", "prefetch_loads")]
        assert rep["total_ttft"] == pytest.approx(mine["report"]["total_ttft"], rel=1e-12)


def test_slice_bounds_cover_uneven_sizes():
    from paper_2601_08743_b200.sharding import slice_bounds
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            spans = [slice_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
