"""NVLink peer KV fetch with two ranks on one GPU: the CUDA IPC + residency-
directory protocol is the same whether the peer pool sits on another GPU (NVLink) or on this one
(one-GPU boxes run the multi-process path this way). Bars: landed bytes are the reference .kv
payload bit for bit whichever source served them; bytes come from the peer exactly while it has
the table published; serving with peer fetch leaves the served order, the per-record hit/miss/
evict trace, counters and first tokens identical to serving without it."""
import json
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here, os.path.join(os.path.dirname(here), "oracle")]
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_08743_b200 import native as N
    from golden_util import demo_path, load

    m = N.Model(dtype="f32", num_layers=2, num_heads=4, head_dim=16, vocab_size=330)
    s = N.Store(m, page_bytes=4096, n_pages=4096)
    for t in range(12):
        s.load_kv_file(demo_path("kv", "%d.kv" % t))
    payload = {t: open(demo_path("kv", "%d.kv" % t), "rb").read()[24:] for t in range(12)}
    blobs = [None] * world
    dist.all_gather_object(blobs, s.peer_export())
    s.peer_attach([b for r, b in enumerate(blobs) if r != rank])
    out = {}

    # ---- protocol: rank 1 publishes 0..5, rank 0 fetches everything
    if rank == 1:
        for t in range(6):
            s.peer_publish(t)
    dist.barrier()
    if rank == 0:
        out["published"] = []
        for t in range(12):
            got, from_peer = s.peer_fetch(t, len(payload[t]))
            out["published"].append([t, got.tobytes() == payload[t], from_peer, len(payload[t])])
    dist.barrier()
    if rank == 1:
        for t in range(6):
            s.peer_unpublish(t)
    dist.barrier()
    if rank == 0:
        got, from_peer = s.peer_fetch(0, len(payload[0]))
        out["revoked"] = [got.tobytes() == payload[0], from_peer]
    dist.barrier()

    # ---- race: rank 1 publishes and revokes tables in a loop while rank 0 fetches them; every
    # fetch must land the exact payload whichever source each CTA ended up reading
    if rank == 1:
        for it in range(120):
            t = it % 12
            s.peer_publish(t)
            s.peer_unpublish(t)
    else:
        ok, from_peer = True, 0
        for it in range(240):
            t = (it * 7) % 12
            got, fp = s.peer_fetch(t, len(payload[t]))
            ok &= got.tobytes() == payload[t]
            from_peer += fp
        out["race"] = [ok, from_peer]
    dist.barrier()

    # ---- serving: each rank serves its half of the demo chain with the other's plan
    g = load("demo64")["result"]
    qs = [(q["assembly_order"], q["remainder"]) for q in g["queries"][:64]]
    halves = [qs[:32], qs[32:]]
    mine, other = halves[rank], halves[1 - rank]
    kw = dict(rerank_on=0, capacity=4, b_c=2, b_m=1)
    base = s.serve(mine, **kw)
    s.peer_plan(0, other)
    dist.barrier()
    peer = s.serve(mine, peer_fetch=1, **kw)
    out["serve"] = {k: [base[k], peer[k]] for k in ("order", "trace", "counters", "argmax")}
    out["bytes"] = {k: peer[k] for k in ("h2d_bytes", "peer_routed_bytes", "peer_bytes", "peer_fallback_bytes")}
    out["base_h2d"] = base["h2d_bytes"]
    # routing: rank 0 serves cluster A (tables 0-3) then cluster B (4-7), rank 1 the reverse, so
    # each rank's switch-over misses find the other cluster resident on the peer (the host-side
    # residency directory routes them to the peer path)
    qa = [([0, 1, 2, 3], r) for _, r in qs[:8]]
    qb = [([4, 5, 6, 7], r) for _, r in qs[8:16]]
    lead, peer_batch = (qa + qb, qb + qa) if rank == 0 else (qb + qa, qa + qb)
    kw2 = dict(rerank_on=0, capacity=4, b_c=2, b_m=1)
    s.peer_plan(0, peer_batch)
    dist.barrier()
    base2 = s.serve(lead, **kw2)
    dist.barrier()
    shifted = s.serve(lead, peer_fetch=1, **kw2)
    out["shifted"] = {k: shifted[k] for k in ("h2d_bytes", "peer_routed_bytes", "peer_bytes", "peer_fallback_bytes")}
    out["shifted_same"] = all(base2[k] == shifted[k] for k in ("order", "trace", "counters", "argmax"))
    out["shifted_base_h2d"] = base2["h2d_bytes"]
    out["free_pages"] = s.info()["free_pages"]
    json.dump(out, open(os.path.join(out_dir, "rank%d.json" % rank), "w"))
    dist.barrier()
    s.close()
    m.close()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks(tmp_path_factory):
    import torch.multiprocessing as mp
    d = tmp_path_factory.mktemp("peer")
    mp.spawn(_worker, args=(2, _free_port(), str(d)), nprocs=2, join=True)
    return [json.load(open(d / ("rank%d.json" % r))) for r in range(2)]


def test_peer_fetch_bytes_and_sources(two_ranks):
    r0 = two_ranks[0]
    for t, exact, from_peer, n in r0["published"]:
        assert exact, t
        assert from_peer == (n if t < 6 else 0), (t, from_peer, n)
    exact, from_peer = r0["revoked"]
    assert exact and from_peer == 0  # a revoked entry is never read
    assert r0["race"][0]  # bytes exact under concurrent publish/revoke


def test_peer_fetch_leaves_trace_and_first_tokens_unchanged(two_ranks):
    for r in two_ranks:
        for k, (base, peer) in r["serve"].items():
            assert base == peer, k
        b = r["bytes"]
        assert b["h2d_bytes"] + b["peer_routed_bytes"] == r["base_h2d"]
        assert b["peer_bytes"] + b["peer_fallback_bytes"] == b["peer_routed_bytes"]
        assert r["free_pages"] == 4096
        assert r["shifted_same"]
        b = r["shifted"]
        assert b["h2d_bytes"] + b["peer_routed_bytes"] == r["shifted_base_h2d"]
        assert b["peer_bytes"] + b["peer_fallback_bytes"] == b["peer_routed_bytes"]
    for r in two_ranks:
        assert r["shifted"]["peer_routed_bytes"] > 0, r["shifted"]
