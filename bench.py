#!/usr/bin/env python3
"""TableCache B200 online-path benchmark (BASELINE.json metric: p50 TTFT and prefill queries/s vs
no-cache prefill; KV load GB/s vs PCIe).

Workload (default `--config c4`, the largest single-GPU configuration of BASELINE.json: configs[2]
prefixes with configs[3]'s capacity pressure): 16 databases / 256 tables of 256-512 tokens,
Zipf popularity, 500 queries per GPU with 8-16 tables each (~4.7k-token cached prefixes) and
32-128 suffix tokens; Llama-3-8B-shaped decoder (32 layers, 32 q / 8 kv heads x 128, SwiGLU
14336, RMSNorm, vocab 128256), random (counter-hash) weights, bf16; table KV precomputed offline
on the GPU into a pinned host arena; LRU fast tier of C = 32 tables over a paged HBM pool (every
window evicts); rerank on; b_c = 100, b_m = 10. `--config c1|c2|c3|c5` selects the others.

One step = one cold-cache batch through the whole online path: global rerank, schedule,
canonical cache trace, H2D page copies of every miss/prefetch from the pinned arena, prefix
gather+RoPE and the batched suffix prefill with the first-token head per window.
`value` = queries/s from CUDA-event makespans (max over ranks); `e2e` = the same batch through
the C ABI from prompt TEXT (host analysis + D2H of first tokens) by wall clock.
Multi-GPU (torchrun): one process per GPU, the globally reranked order is cut into contiguous
slices (weak scaling: the per-GPU query count is fixed), no collective on the data path.
`--impl reference`: the unchanged reference library (oracle/_ref) on the host cores, same metric.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LLAMA8B = dict(num_layers=32, num_heads=32, num_kv_heads=8, head_dim=128, ffn_dim=14336, vocab_size=128256,
               mlp="swiglu", norm="rms")


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def pct(v, p):
    v = sorted(v)
    if not v:
        return 0.0
    i = p * (len(v) - 1)
    lo = int(i)
    hi = min(lo + 1, len(v) - 1)
    return v[lo] + (v[hi] - v[lo]) * (i - lo)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in self.rows if r[7] not in ("0", "[N/A]")] or self.rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows), "samples_under_load": len(loaded)}


def build_workload(cfg_name, n_queries_total):
    from paper_2601_08743_b200 import workloads as W
    if cfg_name == "c1":  # the reference default: the 12-table demo schema, gen_demo queries
        return W.demo_schema(), W.demo_workload(n_queries_total)
    spec = W.CONFIGS["c3" if cfg_name == "c4" else cfg_name]  # c4 = c3 prefixes + capacity pressure
    spec = W.SpiderSpec(**{**spec.__dict__, "n_queries": n_queries_total})
    tables, entries, _ = W.spider_like(spec)
    return tables, entries


METRIC = "p50 TTFT and prefill queries/sec vs no-cache prefill; KV load GB/s vs PCIe"  # BASELINE.json metric, both arms


def ref_serve_sample(tables, entries, threads):
    """The UNCHANGED reference library's cached serving path (oracle/_ref/ref_bench serve) on
    this host: the first `threads` prompts of the workload, one per core, each through the
    reference's own analyze_query + assembly_order + MemorySlowTier loads + assemble +
    query_attend of ONE layer at the served width (hidden 4096, 32 heads x 128; reference MHA /
    LayerNorm / SiLU-4h arithmetic, 12 h^2 MACs per token-layer vs the served GQA/SwiGLU 13 h^2).
    The per-layer part is extrapolated x32 layers; analysis is not. Nothing here loads libtkv.so."""
    import tempfile
    from paper_2601_08743_b200 import workloads as W  # pure Python, no native code
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    L = LLAMA8B["num_layers"]
    with tempfile.TemporaryDirectory() as d:
        sp, wp = W.write_corpus(d, tables, entries[:threads])
        out = subprocess.run([exe, "serve", sp, wp, str(threads), "32", "128", str(threads)], capture_output=True,
                             text=True, check=True)
    r = json.loads(out.stdout)
    per_q = [a + L * l for a, l in zip(r["analysis_s"], r["layer_s"])]  # extrapolated service time per query
    qps = threads / statistics.mean(per_q)  # `threads` cores serving queries back to back
    return {"qps": qps, "wave_wall_s": r["wall_s"], "per_query_s": per_q, "raw": r,
            "sample": "first %d prompts of the workload, one per core: reference analyze_query + assembly_order + "
                      "loads + assemble + query_attend of 1 layer at hidden 4096 (MHA/LN/SiLU-4h; 12h^2 MACs per "
                      "token-layer vs 13h^2 served), layer part x%d (extrapolated); mean prefix %.0f / suffix %.0f "
                      "tokens" % (threads, L, statistics.mean(r["nctx"]), statistics.mean(r["nq"]))}


def cpu_info():
    import multiprocessing
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return multiprocessing.cpu_count(), model


def reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU path (the unchanged library, oracle/_ref) on this
    host's cores for the same workload, metric and unit; rank 0 only. No libtkv.so is loaded.

    c1: ref_bench demo (assemble + query_attend of every demo query, measured in full) once per
    step. c2-c5: one bounded wave (one query per core, see ref_serve_sample) — a full query at
    hidden 4096 costs the reference minutes per core, so the timed region is that single wave and
    ms_per_step = wave wall / steps; the x32-layer extrapolation is in its own keys."""
    if rank != 0:
        return
    cores, cpu_model = cpu_info()
    tables, entries = build_workload(args.config, args.queries)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    base = {"metric": METRIC, "unit": "queries/s", "impl": "reference", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "data": "synthetic", "cpu": {"cores": cores, "model": cpu_model}}
    if args.config == "c1":
        walls, last = [], None
        for step in range(args.warmup + args.steps):
            last = cpu_baseline_demo(tables, entries, cores)
            if step >= args.warmup:
                walls.append(len(entries) / last["value"])
        qps = len(entries) * len(walls) / sum(walls)
        line = dict(base, value=qps, ms_per_step=sum(walls) / len(walls) * 1e3, dtype="f32",
                    config={"workload": workload_name(args, len(tables), len(entries))},
                    p50_ttft_ms=last["p50_query_ms"], p99_ttft_ms=last["p99_query_ms"],
                    cpu_baseline=dict(last, value=qps))
    else:
        s = ref_serve_sample(tables, entries, cores)
        wall = s["wave_wall_s"]
        line = dict(base, value=s["qps"], ms_per_step=wall / args.steps * 1e3, dtype="f32",
                    config={"workload": workload_name(args, len(tables), len(entries))},
                    timed_region="one wave of %d queries (one per core) x 1 layer, %.1f s; ms_per_step = wave wall / "
                                 "steps" % (cores, wall),
                    extrapolated_ms_per_step=wall * LLAMA8B["num_layers"] / args.steps * 1e3,
                    p50_query_latency_ms_extrapolated=pct(s["per_query_s"], 0.5) * 1e3,
                    p99_query_latency_ms_extrapolated=pct(s["per_query_s"], 0.99) * 1e3,
                    cpu_baseline={"value": s["qps"], "unit": "queries/s", "cores": cores, "kind": "reference",
                                  "sample": s["sample"]})
    line["e2e"] = {"value": line["value"], "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    print(json.dumps(line))


def workload_name(args, n_tables, n_queries):
    from paper_2601_08743_b200 import workloads as W
    if args.config == "c1":
        arith = ("bf16 on the tensor-core kernels" if getattr(args, "dtype", None) == "bf16" else
                 "f32 with the reference arithmetic")
        return ("c1 reference default: 12-table demo schema, %d gen_demo queries, the reference model (2 layers, "
                "4 heads x 16, LayerNorm, SiLU FFN) in %s" % (n_queries, arith))
    spec = W.CONFIGS["c3" if args.config == "c4" else args.config]
    label = {"c2": "c2 Spider-like", "c3": "c3 ~4k-token prefixes (C >= working set)",
             "c4": "c4 = c3 prefixes + capacity pressure (evictions every window)",
             "c5": "c5 BIRD-like wide schemas"}[args.config]
    return ("%s: %d DBs / %d tables, Zipf(1.1), %d queries per GPU; Llama-3-8B-shaped (%d layers, 32q/8kv x128, "
            "SwiGLU 14336, RMSNorm, vocab 128256), random weights" % (label, spec.n_db, n_tables, n_queries,
                                                                     args.layers))


def cpu_baseline_demo(tables, entries, threads):
    """C1: the reference's own demo path (assemble + query_attend per query, the unchanged library)
    on `threads` host cores — measured in full, nothing extrapolated."""
    import tempfile
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    from paper_2601_08743_b200 import workloads as W
    with tempfile.TemporaryDirectory() as d:
        sp, wp = W.write_corpus(d, tables, entries)
        out = subprocess.run([exe, "demo", sp, wp, str(len(entries)), str(threads)], capture_output=True, text=True,
                             check=True)
    r = json.loads(out.stdout)
    return {"value": r["cached_qps"], "unit": "queries/s", "cores": threads, "kind": "reference",
            "sample": "all %d demo queries, reference assemble + query_attend (f32, double accumulate), %d threads; "
                      "no-cache prefill %.1f queries/s" % (len(entries), threads, r["nocache_qps"]),
            "p50_query_ms": r["cached_p50_ms"], "p99_query_ms": r["cached_p99_ms"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE configs: c1 = reference default (tiny model, f32 reference arithmetic, demo); "
                         "c2 Spider-like; c3 ~4k-token prefixes; c4 = c3 with capacity pressure (default: the "
                         "largest single-GPU config); c5 BIRD-like <=16k prefixes")
    ap.add_argument("--queries", type=int, default=None, help="queries per GPU (c2: 1000, c3/c4: 500, c5: 1250)")
    ap.add_argument("--layers", type=int, default=LLAMA8B["num_layers"])
    ap.add_argument("--capacity", type=int, default=None, help="cache entries (default 32; c1: 6, c3: 256, c5: 64)")
    ap.add_argument("--policy", default="lru", choices=["lru", "fifo", "lfu"])
    ap.add_argument("--pool-pages", type=int, default=12288, help="2 MiB HBM pages in the fast-tier pool")
    ap.add_argument("--b_c", type=int, default=None, help="default 100 (c1: 1)")
    ap.add_argument("--b_m", type=int, default=None, help="default 10 (c1: 1)")
    ap.add_argument("--copy-engine", type=int, default=0, help="0: DMA copy engines, 1: SM 16-byte copy kernel")
    ap.add_argument("--sm-copy-ctas", type=int, default=16)
    ap.add_argument("--nocache-queries", type=int, default=None,
                    help="queries in the no-cache comparison (c2: 300, c3/c4: 100, c5: 50)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dtype", default=None, choices=["f32", "bf16"],
                    help="c1 only: f32 = the reference arithmetic on the SIMT parity kernels (default), bf16 = the "
                         "same reference model on the tensor-core kernels (tcgen05 GEMMs, mma.sync head_dim-16 "
                         "attention); c2-c5 are always bf16")
    ap.add_argument("--shard", default="contiguous", choices=["interleave", "contiguous"],
                    help="N>1: deal the global chain out in window-sized chunks (interleave) or contiguous slices")
    ap.add_argument("--peer-fetch", type=int, default=None,
                    help="NVLink peer KV fetch between ranks (default: on when N > 1)")
    args = ap.parse_args()

    c1 = args.config == "c1"
    args.dtype = (args.dtype or "f32") if c1 else "bf16"
    c1_simt = c1 and args.dtype == "f32"
    if args.capacity is None:
        args.capacity = {"c1": 6, "c3": 256, "c5": 64}.get(args.config, 32)
    if args.queries is None:
        args.queries = {"c1": 64, "c2": 1000, "c5": 1250}.get(args.config, 500)
    if args.nocache_queries is None:
        args.nocache_queries = {"c1": 64, "c2": 300, "c5": 50}.get(args.config, 100)
    if args.b_c is None:
        args.b_c = 1 if c1 else 100
    if args.b_m is None:
        args.b_m = 1 if c1 else 10
    if c1:
        args.queries = min(args.queries, 64)
    args.nocache_queries = min(args.nocache_queries, args.queries)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if os.environ.get("TKV_BENCH_ONE_DEVICE"):  # test hook: every rank on GPU 0 (one-GPU boxes)
        local = 0
    peer_on = (world > 1) if args.peer_fetch is None else bool(args.peer_fetch)

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("TKV_BENCH_ONE_DEVICE"):  # NCCL refuses two ranks on one GPU
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if os.environ.get("TKV_BENCH_ONE_DEVICE") else "cuda"
    from paper_2601_08743_b200 import native as N
    from paper_2601_08743_b200 import workloads as W

    # ---- setup (untimed): corpus, engine, device model, offline table encode into the arena
    tables, entries = build_workload(args.config, args.queries * world)
    eng = N.Engine(corpus_json=W.dump_schema_corpus(tables))
    mk = dict(LLAMA8B, num_layers=args.layers)
    t0 = time.time()
    if c1:  # the reference's own model (model.hpp defaults) in f32 with the reference arithmetic
        model = N.Model(dtype=args.dtype, device=local, num_layers=2, num_heads=4, head_dim=16,
                        vocab_size=eng.info["vocab_size"])
        store = N.Store(model, page_bytes=64 << 10, n_pages=2048)
    else:
        model = N.Model(dtype="bf16", device=local, **mk)
        store = N.Store(model, page_bytes=2 << 20, n_pages=args.pool_pages)
    store.precompute(eng)
    store.bind_engine(eng)
    setup_s = time.time() - t0
    # offline encode measured (engine.cpp:83-112): the same precompute again (the images
    # are rewritten with identical bytes), device time incl. the D2H into the arena, GEMMs timed
    enc = store.precompute(eng, timed=True)
    analyzed = [eng.analyze(text, qid) for qid, text in entries]
    n_bits = len(tables)
    pcie = N.measure_h2d(256 << 20, 5, local)

    from paper_2601_08743_b200 import sharding as S

    def global_order():
        """The global rerank chain (bit-exact with the host chain), computed ONCE per step: rank 0
        runs it on its GPU (distinct table sets, one thread-block cluster) and broadcasts the
        permutation; every rank then takes its contiguous slice."""
        if world == 1:
            return N.rerank_device([a["assembly_order"] for a in analyzed], n_bits, seed=1, device=local)
        t = torch.empty(len(analyzed), dtype=torch.int32, device=coll_dev)
        if rank == 0:
            t.copy_(torch.tensor(N.rerank_device([a["assembly_order"] for a in analyzed], n_bits, seed=1, device=local),
                                 dtype=torch.int32))
        torch.distributed.broadcast(t, 0)
        return t.tolist()

    chunk = args.b_c if args.shard == "interleave" else None

    def my_slice(order):
        return S.rank_slice(order, rank, world, chunk)

    # NVLink peer fetch: exchange pool/directory IPC blobs; peer slot i = the i-th other rank
    peer_status = "off"
    others = [r for r in range(world) if r != rank]
    if peer_on and world > 1:
        try:
            blob = store.peer_export()
            blobs = [None] * world
            torch.distributed.all_gather_object(blobs, blob)
            store.peer_attach([blobs[r] for r in others])
            peer_status = "on"
        except Exception as e:  # noqa: BLE001  (reported in the JSON line; serving proceeds from host)
            peer_status = "unavailable: %s" % str(e).splitlines()[0][:200]
        flags = [None] * world
        torch.distributed.all_gather_object(flags, peer_status == "on")
        if not all(flags):
            peer_status = peer_status if peer_status != "on" else "off (a peer failed to attach)"

    opts = N.serve_options(rerank_on=0, pipeline_on=1, capacity=args.capacity, policy=args.policy, b_c=args.b_c,
                           b_m=args.b_m, copy_engine=args.copy_engine, sm_copy_ctas=args.sm_copy_ctas, time_kernels=1,
                           peer_fetch=int(peer_status == "on"))

    rerank_ms = []

    def step():
        tr = time.perf_counter()
        order = global_order()  # global rerank inside the step, on every rank (counted in the step time)
        rerank_ms.append((time.perf_counter() - tr) * 1e3)
        sl = my_slice(order)
        qs = [(analyzed[i]["assembly_order"], analyzed[i]["remainder"]) for i in sl]
        if peer_status == "on":  # every peer's slice: the host-side residency prediction
            for slot, r in enumerate(others):
                store.peer_plan(slot, [(analyzed[i]["assembly_order"], len(analyzed[i]["remainder"]))
                                       for i in S.rank_slice(order, r, world, chunk)])
        return store.serve(qs, opts)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    barrier()
    if os.environ.get("TKV_NCU"):
        # profiling run (never a bench number): capture exactly one serving step under ncu
        # --profile-from-start off, then exit
        torch.cuda.cudart().cudaProfilerStart()
        step()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        print(json.dumps({"profiled": "one serving step", "queries": args.queries}))
        return
    results = []
    with ClockSampler(local) as clocks:
        tw = time.perf_counter()
        for _ in range(args.steps):
            results.append(step())
        barrier()
        wall = time.perf_counter() - tw
    timed_rerank_ms = rerank_ms[-args.steps:]
    dev_ms = sum(r["makespan_ms"] for r in results) + sum(timed_rerank_ms)
    total_ms = dev_ms
    if world > 1:
        t = torch.tensor([dev_ms], device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    n_local = len(results[0]["order"])
    value = n_local * world * args.steps / (total_ms / 1e3)
    ttfts = [t for r in results for t in r["ttft_ms"]]
    h2d = sum(r["h2d_bytes"] for r in results) / args.steps
    copy_ms = sum(r["copy_busy_ms"] for r in results) / args.steps
    dem_b = sum(r["h2d_demand_bytes"] for r in results) / args.steps
    dem_ms = sum(r["copy_demand_ms"] for r in results) / args.steps
    # attention work of this rank's queries (algorithmic): per layer 4 * q_heads * head_dim FLOP per
    # (query row, visible key) and the cached prefix's K + V read once per (query, kv head)
    ttok = [len(x) for x in eng.info["table_tokens"]]
    attn_fl = attn_kv_b = 0.0
    if not c1:
        for i in my_slice(global_order()):
            p_ = sum(ttok[t] for t in analyzed[i]["assembly_order"])
            s_ = len(analyzed[i]["remainder"])
            attn_fl += 4.0 * mk["num_heads"] * mk["head_dim"] * s_ * (p_ + (s_ + 1) / 2.0) * mk["num_layers"]
            attn_kv_b += 2.0 * p_ * mk["num_kv_heads"] * mk["head_dim"] * 2 * mk["num_layers"]
    gemm_ms = sum(r["gemm_ms"] for r in results)
    gemm_fl = sum(r["gemm_flops"] for r in results)
    launches = sum(r["launches"] for r in results)

    # ---- e2e: prompt text in, first tokens out, through the C ABI (wall clock)
    # the user path: the rank's prompts in arrival order; serve_text reranks them itself
    e2e_texts = [entries[i][1] for i in sorted(my_slice(global_order()))]
    e2e_opts = N.serve_options(rerank_on=1, capacity=args.capacity, policy=args.policy, b_c=args.b_c, b_m=args.b_m,
                               time_kernels=int(os.environ.get("TKV_E2E_TIMED", "0")))
    for _ in range(args.warmup):
        store.serve_text(eng, e2e_texts, options=e2e_opts)
    barrier()
    e2e_steps = []
    with ClockSampler(local) as e2e_clocks:  # right after the timed steps: same thermal state
        te = time.perf_counter()
        for _ in range(args.steps):  # prompt text in (host analysis, H2D), first tokens out (D2H), per step
            tc = time.perf_counter()
            e2e_res = store.serve_text(eng, e2e_texts, options=e2e_opts)
            e2e_last_wall = time.perf_counter() - tc
            e2e_steps.append([round(e2e_last_wall * 1e3, 1), round(e2e_res["makespan_ms"], 1), round(e2e_res["wall_ms"], 1)])
        e2e_s = (time.perf_counter() - te) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device=coll_dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_h2d = e2e_res["h2d_bytes"] + e2e_res["meta_bytes"] + sum(len(x.encode()) for x in e2e_texts)
    e2e_d2h = 4 * len(e2e_res["argmax"])

    # ---- no-cache baseline on the same kernels (block-masked full prefill), subset
    nc_n = min(args.nocache_queries, n_local)
    sl = my_slice(global_order())[:nc_n]
    qs_nc = [(analyzed[i]["assembly_order"], analyzed[i]["remainder"]) for i in sl]
    if nc_n:
        nc_opts = N.serve_options(rerank_on=0, capacity=args.capacity, b_c=args.b_c, b_m=args.b_m, nocache=1)
        store.serve(qs_nc, nc_opts)  # warm-up
        nc = store.serve(qs_nc, nc_opts)
        cached_sub = store.serve(qs_nc, N.serve_options(rerank_on=0, capacity=args.capacity, policy=args.policy,
                                                        b_c=args.b_c, b_m=args.b_m))
    # global rerank at the 8-GPU job size: the chain over 8x this rank's queries on
    # one GPU, as rank 0 computes it for an 8-GPU run (c5: 10k queries), device-timed by wall clock
    rr8 = None
    if rank == 0 and not c1:
        _, entries8 = build_workload(args.config, args.queries * 8)
        sets8 = [eng.analyze(text, qid)["assembly_order"] for qid, text in entries8]
        N.rerank_device(sets8, n_bits, seed=1, device=local)  # warm-up
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            N.rerank_device(sets8, n_bits, seed=1, device=local)
            ts.append((time.perf_counter() - t) * 1e3)
        rr8 = {"queries": len(sets8), "ms": min(ts), "ms_all": [round(x, 2) for x in ts],
               "breakdown_last_call": N.rerank_device_stats(),
               "what": "rerank_device wall clock: incidence packing + host reduction to distinct table sets + H2D + "
                       "the cluster chain kernel (CUDA events: kernel_ms) + D2H + expansion"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_tf = peaks.get("bf16_tflops_sustained", 1400.0)
    tpath = os.path.join(ROOT, "profiles", "r2", "roofline_traffic.json")
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r1_roofline_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    achieved_tf = gemm_fl / (gemm_ms / 1e3) / 1e12 if gemm_ms else 0.0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores, cpu_model = cpu_info()
        try:
            if c1:
                cpu = cpu_baseline_demo(tables, entries, cores)
            else:
                smp = ref_serve_sample(tables, entries, cores)
                cpu = {"value": smp["qps"], "unit": "queries/s", "cores": cores, "kind": "reference",
                       "sample": smp["sample"], "wave_wall_s": smp["wave_wall_s"],
                       "p50_query_latency_ms_extrapolated": pct(smp["per_query_s"], 0.5) * 1e3}
            cpu["cpu_model"] = cpu_model
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unavailable": str(e)}
    nc_p50, c_p50 = (pct(nc["ttft_ms"], 0.5), pct(cached_sub["ttft_ms"], 0.5)) if nc_n else (None, None)
    line = {
        "metric": METRIC,
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": workload_name(args, len(tables), n_local),
                   "cache": "%s C=%d tables, b_c=%d, b_m=%d, rerank on, %s HBM pages"
                            % (args.policy.upper(), args.capacity, args.b_c, args.b_m, "64 KiB" if c1 else "2 MiB"),
                   "parallelism": "dp%d (request shares of the global rerank: %s)" % (
                       world, "window-sized chunks dealt round-robin" if chunk and world > 1 else "contiguous slices"),
                   "l2": "small model: weights and KV stay L2-resident (a latency-bound parity config)" if c1 else
                         "inputs larger than L2 (16 GB weights streamed per window)"},
        "p50_ttft_ms": pct(ttfts, 0.5), "p99_ttft_ms": pct(ttfts, 0.99),
        "nocache": {"queries": nc_n, "p50_ttft_ms": nc_p50, "p99_ttft_ms": pct(nc["ttft_ms"], 0.99),
                    "qps": nc_n / (nc["makespan_ms"] / 1e3), "cached_p50_ttft_ms_same_subset": c_p50,
                    "cached_qps_same_subset": nc_n / (cached_sub["makespan_ms"] / 1e3),
                    "p50_ttft_reduction": nc_p50 / c_p50 if c_p50 else None,
                    "argmax_agreement": float(np.mean([a == b for a, b in zip(nc["argmax"], cached_sub["argmax"])]))}
                   if nc_n else {"queries": 0},
        "kv_load": {"bytes_per_step": h2d, "copy_busy_ms_per_step": copy_ms,
                    "demand_bytes_per_step": dem_b, "demand_copy_ms_per_step": dem_ms,
                    "gbs": dem_b / (dem_ms / 1e3) / 1e9 if dem_ms else None, "pcie_h2d_peak_gbs": pcie,
                    "frac_of_pcie": (dem_b / (dem_ms / 1e3) / 1e9) / pcie if dem_ms else None,
                    "gbs_definition": "demand-stream bytes / summed per-window spans of its back-to-back copies",
                    "copy_engine": ["dma", "sm-16B-kernel"][args.copy_engine],
                    "peer_fetch": peer_status,
                    "peer_routed_bytes_per_step": sum(r["peer_routed_bytes"] for r in results) / args.steps,
                    "peer_bytes_per_step": sum(r["peer_bytes"] for r in results) / args.steps,
                    "peer_fallback_bytes_per_step": sum(r["peer_fallback_bytes"] for r in results) / args.steps,
                    "hits_misses_swaps_prefetch": results[0]["counters"]},
        "roofline": {"bound": "latency", "kernel": "reference-precision SIMT forward (simt.cu)", "achieved": None,
                     "peak": None, "unit": None, "frac": None, "traffic": None,
                     "note": "c1 runs the reference's f32/double arithmetic for bit-level parity; tensor-core "
                             "rooflines are reported on c2-c5 and on c1 --dtype bf16"} if c1_simt else
                    {"bound": "tensor", "kernel": "gemm_tc (tcgen05 QKV/O/gate-up/down/head)",
                     "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf if peak_tf else None, "traffic": traffic.get("dram_bytes_per_launch"),
                     "traffic_source": traffic.get("source"), "traffic_algorithmic_bytes": traffic.get("algorithmic_bytes_per_launch"),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                     "share_of_step": gemm_ms / dev_ms if dev_ms else None},
        "gather": {"ms_per_step": sum(r["gather_ms"] for r in results) / args.steps,
                   "gbs": (sum(r["gather_bytes"] for r in results) / (sum(r["gather_ms"] for r in results) / 1e3) / 1e9
                           if sum(r["gather_ms"] for r in results) else None),
                   "peak_gbs": peaks.get("hbm_gbs"),
                   "bytes_definition": "slab mode only (TKV_PAGED_K=0): prefix rows x layers x kv_dim x 2 x (read + "
                                       "write element bytes); the default paged prefix runs no gather (0 ms)"},
        "global_rerank_ms_per_step": sum(timed_rerank_ms) / args.steps,
        "global_rerank_at_8x": rr8,
        "encode": {"what": "offline table encode (precompute_corpus) on the GPU: every group as one block-causal "
                           "sequence, packed into batched forwards, raw K/V straight into the pinned arena",
                   "groups": int(enc["groups"]), "tables": int(enc["tables"]), "tokens": int(enc["tokens"]),
                   "forwards": int(enc["forwards"]), "device_ms": enc["device_ms"],
                   "tokens_per_s": enc["tokens"] / (enc["device_ms"] / 1e3) if enc["device_ms"] else None,
                   "gemm_ms": enc["gemm_ms"], "attn_ms": enc["attn_ms"],
                   "gemm_tflops": enc["gemm_flops"] / (enc["gemm_ms"] / 1e3) / 1e12 if enc["gemm_ms"] else None,
                   "gemm_frac_of_peak": (enc["gemm_flops"] / (enc["gemm_ms"] / 1e3) / 1e12) / peak_tf
                   if enc["gemm_ms"] else None,
                   "flops_frac_of_peak_over_device_time": (enc["gemm_flops"] / (enc["device_ms"] / 1e3) / 1e12) / peak_tf
                   if enc["device_ms"] else None},
        "attention_ms_per_step": sum(r["attn_ms"] for r in results) / args.steps,
        "attention": {"kernel": "attn_tc5 (tcgen05/TMEM; paged prefix: K/V TMA'd from the pool pages, K rotated in smem)",
                      "ms_per_step": sum(r["attn_ms"] for r in results) / args.steps,
                      "tflops": attn_fl / (sum(r["attn_ms"] for r in results) / args.steps / 1e3) / 1e12
                      if not c1 and sum(r["attn_ms"] for r in results) else None,
                      "frac_of_bf16_peak": attn_fl / (sum(r["attn_ms"] for r in results) / args.steps / 1e3) / 1e12 / peak_tf
                      if not c1 and sum(r["attn_ms"] for r in results) else None,
                      "prefix_kv_gbs": attn_kv_b / (sum(r["attn_ms"] for r in results) / args.steps / 1e3) / 1e9
                      if not c1 and sum(r["attn_ms"] for r in results) else None,
                      "flops_per_step": attn_fl, "prefix_kv_bytes_per_step": attn_kv_b,
                      "definition": "flops = 4 * q_heads * head_dim * suffix * (prefix + (suffix+1)/2) * layers per "
                                    "query; bytes = the prefix's K and V (bf16) once per query and layer"},
        "e2e": {"value": len(e2e_texts) * world / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": e2e_h2d,
                "d2h_bytes_per_step": e2e_d2h, "p50_ttft_ms": pct(e2e_res["ttft_ms"], 0.5),
                "last_step_ms": {"prompt_analysis": e2e_res.get("analyze_ms"), "host_enqueue": e2e_res["host_ms"],
                                 "device_makespan": e2e_res["makespan_ms"], "serve_wall": e2e_res["wall_ms"],
                                 "call_wall": e2e_last_wall * 1e3},
                "steps_call_makespan_serve_ms": e2e_steps, "clocks": e2e_clocks.summary()},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "setup_s": setup_s, "wall_s_timed": wall,
    }
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
