"""The bench's N > 1 path end to end (the driver's scaling run: torchrun, one process per GPU,
global rerank on every rank, request slices, NVLink peer fetch attach, max-over-ranks timing),
exercised with two ranks sharing GPU 0 (TKV_BENCH_ONE_DEVICE; gloo replaces NCCL, which refuses
two ranks on one device) and a 2-layer model so it runs in about a minute."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_line():
    env = dict(os.environ, TKV_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
           "1", "--warmup", "1", "--layers", "2", "--queries", "200", "--nocache-queries", "20", "--pool-pages", "2048"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["kv_load"]["peer_fetch"] == "on"
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
