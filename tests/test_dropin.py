"""Drop-in check: the reference's OWN test sources (proj/tests/unit/*.cpp and
proj/tests/acceptance/acceptance.cpp), unchanged, compiled against this repo's include/tablekv
headers + libtkv.so with a doctest-compatible shim (oracle/Makefile target `dropin`, built by
__graft_entry__.build() where /root/reference exists; the binaries travel to the GPU box).

Host suites run here; the attention-core and engine suites and the 9-criterion acceptance gate
drive the CUDA model (reference-precision kernels, GPU gather) and run on the B200.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "dropin_unit")
ACCEPT = os.path.join(ROOT, "oracle", "_ref", "dropin_acceptance")
DEMO = os.path.join(ROOT, "tests", "golden", "demo")

HOST_SUITES = ["schema-graph", "table-trie", "rotary", "table-kv-format", "tiered-cache", "rerank", "tokenizer",
               "pipeline"]
GPU_SUITES = ["attention-core", "engine"]

needs_bin = pytest.mark.skipif(not os.path.exists(UNIT), reason="dropin binaries not built (no /root/reference here)")


def _run(args, timeout=900):
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    return p.returncode, p.stdout + p.stderr


@needs_bin
@pytest.mark.parametrize("suite", HOST_SUITES)
def test_reference_unit_suite_passes_against_b200_build(suite):
    rc, out = _run([UNIT, "-ts=" + suite])
    # wall-clock assertions in the reference suite (schema_test.cpp:346, graph build "scales
    # near-linearly") flake on a loaded shared host: only those may be retried, twice
    for _ in range(2):
        failed = [ln for ln in out.splitlines() if ": FAILED in " in ln or ": ERROR in " in ln]
        if rc == 0 or not failed or not all("scales near-linearly" in ln for ln in failed):
            break
        rc, out = _run([UNIT, "-ts=" + suite])
    assert rc == 0 and "0 failed" in out, out[-3000:]
    assert "test cases: 0 " not in out


@pytest.mark.gpu
@needs_bin
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_model_suites_pass_on_gpu(suite):
    rc, out = _run([UNIT, "-ts=" + suite])
    print(out[-2000:])
    assert rc == 0 and "0 failed" in out, out[-3000:]


@pytest.mark.gpu
@needs_bin
def test_reference_acceptance_gate_on_gpu():
    rc, out = _run([ACCEPT, DEMO], timeout=1800)
    print(out)
    assert "9/9 criteria passed" in out, out
