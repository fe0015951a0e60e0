"""bench.py's driver contract, checked on CPU: both arms print BASELINE.json's metric string (the
driver refuses the ours / reference ratio otherwise), and the reference arm's code path never loads
this repo's native library (its line must time only the unchanged reference, oracle/_ref)."""
import ast
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _bench_source():
    with open(os.path.join(ROOT, "bench.py")) as f:
        return f.read()


def test_metric_is_baseline_metric_for_both_arms():
    import bench

    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert bench.METRIC == json.load(f)["metric"]
    tree = ast.parse(_bench_source())
    # every JSON line's "metric" key is the shared constant, never a literal of its own
    for node in ast.walk(tree):
        if isinstance(node, ast.Dict):
            for k, v in zip(node.keys, node.values):
                if isinstance(k, ast.Constant) and k.value == "metric":
                    assert isinstance(v, ast.Name) and v.id == "METRIC", ast.dump(v)


def _functions(tree):
    return {n.name: n for n in ast.walk(tree) if isinstance(n, ast.FunctionDef)}


def _imports_native(fn, funcs, seen=None):
    """True when fn, or a module-level function it calls, imports paper_2601_08743_b200.native."""
    seen = seen if seen is not None else set()
    if fn.name in seen:
        return False
    seen.add(fn.name)
    for node in ast.walk(fn):
        if isinstance(node, ast.ImportFrom) and node.module and node.module.startswith("paper_2601_08743_b200"):
            if any(a.name == "native" for a in node.names) or node.module.endswith(".native"):
                return True
        if isinstance(node, ast.Import) and any("native" in a.name for a in node.names):
            return True
        if isinstance(node, ast.Call) and isinstance(node.func, ast.Name) and node.func.id in funcs:
            if _imports_native(funcs[node.func.id], funcs, seen):
                return True
    return False


def test_reference_arm_never_loads_native_library():
    tree = ast.parse(_bench_source())
    funcs = _functions(tree)
    assert "reference_arm" in funcs
    assert not _imports_native(funcs["reference_arm"], funcs)
    # module level: importing bench must not pull in the native library either
    for node in tree.body:
        if isinstance(node, (ast.Import, ast.ImportFrom)):
            names = [a.name for a in node.names]
            assert "native" not in names and not any(n.endswith(".native") for n in names)


def test_importing_bench_does_not_load_libtkv():
    # a fresh interpreter: other tests in this process may have loaded the library already
    import subprocess

    code = "import sys; sys.path.insert(0, %r); import bench; print('libtkv.so' in open('/proc/self/maps').read())" % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == "False"
