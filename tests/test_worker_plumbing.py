"""CPU check of the multi-process GPU tests' plumbing (no GPU needed).

`tests/test_gpu_multidevice.py` runs only on a box with >= 2 GPUs, which the
development pool never has, and it reuses the workers of `tests/test_gpu_ipc.py`.
So that its argument plumbing cannot rot unseen, this test parses both files and
checks that every `run_workers(target, world, pre=..., post=...)` call passes the
target exactly the positional arguments its signature takes:
`target(rank, world, port, *pre, q, *post)` (see `run_workers`).
"""
import ast
import os

ROOT = os.path.dirname(os.path.abspath(__file__))
FILES = ("test_gpu_ipc.py", "test_gpu_multidevice.py")


def _defs():
    out = {}
    for f in FILES:
        tree = ast.parse(open(os.path.join(ROOT, f)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.FunctionDef) and node.name.startswith("_") and node.name.endswith("worker"):
                a = node.args
                out[node.name] = (len(a.args) - len(a.defaults), len(a.args))
    return out


def _calls():
    for f in FILES:
        tree = ast.parse(open(os.path.join(ROOT, f)).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Call) and getattr(node.func, "id", None) == "run_workers":
                kw = {k.arg: k.value for k in node.keywords}
                n_pre = len(kw["pre"].elts) if "pre" in kw else 0
                n_post = len(kw["post"].elts) if "post" in kw else 0
                yield f, node.lineno, node.args[0].id, 3 + n_pre + 1 + n_post


def test_run_workers_calls_match_worker_signatures():
    defs = _defs()
    calls = list(_calls())
    assert len(calls) >= 10
    for f, line, target, n in calls:
        assert target in defs, f"{f}:{line}: unknown worker {target}"
        lo, hi = defs[target]
        assert lo <= n <= hi, f"{f}:{line}: {target} takes {lo}..{hi} positional args, run_workers passes {n}"
