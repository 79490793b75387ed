"""Static checks of the oracle / product separation (task rule: the oracle and
the CUDA path share no code; only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg -- plus its reference arm -- may touch oracle/; the product
path never does)."""

import ast
import glob
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _oracle_imports(path):
    """(enclosing function name or None, line) of every import of `oracle`."""
    tree = ast.parse(open(path).read())
    out = []

    def visit(node, fn):
        for child in ast.iter_child_nodes(node):
            name = child.name if isinstance(child, (ast.FunctionDef, ast.AsyncFunctionDef)) else fn
            if isinstance(child, ast.Import) and any(a.name.split(".")[0] == "oracle" for a in child.names):
                out.append((fn, child.lineno))
            if isinstance(child, ast.ImportFrom) and (child.module or "").split(".")[0] == "oracle":
                out.append((fn, child.lineno))
            visit(child, name)
    visit(tree, None)
    return out


def test_product_package_never_imports_the_oracle():
    for path in glob.glob(os.path.join(ROOT, "paper_1605_08325_b200", "**", "*.py"), recursive=True):
        assert not _oracle_imports(path), path
    for path in glob.glob(os.path.join(ROOT, "paper_1605_08325_b200", "csrc", "*")):
        incs = [l for l in open(path, errors="ignore") if l.lstrip().startswith("#include")]
        assert not any("oracle" in l for l in incs), path


def test_oracle_never_imports_the_product():
    for path in glob.glob(os.path.join(ROOT, "oracle", "*.py")):
        src = open(path).read()
        tree = ast.parse(src)
        for node in ast.walk(tree):
            if isinstance(node, ast.ImportFrom):
                assert not (node.module or "").startswith("paper_1605_08325_b200"), path
            if isinstance(node, ast.Import):
                assert not any(a.name.startswith("paper_1605_08325_b200") for a in node.names), path


def test_bench_touches_the_oracle_only_in_its_cpu_baseline_leg_and_reference_arm():
    allowed = {"run_reference", "cpu_baseline", "check_sample"}
    found = _oracle_imports(os.path.join(ROOT, "bench.py"))
    assert found, "the cpu_baseline leg imports the oracle"
    assert all(fn in allowed for fn, _ in found), found
    # check_sample is called from the cpu_baseline leg only
    tree = ast.parse(open(os.path.join(ROOT, "bench.py")).read())
    callers = set()
    for fn in [n for n in ast.walk(tree) if isinstance(n, ast.FunctionDef)]:
        for node in ast.walk(fn):
            if isinstance(node, ast.Call) and getattr(node.func, "id", None) == "check_sample":
                callers.add(fn.name)
    assert callers == {"cpu_baseline"}, callers


def test_graft_entry_uses_the_oracle_only_in_smoke():
    found = _oracle_imports(os.path.join(ROOT, "__graft_entry__.py"))
    assert found and all(fn == "smoke" for fn, _ in found), found
