"""CPU-only checks of the boundary: the C-ABI library loads and exports every symbol
include/jz_knn.h declares; the binding declares exactly those; the product path refuses
to run without CUDA (no CPU fallback); the product package never imports oracle/."""
import ast
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "jz_knn.h")).read()
    return sorted(set(re.findall(r"^JZ_API [^(]*?\b(jz_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    from paper_2604_05885_b200 import _binding as B

    syms = _header_symbols()
    assert len(syms) >= 17
    lib = B.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(B.EXPORTS) == syms


def test_header_documents_each_entry_point():
    """Each declaration is preceded by a comment (argument meaning / layout / errors)."""
    src = open(os.path.join(ROOT, "include", "jz_knn.h")).read()
    lines = src.splitlines()
    for i, l in enumerate(lines):
        if l.startswith("JZ_API"):
            back = "\n".join(lines[max(0, i - 12):i])
            assert "*/" in back, l


def test_no_cpu_fallback():
    import torch

    import paper_2604_05885_b200 as jz

    with pytest.raises(TypeError):
        jz.KnnIndex(torch.zeros(10, 3))  # CPU tensor: refused
    if not torch.cuda.is_available():
        with pytest.raises(Exception):
            jz.knn_host(np.zeros((10, 3), np.float32), 2)  # no device: the library errors out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_05885_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
    # and the CUDA sources never include oracle code
    for f in os.listdir(os.path.join(pkg, "csrc")):
        for line in open(os.path.join(pkg, "csrc", f)):
            if line.lstrip().startswith("#include"):
                assert "oracle" not in line, (f, line)


def test_oracle_does_not_import_product():
    od = os.path.join(ROOT, "oracle")
    for f in os.listdir(od):
        path = os.path.join(od, f)
        if f.endswith(".py"):
            for node in ast.walk(ast.parse(open(path).read())):
                if isinstance(node, ast.Import):
                    assert not any("paper_2604_05885_b200" in a.name for a in node.names), f
                if isinstance(node, ast.ImportFrom):
                    assert "paper_2604_05885_b200" not in (node.module or ""), f
        if f.endswith(".c"):
            for line in open(path):
                if line.lstrip().startswith("#include"):
                    assert "csrc" not in line and "jz_knn" not in line, (f, line)
