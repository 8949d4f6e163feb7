"""CPU-side checks of the boundary: libsand.so loads and exports every symbol include/sand.h
declares; argument validation that needs no GPU; the product package never imports the oracle."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sand.h")
PKG = os.path.join(ROOT, "paper_2604_25936_b200")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(sand_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_entry_points():
    names = _declared()
    for f in ("sand_create", "sand_load_weights", "sand_load_depthmap", "sand_query"):
        assert f in names


def test_library_builds_loads_and_exports_every_declared_symbol():
    from paper_2604_25936_b200 import build, load_library
    from paper_2604_25936_b200.sand import EXPORTS
    lib_path = build.build(verbose=False)
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path]).decode()
    exported = set(re.findall(r" T (sand_\w+)", out))
    for name in _declared():
        assert name in exported, name
        assert name in EXPORTS, f"binding lacks {name}"
    lib = load_library()
    assert lib.sand_abi_version() == 1


def test_create_fails_loudly_without_gpu_or_bad_args():
    import torch
    from paper_2604_25936_b200 import SandContext, SandError
    with pytest.raises(SandError) as e:
        SandContext(L=0, H=64)
    assert e.value.code == -1
    with pytest.raises(SandError) as e:
        SandContext(L=4, H=100, prec=2)
    assert e.value.code == -7
    if not torch.cuda.is_available():
        with pytest.raises(SandError) as e:
            SandContext(L=4, H=64, prec=2)
        assert e.value.code == -5   # SAND_ERR_CUDA: no CPU path exists


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", f
