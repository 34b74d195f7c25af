"""CPU-only: the C-ABI library builds, loads and exports every symbol include/cqp_b200.h
declares; without a GPU the constructors fail loudly (no CPU fallback)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "cqp_b200.h")).read()
    return sorted(set(re.findall(r"CQP_API\s+[\w\s\*]+?\b(cqp_\w+)\s*\(", text)))


def test_header_declares_what_the_loader_binds():
    from paper_2311_18056_b200 import _lib
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2311_18056_b200 import _lib
    _lib.build()
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_no_cpu_fallback_without_device():
    from paper_2311_18056_b200 import _lib, solver as S
    lib = _lib.load()
    if lib.cqp_device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(S.CudaError):
        S.Solver([[2.0]], [-2.0], [[1.0]], [0.0], [0.5])


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2311_18056_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".hpp", ".cpp", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "clampqp_oracle" not in text, f
