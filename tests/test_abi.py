"""CPU checks of the C-ABI boundary: libhfta.so loads without a GPU, exports
every function include/hfta.h declares, the binding covers exactly that set,
and calls fail loudly (no fallback) when no B200 is present."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hfta.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hfta_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2102_02344_b200 import build
    build.build()
    lib = ctypes.CDLL(build.LIB)
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_matches_header():
    import paper_2102_02344_b200.hfta as H
    assert sorted(H.EXPORTED) == header_functions()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2102_02344_b200.hfta as H
    with pytest.raises(H.HftaError) as e:
        H.hfta_init(0)
    assert e.value.code == 5          # HFTA_ERR_ARCH: no device, nothing runs
    with pytest.raises(H.HftaError) as e:
        H.hfta_fused_adam(1, 4, 0, 0, 0, 0, 4, 0, 0, 0, 0, 0, 0, None, 4, None)
    assert e.value.code == 8          # HFTA_ERR_NOT_INITIALIZED


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2102_02344_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), fn
