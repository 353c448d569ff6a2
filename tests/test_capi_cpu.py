"""CPU-side checks of the C-ABI boundary (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oscar_kv.h")
LIB = os.path.join(ROOT, "paper_2605_19660_b200", "liboscar_b200.so")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(oscar_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("library not built (run __graft_entry__.build())")
    L = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []


def test_python_binding_covers_header():
    from paper_2605_19660_b200.kv_cache import C_ABI_SYMBOLS

    assert sorted(C_ABI_SYMBOLS) == declared_symbols()


def test_config_validation_without_gpu():
    """PipelineConfig::validate semantics (kv_cache.cpp:51-67) run host-only."""
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    from paper_2605_19660_b200 import PipelineConfig

    PipelineConfig(heads=8).validate()
    for bad in (dict(residual_len=100), dict(bits=5), dict(heads=0), dict(head_dim=48),
                dict(bits=3), dict(head_dim=64)):
        with pytest.raises(ValueError):
            PipelineConfig(**bad).validate()
