"""The C-ABI library builds, loads and exports every symbol declared in
include/glod_b200.h (no GPU needed; no compute calls)."""
from __future__ import annotations

import re

from paper_2507_01110_b200 import _lib

from .conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "glod_b200.h").read_text()
    return sorted(set(re.findall(r"\b(glod_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "glod_lod_select" in syms and "glod_spt_compact" in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"


def test_version_and_error_without_gpu():
    lib = _lib.load()
    assert lib.glod_version() >= 1
    assert isinstance(lib.glod_last_error(), bytes)
