"""The C-ABI library loads on a CPU host and exports every symbol that
include/negf_b200.h declares (no compute calls without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "negf_b200.h").read_text()
    return sorted(set(re.findall(r"\b(negf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "negf_rgf_selected_solve_batched" in syms
    assert len(syms) >= 5


def test_library_exports_declared_symbols():
    lib_path = ROOT / "paper_2508_19138_b200" / "libnegf_b200.so"
    if not lib_path.exists():
        pytest.fail("libnegf_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(lib_path))
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lib.negf_abi_version() >= 100


def test_python_binding_covers_header():
    from paper_2508_19138_b200 import _lib

    assert set(declared_symbols()) == set(_lib.exported_symbols())


def _header_arity():
    text = (ROOT / "include" / "negf_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(negf_[a-z0-9_]+)\s*\(([^)]*)\)\s*;", text):
        args = m.group(2).strip()
        out[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    return out


def test_python_binding_arity_matches_header():
    """ctypes silently accepts extra arguments, so check every binding's
    argument count against the C prototype."""
    from paper_2508_19138_b200 import _lib

    arity = _header_arity()
    for name, (_, args) in _lib._SIGNATURES.items():
        assert len(args) == arity[name], (name, len(args), arity[name])
