"""The C-ABI library loads and exports every symbol include/voxl_b200.h declares."""
import ctypes
import os
import re
import subprocess

import paper_2503_07898_b200 as V

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "voxl_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(voxl_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = ctypes.CDLL(V.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_exports_are_plain_c():
    out = subprocess.run(["nm", "-D", "--defined-only", V.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (voxl_\w+)$", out, re.M))
    assert set(declared_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", V.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_status_and_message():
    import pytest

    with pytest.raises(V.VoxlInvalidArgument, match="unknown lattice"):
        V.lattice_json(7)
