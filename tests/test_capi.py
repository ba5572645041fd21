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


def _build_dropin(tmp_path):
    exe = os.path.join(str(tmp_path), "dropin_dense")
    libdir = os.path.dirname(V.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "dropin_dense.cpp"), "-L", libdir, "-lvoxl_b200",
           "-Wl,-rpath," + libdir, "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_binding_compiles_and_links(tmp_path):
    """include/voxl_b200.hpp: the reference-named C++ wrapper builds against the .so."""
    assert os.path.exists(_build_dropin(tmp_path))


import pytest as _pytest  # noqa: E402


@_pytest.mark.gpu
def test_cpp_dropin_driver_bitwise(tmp_path):
    import numpy as np

    import oracle as O

    exe = _build_dropin(tmp_path)
    out = os.path.join(str(tmp_path), "field.bin")
    r = subprocess.run([exe, out], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(out, np.float64)
    ref = O.port_dense_run("D3Q19", (16, 16, 16), 0.56, "lid_driven_cavity", (0.05, 0, 0), 20)
    assert np.array_equal(got, ref)


def test_host_io_conversion_exact(tmp_path):
    """fp32 wire-format conversions (host pool + AVX2 streaming stores) equal
    the scalar fp64 subtract / round / add for all widths and alignments."""
    import subprocess

    exe = str(tmp_path / "host_io_convert")
    src = os.path.join(ROOT, "tests", "cpp", "host_io_convert.cpp")
    inc = os.path.join(ROOT, "paper_2503_07898_b200", "csrc")
    subprocess.run(["g++", "-O3", "-std=c++17", "-pthread", "-ffp-contract=off", "-I" + inc, src, "-o", exe],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
