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


def test_null_handles_and_buffers_are_invalid_arguments():
    """No CPU-side crash on a null handle or buffer: every handle entry point
    returns VOXL_INVALID_ARGUMENT with the entry point's name (no GPU touched)."""
    import ctypes as C

    from paper_2503_07898_b200._capi import INVALID_ARGUMENT, lib

    for fn, args in [("voxl_dense_step", (None, 1)), ("voxl_dense_set_canonical", (None, None)),
                     ("voxl_dense_get_canonical", (None, None)), ("voxl_sparse_step", (None, 1)),
                     ("voxl_sparse_get_state", (None, None)), ("voxl_mres_step", (None, 1)),
                     ("voxl_mres_set_state", (None, None))]:
        f = getattr(lib, fn)
        assert f(*[C.c_void_p(a) if a is None else a for a in args]) == INVALID_ARGUMENT, fn
        assert lib.voxl_last_error().decode() == fn + ": null argument"


def _build_dropin(tmp_path, name="dropin_dense"):
    exe = os.path.join(str(tmp_path), name)
    libdir = os.path.dirname(V.LIB_PATH)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", libdir, "-lvoxl_b200",
           "-Wl,-rpath," + libdir, "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_binding_compiles_and_links(tmp_path):
    """include/voxl_b200.hpp: the reference-named C++ wrapper (engines and
    run()) builds against the .so."""
    assert os.path.exists(_build_dropin(tmp_path))
    assert os.path.exists(_build_dropin(tmp_path, "dropin_run"))


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


@_pytest.mark.gpu
def test_cpp_run_dropin_matches_oracle_and_python(tmp_path):
    """voxl::b200::run (C++, solver.cpp:369-375 shape) on the three engines:
    fields bitwise equal to the oracle, diagnostics equal to the Python
    front-end's run(), and the reference's abort text on an unstable run."""
    import numpy as np

    import oracle as O
    from paper_2503_07898_b200 import solver as S

    exe = _build_dropin(tmp_path, "dropin_run")
    prefix = os.path.join(str(tmp_path), "run")
    r = subprocess.run([exe, prefix], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "run aborted at step" in r.stdout
    field = lambda n: np.fromfile(f"{prefix}_{n}.bin", np.float64)  # noqa: E731
    diag = lambda n: np.loadtxt(f"{prefix}_{n}.csv", delimiter=",", ndmin=2)  # noqa: E731
    dom = (16, 16, 16)
    assert np.array_equal(field("dense"), O.port_dense_run("D3Q19", dom, 0.56, "lid_driven_cavity", (0.05, 0, 0), 12))
    act = O.obstacle_mask(dom)
    sref = O.sparse_canonical(dom, act, O.port_sparse_run("D3Q19", dom, 0.7, (0.04, 0, 0), 5, act), 19)
    assert np.array_equal(field("sparse"), sref)
    assert np.array_equal(field("multires"), O.port_mres_run("D3Q19", dom, 2, 0.56, (0.05, 0.0, 0.0), 2))
    assert np.array_equal(field("multires2d"), O.port_mres_run("D2Q9", (32, 32, 1), 3, 0.6, (0.05, 0.0, 0.0), 3,
                                                               level_map=O.band_level_map((32, 32, 1), 3, 1)))
    cfgs = {"dense": dict(steps=12, partitions=2),
            "sparse": dict(scenario="flow_over_obstacle", tau=0.7, velocity=[0.04, 0, 0], steps=5,
                           strategy="disag_mem"),
            "multires": dict(levels=2, steps=2)}
    for name, kw in cfgs.items():
        base = dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.56, scenario="lid_driven_cavity",
                    velocity=[0.05, 0, 0])
        base.update(kw)
        c = S.SolverConfig(**base)
        c.domain = tuple(c.domain)
        c.velocity = tuple(c.velocity)
        c.precision = "fp64"
        py = S.run(c)
        got = diag(name)
        assert got.shape[0] == len(py.diagnostics)
        for (st, m, u), row in zip(py.diagnostics, got):
            assert int(row[0]) == st and row[1] == m and row[2] == u, name
