"""The C++ drop-in on the reference's own types, and the C++ `voxl_b200` driver.

* GPU: every shipped configuration (proj/configs/*.json, fixtures in
  tests/golden/configs) through the reference's voxl::run and through
  voxl::b200::run(const voxl::SolverConfig&) (include/voxl_b200_reference.hpp,
  fp64), both artifact sets written as the reference CLI writes them
  (main.cpp:30-55), plus the B200 C++ driver `voxl_b200 run`: fields.bin,
  fields.json, config.json, ledger.csv, trace.json, dispatch.json, graph.dot
  and distribution.txt byte-equal; diagnostics.csv to 1e-11 (the reference
  sums probe_field sequentially, the B200 probe exactly).
* CPU: the driver's configuration errors (ConfigError text and exit code 2 of
  main.cpp:260-263) and the C++ binding's run() validation
  (SolverConfig::validate, solver.cpp:27-60), which throw before any device
  work.
"""
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2503_07898_b200 as V

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = os.path.join(ROOT, "tests", "golden", "configs")
CLI = os.path.join(os.path.dirname(V.LIB_PATH), "voxl_b200")
NAMES = sorted(f[:-5] for f in os.listdir(CONFIGS) if f.endswith(".json"))
BYTE_EQUAL = ["fields.bin", "fields.json", "config.json", "ledger.csv", "trace.json", "dispatch.json", "graph.dot",
              "distribution.txt"]


def _diag_close(a, b):
    ra = [line.split(",") for line in a.strip().split("\n")]
    rb = [line.split(",") for line in b.strip().split("\n")]
    assert ra[0] == rb[0] == ["step", "mass", "max_u"]
    assert len(ra) == len(rb)
    for x, y in zip(ra[1:], rb[1:]):
        assert x[0] == y[0]
        for u, v in zip(x[1:], y[1:]):
            assert abs(float(u) - float(v)) <= 1e-11 * abs(float(v)), (x, y)


def _compare(dir_a, dir_b):
    files_a = sorted(os.listdir(dir_a))
    assert files_a == sorted(os.listdir(dir_b))
    for f in files_a:
        with open(os.path.join(dir_a, f), "rb") as fa, open(os.path.join(dir_b, f), "rb") as fb:
            a, b = fa.read(), fb.read()
        if f == "diagnostics.csv":
            _diag_close(a.decode(), b.decode())
        else:
            assert f in BYTE_EQUAL, f
            assert a == b, f"{f} differs"


@pytest.mark.gpu
@pytest.mark.skipif(O.dropin_driver() is None, reason="drop-in driver not built (needs the reference sources)")
def test_dropin_on_reference_types_and_cli_artifacts_equal_reference(tmp_path):
    cfgs = [os.path.join(CONFIGS, n + ".json") for n in NAMES]
    r = subprocess.run([O.dropin_driver(), str(tmp_path)] + cfgs, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stderr
    for n in NAMES:
        out = tmp_path / n
        c = subprocess.run([CLI, "run", "--config", os.path.join(CONFIGS, n + ".json"), "--out", str(out / "cli")],
                           capture_output=True, text=True, timeout=600)
        assert c.returncode == 0, c.stderr
        assert c.stdout.startswith("run complete: ")
        _compare(out / "b200", out / "ref")
        _compare(out / "cli", out / "ref")
        assert (out / "ref" / "fields.bin").stat().st_size > 0


@pytest.mark.gpu
def test_cli_verify_passes():
    r = subprocess.run([CLI, "verify"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all verification suites passed" in r.stdout
    assert "FAIL" not in r.stdout


@pytest.mark.gpu
def test_cli_fp32_run_within_tolerance(tmp_path):
    cfg = os.path.join(CONFIGS, "cavity32.json")
    for prec in ("fp64", "fp32"):
        r = subprocess.run([CLI, "run", "--config", cfg, "--out", str(tmp_path / prec), "--precision", prec],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr
    a = np.fromfile(tmp_path / "fp64" / "fields.bin", np.float64)
    b = np.fromfile(tmp_path / "fp32" / "fields.bin", np.float64)
    assert np.max(np.abs(b - a) / np.abs(a)) <= 1e-5


@pytest.mark.parametrize("text,expect", [
    ('{"tau": 0.4}', "configuration error: invalid configuration: tau must be > 0.5; "),
    ('{"scenario": "wind"}', "configuration error: unknown scenario: wind"),
    ('{"lattice": "D3Q15"}', "configuration error: configuration error: unknown lattice kind: D3Q15"),
    ('{"domain": [4]}', "configuration error: domain must be [nx, ny] or [nx, ny, nz]"),
    ('{"levels": 2, "scenario": "periodic_box", "velocity": [0.2, 0, 0]}',
     "configuration error: invalid configuration: |velocity| must be <= 0.1 (stability envelope); multi-level runs "
     "support the lid_driven_cavity scenario only; "),
    ('{"tau": ', "configuration error: configuration is not valid JSON: "),
])
def test_cli_configuration_errors(tmp_path, text, expect):
    """main.cpp:260-263: ConfigError -> 'configuration error: ' + what + the schema, exit 2."""
    p = tmp_path / "c.json"
    p.write_text(text)
    r = subprocess.run([CLI, "run", "--config", str(p), "--out", str(tmp_path / "o")], capture_output=True,
                       text=True, timeout=60)
    assert r.returncode == 2
    assert r.stderr.startswith(expect), r.stderr
    assert "configuration keys (JSON object):" in r.stderr
    assert not (tmp_path / "o").exists()


def test_cpp_binding_run_validates(tmp_path):
    """voxl::b200::run validates first (solver.cpp:370): ConfigError with the
    reference's text, no engine built for an invalid configuration."""
    src = tmp_path / "v.cpp"
    src.write_text(r'''
#include <iostream>
#include "voxl_b200.hpp"
int main() {
    voxl::b200::SolverConfig c;
    c.levels = 2;
    c.scenario = VOXL_PERIODIC;
    c.obstacle_radius = 0;
    c.perturbation = 0.7;
    try { voxl::b200::run(c); } catch (const voxl::b200::ConfigError& e) { std::cout << e.what(); return 0; }
    return 1;
}''')
    exe = tmp_path / "v"
    libdir = os.path.dirname(V.LIB_PATH)
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-L", libdir, "-lvoxl_b200",
                    "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    assert r.stdout == ("invalid configuration: multi-level runs support the lid_driven_cavity scenario only; "
                        "perturbation must be in [0, 0.5]; ")
