"""Solver front-end (run / config / CLI artifacts) vs the reference's voxl::run."""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from paper_2503_07898_b200 import solver as S

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_config(text):
    lib = O.ref_lib()
    lib.vref_config_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int64]
    buf = C.create_string_buffer(1 << 16)
    n = lib.vref_config_roundtrip(text.encode(), buf, 1 << 16)
    return n >= 0, buf.value.decode()


BAD = ['{ not json', '{"tau": 0.4}', '{"velocity": [0.5, 0, 0]}', '{"domain": [16, 16, 16], "partitions": 9}',
       '{"scenario": "periodic_box", "levels": 2, "domain": [16,16,16]}', '{"lattice": "D2Q9"}',
       '{"domain": [4, 4, 4], "scenario": "flow_over_obstacle"}', '{"levels": 3, "domain": [18, 16, 16]}',
       '{"steps": -1, "perturbation": 0.7}']
GOOD = ['{"lattice": "D3Q19", "domain": [16, 16, 16], "tau": 0.56, "layout": "DisagSoA", "partitions": 2}',
        '{"lattice": "D2Q9", "domain": [64, 64], "tau": 0.6, "steps": 1000, "partitions": 4}',
        '{"scenario": "flow_over_obstacle", "strategy": "disag_mem", "tau": 0.7, "velocity": [0.04, 0, 0]}',
        '{"levels": 3, "fused": false, "seed": 7, "obstacle_radius": 3.5}']


@needs_ref
@pytest.mark.parametrize("text", BAD + GOOD)
def test_config_parse_validate_roundtrip_vs_reference(text):
    ok, ref = _ref_config(text)
    if not ok:
        with pytest.raises(S.ConfigError) as ei:
            S.config_from_json(text)
        if not text.startswith("{ not"):  # the JSON parser's own message text differs
            assert str(ei.value) == ref
    else:
        assert S.config_to_json(S.config_from_json(text)) == ref


@needs_ref
def test_cli_model_matches_reference_tables():
    lib = O.ref_lib()
    lib.vref_model_text.argtypes = [C.c_char_p, C.c_int64]
    buf = C.create_string_buffer(1 << 14)
    lib.vref_model_text(buf, 1 << 14)
    out = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "model"], capture_output=True, text=True,
                         cwd=ROOT).stdout
    lines = [x for x in out.splitlines() if not x.startswith("#")]
    assert "\n".join(lines) + "\n" == buf.value.decode()


def test_cli_ledger_and_config_error_exit_codes(tmp_path):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"lattice": "D3Q19", "domain": [16, 16, 16], "layout": "SoA", "partitions": 4,
                               "steps": 3}))
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "ledger", "--config", str(cfg)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "1,1,10,2560,10,2560,yes" in r.stdout  # SoA D3Q19: alpha 10, beta 10 s (Table 3)
    bad = tmp_path / "b.json"
    bad.write_text('{"tau": 0.3}')
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "run", "--config", str(bad)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 2 and "tau must be > 0.5" in r.stderr


@needs_ref
@pytest.mark.parametrize("name", ["dense", "sparse", "multires"])
def test_cli_report_on_reference_artifacts(name, tmp_path):
    """`report` (main.cpp:186-229) over a directory holding the reference run's own
    artifacts: one line per artifact, in the reference's wording."""
    cfg = CASES[name]
    ref = O.RefRun(cfg)
    (tmp_path / "config.json").write_text(json.dumps(cfg))
    (tmp_path / "diagnostics.csv").write_text(ref.diagnostics_csv)
    expect = [f"report for {tmp_path}",
              f"  scenario: {cfg['scenario']}, lattice {cfg['lattice']}, domain 16x16x16, steps {cfg['steps']}",
              "  final diagnostics (step,mass,max_u): " + ref.diagnostics_csv.strip().split("\n")[-1]]
    rows = [ln for ln in ref.ledger_csv.split("\n")[1:] if ln]
    if rows:
        (tmp_path / "ledger.csv").write_text(ref.ledger_csv)
        expect.append(f"  ledger: {len(rows)} transfer records, "
                      f"{sum(int(r.rsplit(',', 1)[1]) for r in rows)} elements total")
    if ref.dispatch_json:
        (tmp_path / "dispatch.json").write_text(ref.dispatch_json)
        expect += ("  dispatch: " + ref.dispatch_json).rstrip("\n").split("\n")
    if ref.distribution:
        (tmp_path / "distribution.txt").write_text(ref.distribution)
        expect += ("  level distribution (% of finest cells): " + ref.distribution).rstrip("\n").split("\n")
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "report", "--dir", str(tmp_path)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert r.stdout.rstrip("\n").split("\n") == expect
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "report", "--dir", str(tmp_path / "nope")],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 2 and "directory not found" in r.stderr


# ---- GPU: run() vs voxl::run ---------------------------------------------------------

CASES = {
    "dense": dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.56, scenario="lid_driven_cavity",
                  velocity=[0.05, 0, 0], steps=12, layout="DisagSoA", partitions=3),
    "dense_soa_2d": dict(lattice="D2Q9", domain=[24, 20], tau=0.6, scenario="lid_driven_cavity",
                         velocity=[0.05, 0, 0], steps=15, layout="SoA", partitions=2),
    "periodic": dict(lattice="D3Q19", domain=[12, 12, 12], tau=0.8, scenario="periodic_box", velocity=[0, 0, 0],
                     steps=10, partitions=2, perturbation=0.05, seed=99),
    "sparse": dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.7, scenario="flow_over_obstacle",
                   velocity=[0.04, 0, 0], steps=8, strategy="disag_bitmask"),
    "multires": dict(lattice="D3Q19", domain=[16, 16, 16], tau=0.56, scenario="lid_driven_cavity",
                     velocity=[0.05, 0, 0], steps=3, levels=2, fused=True),
    "multires_2d": dict(lattice="D2Q9", domain=[32, 32], tau=0.6, scenario="lid_driven_cavity",
                        velocity=[0.05, 0, 0], steps=4, levels=3, fused=True),
    "multires_2d_staged": dict(lattice="D2Q9", domain=[48, 32], tau=0.6, scenario="lid_driven_cavity",
                               velocity=[0.05, 0, 0], steps=3, levels=2, fused=False),
}


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name", list(CASES))
def test_run_matches_reference_run(name, tmp_path):
    cfg = CASES[name]
    ref = O.RefRun(cfg)
    c = S.config_from_json(json.dumps({**cfg, "precision": "fp64"}))
    res = S.run(c)
    assert np.array_equal(res.field, ref.field)
    assert len(res.diagnostics) == len(ref.diagnostics)
    # mass: the reference sums sequentially (error ~ N eps |m|), the device
    # reduces pairwise; fields are compared bitwise above.
    for (s, m, u), (rs, rm, ru) in zip(res.diagnostics, ref.diagnostics):
        assert s == rs and abs(m - rm) <= 1e-11 * abs(rm) and abs(u - ru) <= 1e-14
    assert res.ledger_csv() == ref.ledger_csv if ref.ledger_csv.count("\n") > 1 else True
    assert (res.trace_json() if res.trace else "") == (ref.trace_json if ref.trace_json.strip() != "[\n]" else "")
    assert res.dispatch_json == ref.dispatch_json
    assert res.graph_dot == ref.graph_dot
    assert res.distribution == ref.distribution
    assert res.field_header_json == ref.header_json


@pytest.mark.gpu
def test_cli_run_writes_reference_artifacts(tmp_path):
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({**CASES["dense"], "precision": "fp64"}))
    out = tmp_path / "out"
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "run", "--config", str(cfg), "--out",
                        str(out)], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    for f in ("fields.bin", "fields.json", "diagnostics.csv", "config.json", "ledger.csv", "trace.json"):
        assert (out / f).exists(), f
    ref = O.port_dense_run("D3Q19", (16, 16, 16), 0.56, "lid_driven_cavity", (0.05, 0, 0), 12)
    assert np.array_equal(np.fromfile(out / "fields.bin", np.float64), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("parts", [1, 3])
def test_step_probe_equals_step_plus_probe(precision, parts):
    import paper_2503_07898_b200 as V

    init = O.port_initial_state("D3Q19", (24, 20, 18))
    a = V.DenseEngine(domain=(24, 20, 18), precision=precision, partitions=parts)
    b = V.DenseEngine(domain=(24, 20, 18), precision=precision, partitions=parts)
    a.set_canonical(init)
    b.set_canonical(init)
    # fp64: same values, only the summation order differs. fp32: the fused
    # probe forms each voxel's moments from the shifted fp32 populations in
    # fp32 (probe() promotes every population to fp64 first), so the
    # diagnostics row agrees to fp32 moment rounding.
    tol_m, tol_u = (1e-12, 1e-12) if precision == "fp64" else (1e-9, 1e-6)
    for _ in range(7):
        da = a.step_probe()
        b.step(1)
        db = b.probe()
        assert abs(da.mass - db.mass) <= tol_m * db.mass
        assert abs(da.max_speed - db.max_speed) <= tol_u * db.max_speed + 1e-12
    assert np.array_equal(a.get_canonical(), b.get_canonical())


@pytest.mark.gpu
def test_cli_run_observed_trace(tmp_path):
    """`run --observed-trace` adds trace_observed.json: one record per launched
    phase of every step (single-stream schedule: one "step" kernel per
    partition), device-timed; the reference's logical trace.json is unchanged."""
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({**CASES["dense"], "precision": "fp64", "partitions": 2}))
    out = tmp_path / "out"
    r = subprocess.run([sys.executable, "-m", "paper_2503_07898_b200", "run", "--config", str(cfg), "--out",
                        str(out), "--observed-trace"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    rec = json.loads((out / "trace_observed.json").read_text())
    steps = json.loads(cfg.read_text())["steps"]
    assert [(x["step"], x["phase"], x["partition"]) for x in rec] == [(s, "step", p) for s in range(steps)
                                                                        for p in range(2)]
    assert all(0.0 <= x["begin_ms"] <= x["end_ms"] for x in rec)
    assert (out / "trace.json").exists()


@pytest.mark.gpu
def test_cpp_cli_run_observed_trace(tmp_path):
    """The C++ driver's `run --observed-trace` (voxl::b200::run with
    SolverConfig::observed_trace) writes the same executed-schedule record."""
    exe = os.path.join(ROOT, "paper_2503_07898_b200", "_lib", "voxl_b200")
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({**CASES["dense"], "partitions": 2}))
    out = tmp_path / "out"
    r = subprocess.run([exe, "run", "--config", str(cfg), "--out", str(out), "--precision", "fp64",
                        "--observed-trace"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    rec = json.loads((out / "trace_observed.json").read_text())
    steps = json.loads(cfg.read_text())["steps"]
    assert [(x["step"], x["partition"]) for x in rec] == [(s, p) for s in range(steps) for p in range(2)]
    assert all(x["phase"] == "step" and 0.0 <= x["begin_ms"] <= x["end_ms"] for x in rec)
